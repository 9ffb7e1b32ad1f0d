"""Summarise an ncu launch list and full captures into profiles/<tag>_summary.md."""
import csv, collections, json, statistics, sys
from pathlib import Path

tag = sys.argv[1]
G = Path("gpurun_out")
out = [f"# ncu summary ({tag})", ""]

def raw(path):
    rows = list(csv.reader(open(path)))
    return {rows[0][i]: (rows[2][i], rows[1][i]) for i in range(len(rows[0]))}

lp = G / f"{tag}_launches.csv"
if lp.exists():
    rows = list(csv.reader(l for l in open(lp) if not l.startswith("==")))
    h = rows[0]; iname, ival = h.index("Kernel Name"), h.index("Metric Value")
    d = collections.defaultdict(list)
    for r in rows[1:]:
        try: d[r[iname][:70]].append(float(r[ival].replace(",", "")))
        except ValueError: pass
    tot = sum(sum(v) for v in d.values())
    out += ["## Launch list (`--metrics gpu__time_duration.sum --clock-control none`, serialised, cold cache)", "",
            "| kernel | launches | total ms | mean us | share |", "|---|---:|---:|---:|---:|"]
    for k, v in sorted(d.items(), key=lambda x: -sum(x[1])):
        out.append(f"| `{k}` | {len(v)} | {sum(v)/1e6:.3f} | {statistics.mean(v)/1e3:.2f} | {100*sum(v)/tot:.1f}% |")
    out.append("")

for name, label in (("stream", "persistent decode kernel `k_decode_streams` (config b)"),
                    ("hsq", "HS + MaxEnt query kernel `k_word_logprob_ring` (config d, fast mode)")):
    p = G / f"{tag}_{name}_raw.csv"
    if not p.exists():
        continue
    m = raw(p)
    keys = ["gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
            "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
            "lts__t_sector_hit_rate.pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__inst_executed.avg.per_cycle_active",
            "smsp__issue_active.avg.per_cycle_active", "sm__warps_active.avg.per_cycle_active",
            "smsp__inst_executed.sum"]
    out += [f"## {label}: `ncu --set full`", "", "| metric | value | unit |", "|---|---:|---|"]
    for k in keys:
        if k in m:
            out.append(f"| {k} | {m[k][0]} | {m[k][1]} |")
    out.append("")

sp = G / f"{tag}_stream_src.csv"
if sp.exists():
    rows = list(csv.reader(open(sp)))
    f = hdr = None; agg = []
    for r in rows:
        if r and r[0] == "File Path": f = r[1].split("/")[-1]; continue
        if r and r[0] == "Line No": hdr = r; continue
        if not r or r[0] in ("", "Function Name") or hdr is None: continue
        try: agg.append((int(r[7]), int(r[4]), f, r[0], r[1][:90]))
        except (ValueError, IndexError): pass
    ti = sum(a[0] for a in agg) or 1; ts = sum(a[1] for a in agg) or 1
    out += ["## `k_decode_streams`: top source lines by executed warp instructions", "",
            "| % inst | % stall samples | line | source |", "|---:|---:|---|---|"]
    for a in sorted(agg, reverse=True)[:20]:
        out.append(f"| {100*a[0]/ti:.1f} | {100*a[1]/ts:.1f} | {a[2]}:{a[3]} | `{a[4].strip()}` |")
    out.append("")
Path(f"profiles/{tag}_summary.md").write_text("\n".join(out) + "\n")
print("\n".join(out[:60]))
