"""Top source lines by warp-stall samples from `ncu -i REP --page source --csv
--print-source cuda,sass` output:  python tools/ncu_lines.py FILE.csv [N]"""
import csv
import sys

rows, cur, hdr = [], None, None
with open(sys.argv[1], newline="") as f:
    for r in csv.reader(f):
        if not r:
            continue
        if r[0] == "File Path":
            cur = r[1].rsplit("/", 1)[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr and r[0] and r[0].isdigit():
            d = dict(zip(hdr[2:], r[2:]))
            try:
                s = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
            except ValueError:
                continue
            stalls = {k: int(v) for k, v in d.items() if k.startswith("stall_") and "Not Issued" not in k and v.isdigit() and int(v) > 0}
            top = sorted(stalls.items(), key=lambda kv: -kv[1])[:3]
            rows.append((s, cur, int(r[0]), r[1].strip()[:70], top))
tot = sum(x[0] for x in rows)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
print(f"total samples {tot}")
for s, fn, ln, src, top in sorted(rows, key=lambda x: -x[0])[:n]:
    print(f"{100 * s / tot:5.1f}% {fn}:{ln}  {src}  {top}")
