"""Per-source-line warp-stall samples from `ncu --page source --csv --print-source cuda,sass`."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out, f = [], None
hdr = None
for r in rows:
    if r and r[0] == "File Path":
        f = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No":
        hdr = r; continue
    if not r or r[0] in ("", "Function Name") or hdr is None:
        continue
    try:
        s = int(r[4])
    except ValueError:
        continue
    stalls = {hdr[i]: r[i] for i in range(len(hdr)) if hdr[i].startswith("stall_") and "Not Issued" not in hdr[i]}
    top = sorted(((int(v), k[6:]) for k, v in stalls.items() if v.isdigit()), reverse=True)[:3]
    out.append((s, f, r[0], r[1][:70], top))
tot = sum(o[0] for o in out)
print("total samples", tot)
for s, f, ln, src, top in sorted(out, reverse=True)[:n]:
    print(f"{100*s/tot:5.1f}% {f}:{ln:5s} {src:70s} {top}")
