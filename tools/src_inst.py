"""Per-source-line executed warp instructions from `ncu --page source --print-source cuda,sass` CSV."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
f = None
hdr = None
out = []
for r in rows:
    if r and r[0] == "File Path":
        f = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No":
        hdr = r; continue
    if not r or r[0] in ("", "Function Name") or hdr is None:
        continue
    try:
        ie = int(r[7])
    except (ValueError, IndexError):
        continue
    out.append((ie, f, r[0], r[1][:80]))
tot = sum(o[0] for o in out)
print("total warp instructions", tot)
for ie, f, ln, src in sorted(out, reverse=True)[:n]:
    print(f"{100*ie/tot:5.1f}% {ie:12d} {f}:{ln:5s} {src}")
