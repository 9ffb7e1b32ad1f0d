import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ia, isrc, iss = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[2:]:
    if len(r) <= iss: continue
    try: s = int(r[iss])
    except: s = 0
    data.append((r[ia], r[isrc], s))
tot = sum(d[2] for d in data)
print("total samples", tot, "instructions", len(data))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
top = sorted(range(len(data)), key=lambda i: -data[i][2])[:n]
for i in sorted(top):
    print(f"{i:5d} {data[i][0]} {data[i][2]:6d} {100*data[i][2]/tot:5.1f}%  {data[i][1][:90]}")
