"""Per-kernel share of an ncu launch list (--metrics gpu__time_duration.sum --csv):
    python tools/launch_shares.py gpurun_out/x_launches.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
tot, cnt = collections.Counter(), collections.Counter()
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = d["Kernel Name"].split("(")[0].split("<")[0].replace("void ", "")
        v = float(d["Metric Value"].replace(",", ""))
        v *= {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6}.get(d.get("Metric Unit", "nsecond"), 1.0)
        tot[k] += v
        cnt[k] += 1
T = sum(tot.values())
for k, v in tot.most_common(16):
    print(f"{k:28s} {cnt[k]:6d} launches {v / 1e6:10.3f} ms {100 * v / T:6.1f} %")
