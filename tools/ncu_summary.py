"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list by kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            k = d["Kernel Name"].split("(")[0][:70]
            unit = d.get("Metric Unit", "nsecond")
            v = float(d["Metric Value"].replace(",", ""))
            v *= {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(unit, 1e-3)
            agg[k][0] += 1
            agg[k][1] += v
tot = sum(v[1] for v in agg.values())
print(f"{'us':>12} {'share':>6} {'n':>4}  kernel")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{v[1]:12.1f} {100 * v[1] / tot:5.1f}% {v[0]:4d}  {k}")
print(f"total {tot / 1e3:.3f} ms over {sum(v[0] for v in agg.values())} launches")
