"""Top SASS instructions / regions of an ncu source page (sass) CSV by
instructions executed and stall samples: python tools/sass_hot.py file.csv"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    try:
        ie = float(r[ix["Instructions Executed"]] or 0)
        st = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    except ValueError:
        continue
    data.append((r[ix["Address"]], r[ix["Source"]], ie, st))
tot_ie = sum(d[2] for d in data)
tot_st = sum(d[3] for d in data)
print(f"total inst {tot_ie:.3e}  stall samples {tot_st:.0f}")
# windows of 16 instructions
W = 24
best = []
for i in range(0, len(data), W):
    seg = data[i:i + W]
    best.append((sum(d[3] for d in seg), sum(d[2] for d in seg), i))
best.sort(reverse=True)
for st, ie, i in best[:int(sys.argv[2]) if len(sys.argv) > 2 else 8]:
    print(f"== region @{data[i][0]}  stall {100*st/tot_st:.1f}%  inst {100*ie/tot_ie:.1f}%")
    for d in data[i:i + W]:
        print(f"   {d[0]:>6} {d[2]:10.3e} {d[3]:7.0f}  {d[1][:90]}")
