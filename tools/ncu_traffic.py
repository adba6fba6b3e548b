"""Per-kernel time and DRAM traffic from an ncu CSV with gpu__time_duration,
dram__bytes_read.sum and dram__bytes_write.sum."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.defaultdict(lambda: collections.defaultdict(float))
cnt = collections.Counter()
# times normalised to microseconds, bytes to bytes
units = {"ns": 1e-3, "us": 1.0, "ms": 1e3, "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "KB": 1e3, "MB": 1e6, "GB": 1e9,
         "Gbyte": 1e9, "Tbyte": 1e12}
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        k = d["Kernel Name"].split("(")[0][:60]
        v = float(d["Metric Value"].replace(",", "")) * units.get(d.get("Metric Unit", ""), 1.0)
        agg[k][d["Metric Name"]] += v
        if d["Metric Name"] == "gpu__time_duration.sum":
            cnt[k] += 1
if "--json" in sys.argv:
    # per kernel family (template arguments dropped): DRAM bytes and time per launch
    import json
    fam = collections.defaultdict(lambda: [0.0, 0.0, 0])
    for k, a in agg.items():
        name = k.split("<")[0].replace("void ", "").replace("sg::", "").strip()
        targs = k.split("<")[1].split(",") if "<" in k else []
        if name in ("k_hash_warp", "k_hash_block", "k_bitmap") and len(targs) > 1 and targs[1].strip() == "0":
            name += ":count"  # MODE 0 = counting pass (sg_kernel_time naming)
        f = fam[name]
        f[0] += a["dram__bytes_read.sum"] + a["dram__bytes_write.sum"]
        f[1] += a["gpu__time_duration.sum"]
        f[2] += cnt[k]
    print(json.dumps({k: {"dram_bytes_per_launch": v[0] / v[2], "us_per_launch": v[1] / v[2], "launches": v[2],
                          "dram_bytes_per_step": v[0], "us_per_step": v[1]}
                      for k, v in fam.items()}, indent=1))
    sys.exit(0)
tot_t = sum(a["gpu__time_duration.sum"] for a in agg.values())
print(f"{'ms':>9} {'share':>6} {'DRAM GB':>8} {'GB/s':>7}  kernel  (ncu: serialised, cold cache)")
for k, a in sorted(agg.items(), key=lambda x: -x[1]["gpu__time_duration.sum"])[:int(sys.argv[2]) if len(sys.argv) > 2 else 15]:
    t = a["gpu__time_duration.sum"] / 1e3  # ms
    b = (a["dram__bytes_read.sum"] + a["dram__bytes_write.sum"]) / 1e9
    print(f"{t:9.3f} {100 * a['gpu__time_duration.sum'] / tot_t:5.1f}% {b:8.2f} {b / max(t, 1e-9) * 1e3:7.0f}  {k} (x{cnt[k]})")
print(f"total {tot_t / 1e3:.2f} ms")
