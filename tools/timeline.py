"""GPU timeline of one spgemm step (torch profiler / CUPTI; no nsys here):
python tools/timeline.py CONFIG [reps] -> per-step GPU busy time, idle gaps
and the largest gaps with the activities around them."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2604_19004_b200 import EngineConfig, matgen, spgemm  # noqa: E402
from paper_2604_19004_b200.device import to_device  # noqa: E402

name = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
a, b = matgen.make_config(name)
dev = torch.device("cuda", 0)
A = to_device(a, dev)
B = A if b is a else to_device(b, dev)
cfg = EngineConfig(return_device=True)
for _ in range(3):
    c, rep = spgemm(A, B, cfg)
    del c
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for _ in range(reps):
        c, rep = spgemm(A, B, cfg)
        del c
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
t1 = max(e.time_range.end for e in ev)
busy = []
for e in ev:
    s, f = e.time_range.start, e.time_range.end
    if busy and s <= busy[-1][1]:
        busy[-1][1] = max(busy[-1][1], f)
    else:
        busy.append([s, f])
tot_busy = sum(f - s for s, f in busy)
print(f"{reps} steps: span {(t1 - t0) / 1e3:.3f} ms, GPU busy {tot_busy / 1e3:.3f} ms, "
      f"idle {(t1 - t0 - tot_busy) / 1e3:.3f} ms, {len(ev)} device activities")
gaps = []
for i in range(1, len(busy)):
    g = busy[i][0] - busy[i - 1][1]
    gaps.append((g, busy[i - 1][1], busy[i][0]))
gaps.sort(reverse=True)


def around(t):
    before = [e for e in ev if e.time_range.end <= t + 0.5]
    after = [e for e in ev if e.time_range.start >= t - 0.5]
    b = before[-1].name[:50] if before else "-"
    a_ = min(after, key=lambda e: e.time_range.start).name[:50] if after else "-"
    return b, a_


for g, s, f in gaps[:int(os.environ.get("NGAPS", "15"))]:
    b, a_ = around(s)
    print(f"gap {g / 1e3:8.3f} ms  after [{b}]  before [{a_}]")
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25, max_name_column_width=60))
