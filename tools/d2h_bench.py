"""Device -> host download strategies for C (the e2e path): python tools/d2h_bench.py [GB]"""
import mmap
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2604_19004_b200.device import download  # noqa: E402

for f in ("enabled", "defrag"):
    try:
        print(f, open(f"/sys/kernel/mm/transparent_hugepage/{f}").read().strip())
    except OSError as e:
        print(f, e)
print("cpus", os.cpu_count())
gb = float(sys.argv[1]) if len(sys.argv) > 1 else 16
n = int(gb * (1 << 30)) // 4
dev = torch.device("cuda", 0)
t = torch.arange(n, dtype=torch.int32, device=dev)
torch.cuda.synchronize()

# raw link bandwidth into a reused pinned buffer
pin = torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True)
src = t.view(torch.uint8)
torch.cuda.synchronize()
t0 = time.perf_counter()
for i in range(8):
    pin.copy_(src[(i % 4) << 30:((i % 4) + 1) << 30], non_blocking=True)
torch.cuda.synchronize()
print(f"raw D2H into pinned: {8 / (time.perf_counter() - t0):.1f} GB/s")

# first-touch cost of fresh pages (page faults), 1 and 8 threads
a = np.empty(n, np.int32)
t0 = time.perf_counter()
a.view(np.uint8)[::4096] = 1
print(f"first touch 4K pages, 1 thread: {gb / (time.perf_counter() - t0):.1f} GB/s")
del a


def hp_empty(nbytes):
    m = mmap.mmap(-1, nbytes, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    try:
        m.madvise(mmap.MADV_HUGEPAGE)
    except (AttributeError, OSError) as e:
        print("madvise failed", e)
    return m


m = hp_empty(n * 4)
b = np.frombuffer(m, dtype=np.uint8)
t0 = time.perf_counter()
b[::4096] = 1
print(f"first touch with MADV_HUGEPAGE, 1 thread: {gb / (time.perf_counter() - t0):.1f} GB/s")
del b
m.close()

# parallel first touch
a = np.empty(n * 4, np.uint8)
t0 = time.perf_counter()
step = (n * 4 + 15) // 16
with ThreadPoolExecutor(16) as ex:
    list(ex.map(lambda i: a[i * step:(i + 1) * step:4096].fill(1), range(16)))
print(f"first touch 4K pages, 16 threads: {gb / (time.perf_counter() - t0):.1f} GB/s")
del a

for mode, ns in (("0", 16), ("1", 8), ("1", 16)):
    os.environ["SG_DOWNLOAD_MODE"] = mode
    t0 = time.perf_counter()
    out = download(t, ns)
    print(f"download() mode {mode} {ns} native threads: {gb / (time.perf_counter() - t0):.1f} GB/s  ok={int(out[-1]) == int(t[-1])}")
    del out
