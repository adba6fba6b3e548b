"""Throughput of the device CSR construction (from_triplets / transpose) on
R-MAT-20 (16.1M entries) vs the host numpy paths (reference csr.py:52-97):
python tools/bench_build.py [scale]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import ocean_cpu as oc  # noqa: E402  (host baseline only)
from paper_2604_19004_b200 import matgen  # noqa: E402
from paper_2604_19004_b200.build import from_triplets_device, transpose_device  # noqa: E402
from paper_2604_19004_b200.device import to_device  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 20
a = matgen.rmat(scale)
dev = torch.device("cuda", 0)
rows = np.repeat(np.arange(a.nrows), np.diff(a.row_ptr))
perm = np.random.default_rng(0).permutation(a.nnz)
r_d = torch.from_numpy(rows[perm]).to(dev)
c_d = torch.from_numpy(a.col_idx[perm].astype(np.int64)).to(dev)
v_d = torch.from_numpy(a.values[perm]).to(dev)
A = to_device(a, dev)


def timeit(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


t_coo = timeit(lambda: from_triplets_device(a.nrows, a.ncols, r_d, c_d, v_d, device=dev))
t_tr = timeit(lambda: transpose_device(A))
t0 = time.perf_counter()
oc.triplets_to_csr(a.nrows, a.ncols, rows[perm], a.col_idx[perm], a.values[perm])
h_coo = (time.perf_counter() - t0) * 1e3
t0 = time.perf_counter()
oc.transpose(a)
h_tr = (time.perf_counter() - t0) * 1e3
n = a.nnz
# compulsory bytes: triplets in (8+8+8) + CSR out (4+8 per entry, 8 per row)
b_coo = 24 * n + 12 * n + 8 * (a.nrows + 1)
b_tr = 2 * (12 * n + 8 * (a.nrows + 1))
print(f"R-MAT-{scale}: nnz {n}")
print(f"from_triplets: device {t_coo:.3f} ms ({b_coo / t_coo / 1e6:.0f} GB/s compulsory), "
      f"host numpy {h_coo:.0f} ms -> {h_coo / t_coo:.0f}x")
print(f"transpose:     device {t_tr:.3f} ms ({b_tr / t_tr / 1e6:.0f} GB/s compulsory), "
      f"host numpy {h_tr:.0f} ms -> {h_tr / t_tr:.0f}x")
