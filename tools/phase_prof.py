"""Per-phase cycle split of the window kernel (profiling build):
SGB200_LIB=paper_2604_19004_b200/libsgb200_prof.so python tools/phase_prof.py rmat17"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_19004_b200 import EngineConfig, _lib, matgen, spgemm  # noqa: E402
from paper_2604_19004_b200.device import to_device  # noqa: E402

a, b = matgen.make_config(sys.argv[1])
dev = torch.device("cuda", 0)
A = to_device(a, dev)
B = A if b is a else to_device(b, dev)
lib = _lib.load()
out = (ctypes.c_ulonglong * 12)()
for rep in range(2):
    lib.sg_debug_phase_cycles(out)
    c, r = spgemm(A, B, EngineConfig(return_device=True))
    torch.cuda.synchronize()
    lib.sg_debug_phase_cycles(out)
    v = list(out)
    names = ["setup+zero", "load+search", "pass1(bitmap)", "prefix", "pass2(values)", "emit vals",
             "cols->smem", "emit cols"]
    tot = sum(v[:8])
    nwin = max(v[9], 1)
    print(f"windows {v[9]}  products(single-chunk) {v[8]}  products/window {v[8] / nwin:.0f}  "
          f"words/window {v[10] / nwin:.0f}  outputs/window {v[11] / nwin:.0f}")
    for i, nm in enumerate(names):
        print(f"  {nm:14s} {100 * v[i] / tot:5.1f}%  {v[i] / nwin:9.0f} cyc/window")
    print("  stage ms", {k: round(x, 2) for k, x in r.kernel_ms.items()})
    del c
