"""Producer / consumer phase split of k_win (profiling build):
SGB200_LIB=paper_2604_19004_b200/libsgb200_prof.so python tools/kw_prof.py rmat20"""
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
out = (ctypes.c_ulonglong * 16)()
for rep in range(2):
    lib.sg_debug_kw_cycles(out)
    c, r = spgemm(A, B, EngineConfig(return_device=True))
    torch.cuda.synchronize()
    lib.sg_debug_kw_cycles(out)
    v = list(out)
    ctas = 148
    kms = r.kernel_ms
    print("stage ms", {k: round(x, 2) for k, x in kms.items()})
    wins = max(v[5], 1)
    print(f"windows {wins}, chunks seen by consumers (per warp avg) {v[13] / (ctas * 24):.0f}")
    pn = ["win_free wait", "empty wait", "append", "publish", "clip(next)"]
    for i, nm in enumerate(pn):
        print(f"  producer {nm:14s} {v[i] / ctas / 1.965e6:8.2f} ms/CTA  {v[i] / wins:8.0f} cyc/window")
    cn = ["full wait", "bm_full wait", "groups", "columns", "store(last)"]
    for i, nm in enumerate(cn):
        print(f"  consumer {nm:14s} {v[8 + i] / (ctas * 24) / 1.965e6:8.2f} ms/warp")
    del c
