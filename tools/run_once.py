"""Run one spgemm on a config (for ncu captures): python tools/run_once.py CONFIG [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_19004_b200 import EngineConfig, matgen, spgemm  # noqa: E402
from paper_2604_19004_b200.device import to_device  # noqa: E402

name = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
a, b = matgen.make_config(name)
dev = torch.device("cuda", 0)
A = to_device(a, dev)
B = A if b is a else to_device(b, dev)
for _ in range(reps):
    c, rep = spgemm(A, B, EngineConfig(return_device=True))
    torch.cuda.synchronize()
    print(rep.workflow, rep.nnz_c, {k: round(v, 3) for k, v in rep.kernel_ms.items()}, flush=True)
    del c
