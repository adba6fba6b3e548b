"""Which rows take the fallback stage on a config (analysis): plan kinds,
products and exact counts of the planned-FALLBACK rows without windows.
python tools/fb_rows.py CONFIG"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2604_19004_b200 import EngineConfig, matgen, spgemm  # noqa: E402
from paper_2604_19004_b200.device import to_device  # noqa: E402
from paper_2604_19004_b200 import engine  # noqa: E402

name = sys.argv[1]
a, b = matgen.make_config(name)
dev = torch.device("cuda", 0)
A = to_device(a, dev)
B = A if b is a else to_device(b, dev)
seen = {}
orig = engine.select_fallback


def spy(ctx, m, kind, products, overflow, exclude):
    rows, n = orig(ctx, m, kind, products, overflow, exclude)
    if exclude is not None and n:
        seen["rows"] = rows.clone()
        seen["products"] = products[rows].clone()
    return rows, n


engine.select_fallback = spy
c, rep = spgemm(A, B, EngineConfig(return_device=True))
torch.cuda.synchronize()
if "rows" in seen:
    r = seen["rows"].cpu().numpy()
    p = seen["products"].cpu().numpy()
    rl = (c.row_ptr[1:] - c.row_ptr[:-1])[seen["rows"]].cpu().numpy()
    print(f"fallback rows without windows: {len(r)}, products {p.sum():.4e} "
          f"(of {rep.total_products:.4e}), nnz {rl.sum():.4e}")
    for q in (0, 10, 50, 90, 100):
        print(f"  p{q}: products {np.percentile(p, q):.0f} count {np.percentile(rl, q):.0f}")
else:
    print("no fallback rows without windows")
print(rep.overflow_row_count, rep.workflow)
