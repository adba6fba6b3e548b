import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
from golden_io import Case
from paper_2604_19004_b200 import _lib
from paper_2604_19004_b200.device import to_device, ptr
from paper_2604_19004_b200.engine import _Ctx, Windows, btile
c = Case(sys.argv[1])
dev = torch.device("cuda", 0)
ctx = _Ctx(dev, torch.cuda.current_stream(dev))
B = to_device(c.B, dev)
w = Windows(None, None, None, None, None, None, 0)
btile(ctx, B, w)
off = w.btile_off.cpu().numpy(); tbl = w.btile.cpu().numpy()
ntiles = (B.ncols + 4095) // 4096
bad = 0
for k in range(B.nrows):
    if off[k] < 0: continue
    s, e = c.B.row_ptr[k], c.B.row_ptr[k + 1]
    cols = c.B.col_idx[s:e]
    want = np.searchsorted(cols, np.arange(ntiles + 1) * 4096, side="left")
    got = tbl[off[k]: off[k] + ntiles + 1]
    if not np.array_equal(want, got):
        bad += 1
        if bad < 4: print("row", k, "len", e - s, "want", want, "got", got)
print("rows with tables", int((off >= 0).sum()), "bad", bad)
