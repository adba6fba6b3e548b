import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from golden_io import Case
import paper_2604_19004_b200.engine as E
from paper_2604_19004_b200 import EngineConfig, WorkflowOverride, spgemm
c = Case(sys.argv[1])
for save, tb in ((0.35, 1 << 30), (0.0, 1 << 30), (0.35, 0), (0.0, 0)):
    E.BITMAP_SAVE_SHARE = save
    E.BTILE_BUDGET = tb
    C, rep = spgemm(c.A, c.B, EngineConfig(workflow=WorkflowOverride.FORCE_SYMBOLIC))
    vals = C.values
    rows = np.repeat(np.arange(C.nrows), np.diff(c.d["C_ptr"]))
    if c.stride > 1:
        vals = vals[rows % c.stride == 0]
    bad = ~np.isclose(vals, c.d["C_val"], rtol=1e-12, atol=0)
    print(f"save={save} btile={tb}: bad {int(bad.sum())}")
