import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from golden_io import Case
from paper_2604_19004_b200 import EngineConfig, WorkflowOverride, spgemm
c = Case(sys.argv[1])
for w in WorkflowOverride:
    C, rep = spgemm(c.A, c.B, EngineConfig(workflow=w, tiers=c.tiers() or EngineConfig().tiers))
    ok_s = np.array_equal(C.row_ptr, c.d["C_ptr"]) and np.array_equal(C.col_idx, c.d["C_col"])
    vals = C.values
    if c.stride > 1:
        rows = np.repeat(np.arange(C.nrows), np.diff(c.d["C_ptr"]))
        vals = vals[rows % c.stride == 0]
    bad = ~np.isclose(vals, c.d["C_val"], rtol=1e-12, atol=0)
    print(w.value, "structure", ok_s, "bad values", int(bad.sum()), "overflow rows", rep.overflow_row_count, rep.workflow)
    if bad.any():
        rows = np.repeat(np.arange(C.nrows), np.diff(c.d["C_ptr"]))
        if c.stride > 1: rows = rows[rows % c.stride == 0]
        br = np.unique(rows[bad])
        print("  bad rows", br[:20], "n", len(br))
