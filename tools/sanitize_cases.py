"""Small parity cases for compute-sanitizer (tools/sanitize.sh): golden cases
under every workflow override, five stress shapes (hub-row windows, sparse
wide spans, columns >= 2^23, heavy merging, empty rows), the no-saved-bitmap
window path and the staged short rows -- each result checked against the
oracle / reference fixture so a sanitizer run is also a parity run."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

from golden_io import Case  # noqa: E402
from oracle import ocean_cpu as oc  # noqa: E402
from paper_2604_19004_b200 import EngineConfig, WorkflowOverride, engine, matgen, spgemm  # noqa: E402

OVR = [WorkflowOverride.AUTO, WorkflowOverride.FORCE_SYMBOLIC, WorkflowOverride.FORCE_ESTIMATE,
       WorkflowOverride.FORCE_UPPER_BOUND]


def check(c, ref):
    np.testing.assert_array_equal(c.row_ptr, ref.row_ptr)
    np.testing.assert_array_equal(c.col_idx, ref.col_idx)
    np.testing.assert_allclose(c.values, ref.values, rtol=1e-12, atol=0)


def main():
    n = 0
    # SANITIZE_ONLY=stress: only the stress shapes (the window kernels)
    only = os.environ.get("SANITIZE_ONLY")
    for name in (() if only == "stress" else ("fig2", "pair00", "pair05", "corpus1", "enhanced", "tiny_tiers",
                                              "bitmapq")):
        cs = Case(name)
        for o in OVR:
            c, _ = spgemm(cs.A, cs.B, EngineConfig(workflow=o, tiers=cs.tiers() or EngineConfig().tiers))
            cs.check_product(c)
            n += 1
    from test_gpu_stress import _case
    for seed in (0, 1, 2, 3, 4):
        a, b = _case(seed)
        ref, _ = oc.spgemm(a, b)
        for o in (WorkflowOverride.AUTO, WorkflowOverride.FORCE_ESTIMATE):
            c, _ = spgemm(a, b, EngineConfig(workflow=o))
            check(c, ref)
            n += 1
    if only == "stress":
        print(f"sanitize cases ok: {n} multiplies checked")
        return
    a = matgen.rmat(11, seed=5)
    ref, _ = oc.spgemm(a, a)
    engine.BITMAP_SAVE_SHARE = 0.0  # window pass rebuilding keys itself
    c, _ = spgemm(a, a)
    check(c, ref)
    engine.BITMAP_SAVE_SHARE = 0.35
    n += 1
    print(f"sanitize cases ok: {n} multiplies checked")


if __name__ == "__main__":
    main()
