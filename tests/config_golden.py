"""Loader / comparator for the config-scale fixtures (tests/golden/configs),
made by the real reference with tests/golden/make_config_golden.py."""
import hashlib
import json
import os

import numpy as np

CFG = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "configs")


def load(name):
    with open(os.path.join(CFG, name + ".json")) as fh:
        meta = json.load(fh)
    arrays = dict(np.load(os.path.join(CFG, name + ".npz")))
    return meta, arrays


def available(name) -> bool:
    return os.path.exists(os.path.join(CFG, name + ".json"))


def _sha(x) -> str:
    return hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest()


def check(c, meta, arrays, prefix="", rtol=1e-12):
    """C (host CSR, or a block of rows of C) against one fixture: structure
    by sha256 (bit-exact), values by group sums and sampled rows (rtol, atol 0;
    all values positive, so a group sum inherits the per-entry tolerance).
    Returns the largest relative value error seen."""
    rp = np.asarray(c.row_ptr, dtype=np.int64)
    ci = np.asarray(c.col_idx, dtype=np.int32)
    vv = np.asarray(c.values, dtype=np.float64)
    assert int(rp[-1]) == meta["nnz"], (prefix, int(rp[-1]), meta["nnz"])
    assert _sha(rp) == meta["sha_row_ptr"], f"{prefix}: row_ptr differs from the reference"
    assert _sha(ci) == meta["sha_col_idx"], f"{prefix}: col_idx differs from the reference"
    g = meta["group"]
    gs = np.add.reduceat(vv, np.arange(0, len(vv), g)) if len(vv) else np.zeros(0)
    want = arrays[prefix + "group_sums"]
    np.testing.assert_allclose(gs, want, rtol=rtol, atol=0, err_msg=prefix + " group sums")
    worst = float(np.max(np.abs(gs - want) / np.abs(want))) if len(want) else 0.0
    rows, lens = arrays[prefix + "sample_rows"], arrays[prefix + "sample_lens"]
    cols, vals = arrays[prefix + "sample_cols"], arrays[prefix + "sample_vals"]
    o = 0
    for r, n in zip(rows, lens):
        s = int(rp[r])
        np.testing.assert_array_equal(ci[s:s + n], cols[o:o + n], err_msg=f"{prefix} row {r}")
        np.testing.assert_allclose(vv[s:s + n], vals[o:o + n], rtol=rtol, atol=0, err_msg=f"{prefix} row {r}")
        if n:
            worst = max(worst, float(np.max(np.abs(vv[s:s + n] - vals[o:o + n]) / np.abs(vals[o:o + n]))))
        o += n
    return worst


def compare_exact(c, ref, rtol=1e-12):
    """The reference comparator (pkg/tests/matgen.py:151-156): structure
    array_equal, values allclose(rtol, atol=0).  Returns max relative error."""
    np.testing.assert_array_equal(np.asarray(c.row_ptr), np.asarray(ref.row_ptr))
    np.testing.assert_array_equal(np.asarray(c.col_idx), np.asarray(ref.col_idx))
    a, b = np.asarray(c.values, dtype=np.float64), np.asarray(ref.values, dtype=np.float64)
    np.testing.assert_allclose(a, b, rtol=rtol, atol=0)
    return float(np.max(np.abs(a - b) / np.abs(b))) if len(b) else 0.0
