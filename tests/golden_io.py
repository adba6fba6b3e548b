"""Loader for the committed golden fixtures (tests/golden/*.npz + *.json).

The fixtures were produced by the real reference (tests/golden/make_golden.py).
"""
import glob
import json
import os

import numpy as np

from paper_2604_19004_b200.csr import CsrMatrix

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def names():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "*.npz")))


class Case:
    def __init__(self, name):
        self.name = name
        self.d = dict(np.load(os.path.join(GOLDEN, name + ".npz")))
        with open(os.path.join(GOLDEN, name + ".json")) as fh:
            self.meta = json.load(fh)
        self.A = self._csr("A")
        self.B = self._csr("B")
        self.stride = int(self.d["value_stride"])

    def _csr(self, k):
        d = self.d
        r, c = d[k + "_shape"]
        return CsrMatrix(int(r), int(c), d[k + "_ptr"], d[k + "_col"], d[k + "_val"])

    @property
    def has_intermediates(self):
        return "products" in self.d

    def tiers(self):
        t = self.meta.get("tiers")
        if t is None:
            return None
        from paper_2604_19004_b200.config import TierConfig
        return TierConfig(hash_capacities=tuple(t["hash_capacities"]),
                          enhanced_hash_capacity=t["enhanced_hash_capacity"],
                          dense_spans=tuple(t["dense_spans"]),
                          esc_max_products=t["esc_max_products"],
                          expansion_coef=t["expansion_coef"],
                          bitmap_query_threshold=t["bitmap_query_threshold"])

    def check_product(self, c, rtol=1e-12):
        """Structure bit-exact, values within rtol (atol 0) of the reference C
        (the comparator of pkg/tests/matgen.py:151-156)."""
        d = self.d
        assert (c.nrows, c.ncols) == tuple(int(x) for x in d["C_shape"])
        np.testing.assert_array_equal(np.asarray(c.row_ptr), d["C_ptr"])
        np.testing.assert_array_equal(np.asarray(c.col_idx), d["C_col"])
        vals = np.asarray(c.values)
        if self.stride > 1:
            rows = np.repeat(np.arange(c.nrows), np.diff(d["C_ptr"]))
            vals = vals[rows % self.stride == 0]
        np.testing.assert_allclose(vals, d["C_val"], rtol=rtol, atol=0)
