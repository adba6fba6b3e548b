"""Pin the CPU oracle restatement to the reference's own outputs (CPU only).

Fixtures: tests/golden/*.npz, produced by the real reference
(tests/golden/make_golden.py).  Every stage is compared: row stats and exact
counts (integer-exact), sketches (register-exact), estimates (bit-exact: same
numpy ops), plans (exact), reports, and C (structure exact, values rtol 1e-12).
"""
import json
import os

import numpy as np
import pytest

from golden_io import GOLDEN, Case, names
from oracle import ocean_cpu as oc

CASES = [n for n in names()]
OVR = ("auto", "symbolic", "estimate", "upper")


def test_kats_hash_rank_estimate():
    with open(os.path.join(GOLDEN, "kats.json")) as fh:
        k = json.load(fh)
    for key, h in k["hash64"].items():
        assert int(oc.hash64(np.uint64(int(key)))) == int(h, 16)
    for p, r in k["ranks"].items():
        idx, rank = oc.register_index_rank(np.arange(4096, dtype=np.uint64), int(p))
        assert int(idx.sum()) == r["idx_sum"] and int(rank.sum()) == r["rank_sum"]
        assert [[int(i), int(j)] for i, j in zip(idx[:16], rank[:16])] == r["first16"]

    def est(keys, p):
        regs = np.zeros(1 << p, np.uint8)
        idx, rank = oc.register_index_rank(keys, p)
        np.maximum.at(regs, idx, rank)
        return float(oc.hll_estimate(regs[None])[0])

    assert est(np.arange(1000), 6) == k["estimates"]["p6_0_999"]
    assert est(np.arange(10), 5) == k["estimates"]["p5_0_9"]
    assert est(np.arange(5000), 7) == k["estimates"]["p7_0_4999"]
    # published KATs quoted in SURVEY §8(c)
    assert int(oc.hash64(np.uint64(0))) == 0xE220A8397B1DCDAF
    assert est(np.arange(1000), 6) == pytest.approx(1102.1074904104512, rel=0, abs=0)


def test_rank_edge_bits():
    # bit_length at exact powers of two and all-ones words
    w = [0, 1, 2, 3, (1 << 31), (1 << 32) - 1, (1 << 32), (1 << 57) - 1]
    for p in (5, 6, 7):
        for x in w:
            x &= (1 << (64 - p)) - 1
            # find a key whose hash >> p == x is impossible; test the helper directly
            hi, lo = x >> 32, x & 0xFFFFFFFF
            bl = x.bit_length()
            got = (np.frexp(float(hi))[1] + 32) if hi else np.frexp(float(lo))[1]
            assert got == bl


@pytest.mark.parametrize("name", [n for n in CASES])
def test_oracle_stages_match_reference(name):
    c = Case(name)
    if not c.has_intermediates:
        pytest.skip("no intermediates recorded")
    a, b = oc.as_csr(c.A), oc.as_csr(c.B)
    st = oc.row_stats(a, b)
    np.testing.assert_array_equal(st.products, c.d["products"])
    np.testing.assert_array_equal(st.span_lo, c.d["span_lo"])
    np.testing.assert_array_equal(st.span_hi, c.d["span_hi"])
    np.testing.assert_array_equal(oc.exact_counts(a, b, st), c.d["exact"])
    for p in (5, 6, 7):
        regs = oc.b_sketches(b, p)
        np.testing.assert_array_equal(regs, c.d[f"regs_p{p}"])
        np.testing.assert_array_equal(oc.estimate_all(a, regs), c.d[f"est_p{p}"])
    t = oc.Tiers.of(c.tiers())
    regs6 = oc.b_sketches(b, 6)
    for wf in ("symbolic", "estimate", "upper"):
        if wf == "symbolic":
            pred, pk = oc.exact_counts(a, b, st), "exact"
        elif wf == "estimate":
            pred, pk = oc.estimate_all(a, regs6), "estimated"
        else:
            pred, pk = st.products.copy(), "upper_bound"
        kind, cap, alloc = oc.plan(pred, pk, wf, st, t)
        np.testing.assert_array_equal(kind, c.d[f"plan_{wf}_kind"])
        np.testing.assert_array_equal(cap, c.d[f"plan_{wf}_cap"])
        np.testing.assert_array_equal(alloc, c.d[f"plan_{wf}_alloc"])
    rows = oc.sample_rows(a.nrows, oc.SAMPLE_RATIO, oc.SAMPLE_MIN, oc.SAMPLE_MAX, 0)
    if a.nrows:
        cr = oc.cr_from_sample(st.products[rows], oc.merged_estimates(a, regs6, rows))
        assert list(cr) + [len(rows)] == c.meta["sample_cr_p6_seed0"]


@pytest.mark.parametrize("name", CASES)
def test_oracle_spgemm_matches_reference(name):
    c = Case(name)
    for o in OVR:
        C, rep = oc.spgemm(c.A, c.B, workflow=o, tiers=c.tiers())
        c.check_product(C)
        want = c.meta["reports"][o]
        for key, v in rep.items():
            if key.endswith("_ms"):
                continue
            if isinstance(v, float) and want[key] is not None:
                assert v == pytest.approx(want[key], rel=1e-12), (o, key)
            else:
                assert v == want[key], (o, key)


def test_dict_oracle_agrees_on_small_cases():
    for name in ("pair00", "pair01", "pair05", "fig2", "empty"):
        c = Case(name)
        c.check_product(oc.dict_spgemm(c.A, c.B))


def test_oracle_worker_count_invariance():
    c = Case("corpus1")
    C1, _ = oc.spgemm(c.A, c.B, workers=1)
    C4, _ = oc.spgemm(c.A, c.B, workers=4)
    np.testing.assert_array_equal(C1.col_idx, C4.col_idx)
    assert (C1.values == C4.values).all()
