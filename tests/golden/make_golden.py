"""Generate golden fixtures by running the REAL reference (build container only).

    PYTHONPATH=. python tests/golden/make_golden.py

Imports ``sketchgemm`` (and its test generators) read-only from
``/root/reference/pkg`` and records, for a corpus of seeded inputs, the
reference's own outputs: C (per workflow override), RunReport fields, row
statistics, B sketches (p = 5/6/7), estimates, exact counts and plans.  The
fixtures are committed under ``tests/golden/`` so that the oracle restatement
(``oracle/ocean_cpu.py``) and the GPU path can be checked against the
reference on the GPU box, where ``/root/reference`` does not exist.
"""

from __future__ import annotations

import dataclasses
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg"
sys.path.insert(0, f"{REF}/src")
sys.path.insert(0, f"{REF}/tests")

import matgen as rmg  # noqa: E402  (reference test generators)
import sketchgemm as sg  # noqa: E402
from sketchgemm import accumulate as acc  # noqa: E402
from sketchgemm.analysis import WorkflowChoice, WorkflowKind  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
OVR = {"auto": sg.WorkflowOverride.AUTO, "symbolic": sg.WorkflowOverride.FORCE_SYMBOLIC,
       "estimate": sg.WorkflowOverride.FORCE_ESTIMATE, "upper": sg.WorkflowOverride.FORCE_UPPER_BOUND}
WK = {"symbolic": WorkflowKind.SYMBOLIC, "estimate": WorkflowKind.HLL_ESTIMATION,
      "upper": WorkflowKind.UPPER_BOUND}


def put_csr(d, name, m):
    d[f"{name}_shape"] = np.array([m.nrows, m.ncols], np.int64)
    d[f"{name}_ptr"] = m.row_ptr
    d[f"{name}_col"] = m.col_idx
    d[f"{name}_val"] = m.values


def report_dict(r):
    return {k: v for k, v in dataclasses.asdict(r).items() if not k.endswith("_ms")}


def record_case(name, a, b, overrides=("auto", "symbolic", "estimate", "upper"),
                tiers=None, intermediates=True, extra_cfg=None,
                value_stride=1):
    d = {}
    put_csr(d, "A", a)
    put_csr(d, "B", b)
    meta = {"name": name, "reports": {}, "tiers": None}
    if tiers is not None:
        meta["tiers"] = dataclasses.asdict(tiers)
    first = None
    for o in overrides:
        cfg = sg.EngineConfig(workflow=OVR[o], **({"tiers": tiers} if tiers else {}),
                              **(extra_cfg or {}))
        c, r = sg.spgemm(a, b, cfg)
        meta["reports"][o] = report_dict(r)
        if first is None:
            first = c
            continue
        # structure is workflow-invariant in the reference (test_acceptance.py:228-239)
        assert np.array_equal(c.row_ptr, first.row_ptr) and np.array_equal(c.col_idx, first.col_idx)
        np.testing.assert_allclose(c.values, first.values, rtol=1e-12, atol=0)
    put_csr(d, "C", first)
    if value_stride > 1:
        # large products: keep the structure whole, values for every k-th row only
        rows = np.repeat(np.arange(first.nrows), np.diff(first.row_ptr))
        d["C_val"] = first.values[rows % value_stride == 0]
    d["value_stride"] = np.array(value_stride, np.int64)
    if intermediates:
        st = sg.compute_row_stats(a, b)
        d["products"] = st.products
        d["span_lo"] = st.span_lo
        d["span_hi"] = st.span_hi
        d["exact"] = sg.symbolic_pass(a, b, st).per_row
        for p in (5, 6, 7):
            sk = sg.build_b_sketches(b, p)
            d[f"regs_p{p}"] = sk.registers
            d[f"est_p{p}"] = sg.estimate_pass(a, sk).per_row
        t = tiers or sg.TierConfig()
        for wf in ("symbolic", "estimate", "upper"):
            if wf == "symbolic":
                pred = sg.symbolic_pass(a, b, st)
            elif wf == "estimate":
                pred = sg.estimate_pass(a, sg.build_b_sketches(b, 6))
            else:
                pred = sg.upper_bound_pass(st)
            pl = acc.plan_rows(pred, st, WorkflowChoice(WK[wf], 64), t)
            d[f"plan_{wf}_kind"] = pl.kind
            d[f"plan_{wf}_cap"] = pl.capacity
            d[f"plan_{wf}_alloc"] = pl.alloc
        rows = np.arange(a.nrows, dtype=np.int64)
        sampled = sg.sample_cr(a, sg.build_b_sketches(b, 6), st, seed=0)
        meta["sample_cr_p6_seed0"] = [sampled.cr_hat, sampled.mean_row_cr, sampled.std_row_cr,
                                      sampled.n_sampled]
        del rows
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **d)
    with open(os.path.join(HERE, f"{name}.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
    print(name, a.nrows, b.ncols, "nnzC", int(d["C_ptr"][-1]))


def kats():
    out = {"hash64": {}, "ranks": {}, "estimates": {}}
    for k in [0, 1, 2, 12345, 2 ** 31 - 1, 2 ** 32 - 1, 999, 65535]:
        out["hash64"][str(k)] = hex(sg.hash64(k))
    from sketchgemm.hll import hash_ranks
    for p in (5, 6, 7):
        idx, rank = hash_ranks(np.arange(0, 4096, dtype=np.uint64), p)
        out["ranks"][str(p)] = {"idx_sum": int(idx.sum()), "rank_sum": int(rank.sum()),
                                "first16": [[int(i), int(r)] for i, r in zip(idx[:16], rank[:16])]}
    out["estimates"]["p6_0_999"] = sg.HllSketch.from_keys(np.arange(1000), 6).estimate()
    out["estimates"]["p5_0_9"] = sg.HllSketch.from_keys(np.arange(10), 5).estimate()
    out["estimates"]["p7_0_4999"] = sg.HllSketch.from_keys(np.arange(5000), 7).estimate()
    out["cr_variance_bound_1_64_6000"] = sg.cr_variance_bound(1.0, 64, 6000)
    with open(os.path.join(HERE, "kats.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)


def build_cases():
    """csr.from_triplets / csr.transpose goldens (tests/golden/csr_build/): seeded
    triplets with duplicates, arbitrary order, empty rows and empty input."""
    out = os.path.join(HERE, "csr_build")
    os.makedirs(out, exist_ok=True)
    specs = [(0, 1, 1, 0), (1, 7, 5, 40), (2, 300, 200, 5000), (3, 2000, 70_000, 60_000),
             (4, 50_000, 3, 200_000), (5, 1, 100_000, 30_000)]
    for seed, nr, nc, n in specs:
        rng = np.random.default_rng(1000 + seed)
        # skewed rows and a small column pool so duplicates are common
        rows = np.minimum((rng.pareto(1.2, n) * nr / 20).astype(np.int64), nr - 1) if n else np.empty(0, np.int64)
        cols = rng.integers(0, max(1, min(nc, 4 * max(1, n // max(1, nr)) + 3)), n) * (nc // max(1, min(nc, 4 * max(1, n // max(1, nr)) + 3)))
        cols = np.minimum(cols, nc - 1).astype(np.int64)
        vals = rng.uniform(-1.0, 1.0, n)
        c = sg.from_triplets(nr, nc, rows, cols, vals)
        t = sg.transpose(c)
        np.savez_compressed(os.path.join(out, f"triplets{seed}.npz"), shape=np.array([nr, nc], np.int64),
                            rows=rows, cols=cols, vals=vals, ptr=c.row_ptr, col=c.col_idx, val=c.values,
                            t_ptr=t.row_ptr, t_col=t.col_idx, t_val=t.values)
        print("triplets", seed, nr, nc, n, "-> nnz", int(c.row_ptr[-1]))


def est_eval_cases():
    """cmd_est_eval's per-register records (cli.py:301-341) for golden inputs:
    FORCE_ESTIMATE with compute_estimation_errors at m = 32 / 64 / 128."""
    out = {}
    for name in ["corpus0", "corpus1", "corpus2", "corpus3", "pair03", "pair07", "pair11", "bitmapq"]:
        d = dict(np.load(os.path.join(HERE, name + ".npz")))
        mk = lambda k: sg.CsrMatrix(int(d[k + "_shape"][0]), int(d[k + "_shape"][1]), d[k + "_ptr"],  # noqa: E731
                                    d[k + "_col"], d[k + "_val"])
        a, b = mk("A"), mk("B")
        for m in (32, 64, 128):
            cfg = sg.EngineConfig(workflow=sg.WorkflowOverride.FORCE_ESTIMATE, registers=m,
                                  compute_estimation_errors=True)
            _, r = sg.spgemm(a, b, cfg)
            out[f"{name}/{m}"] = {k: getattr(r, k) for k in ("est_mean_rel_err", "est_std_rel_err",
                                                             "overflow_row_count", "cr_hat", "cr_true", "nnz_c")}
    with open(os.path.join(HERE, "est_eval.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)
    print("est_eval", len(out))


def main():
    if sys.argv[1:] == ["build"]:
        build_cases()
        return
    if sys.argv[1:] == ["est_eval"]:
        est_eval_cases()
        return
    kats()
    build_cases()
    est_eval_cases()
    # mixed corpus (reference test_acceptance criterion 1 / test_engine)
    for i in range(24):
        a, b = rmg.pair_for_case(100 + i, i)
        record_case(f"pair{i:02d}", a, b)
    # Fig. 2 row (test_engine.py:31-36)
    a = sg.from_triplets(1, 2, [0, 0], [0, 1], [1.0, 1.0])
    b = sg.from_triplets(2, 10, [0, 0, 1, 1], [2, 4, 2, 9], [3.0, 5.0, 7.0, 11.0])
    record_case("fig2", a, b)
    # empty operands (test_engine.py:50-55)
    record_case("empty", sg.from_triplets(5, 3, [], [], []), sg.from_triplets(3, 4, [], [], []))
    # estimation corpus (ER >= 8; estimate workflow chosen by AUTO for some)
    for s in range(4):
        a, b = rmg.corpus_matrix(s)
        record_case(f"corpus{s}", a, b, value_stride=16)
    # forced overflow with tiny tiers (test_engine.py:280-292)
    rng = np.random.default_rng(5)
    a = rmg.random_csr(rng, 120, 60, 0.25)
    b = rmg.random_csr(rng, 60, 900, 0.25)
    tiny = sg.TierConfig(hash_capacities=(16, 32), enhanced_hash_capacity=96,
                         dense_spans=(8, 16), esc_max_products=4)
    record_case("tiny_tiers", a, b, tiers=tiny, value_stride=4)
    # enhanced-hash tier on wide rows (test_engine.py:245-268)
    rng = np.random.default_rng(6)
    ncols = 40_000
    b = sg.from_triplets(200, ncols, np.repeat(np.arange(200), 40),
                         np.concatenate([rng.choice(ncols, 40, replace=False) for _ in range(200)]),
                         np.ones(200 * 40))
    a = sg.from_triplets(40, 200, np.repeat(np.arange(40), 150),
                         np.concatenate([rng.choice(200, 150, replace=False) for _ in range(40)]),
                         np.ones(40 * 150))
    record_case("enhanced", a, b, value_stride=4)
    # bitmap-query case (test_engine.py:121-139)
    rng = np.random.default_rng(3)
    shared = np.sort(rng.choice(400, 120, replace=False))
    b = sg.from_triplets(40, 400, np.repeat(np.arange(40), 120), np.tile(shared, 40), np.ones(40 * 120))
    a = sg.from_triplets(300, 40, np.repeat(np.arange(300), 10),
                         np.concatenate([rng.choice(40, 10, replace=False) for _ in range(300)]),
                         np.ones(3000))
    record_case("bitmapq", a, b)
    # BASELINE config 1 (ER 10k, ~8/row), all overrides; generator from the repo
    sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
    from paper_2604_19004_b200 import matgen as mg
    a = mg.erdos_renyi()
    a = sg.CsrMatrix(a.nrows, a.ncols, a.row_ptr, a.col_idx, a.values)
    record_case("cfg1_er10k", a, a, intermediates=False, value_stride=4)


if __name__ == "__main__":
    main()
