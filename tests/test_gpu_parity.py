"""GPU parity: the sm_100a path (through the C ABI) against the reference.

Every golden case was produced by the real reference (tests/golden); structure
must be bit-exact, values within rtol 1e-12 (fp64, atol 0; matgen.py:151-156),
report fields equal.  Stage kernels are checked one by one against the
reference's intermediates (row stats, sketches, estimates, exact counts,
plans: all exact).
"""
import time

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from golden_io import Case, names  # noqa: E402

pytestmark = pytest.mark.gpu

OVR = ("auto", "symbolic", "estimate", "upper")
REPORT_EXACT = ("workflow", "registers", "overflow_row_count", "nnz_c", "total_products", "bitmap_query")
REPORT_FLOAT = ("er", "cr_hat", "cr_true")


def _cfg(o, tiers=None, **kw):
    from paper_2604_19004_b200 import EngineConfig, WorkflowOverride
    ov = {"auto": WorkflowOverride.AUTO, "symbolic": WorkflowOverride.FORCE_SYMBOLIC,
          "estimate": WorkflowOverride.FORCE_ESTIMATE, "upper": WorkflowOverride.FORCE_UPPER_BOUND}[o]
    if tiers is not None:
        kw["tiers"] = tiers
    return EngineConfig(workflow=ov, **kw)


@pytest.fixture(scope="module")
def gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2604_19004_b200 import _lib
    _lib.load()
    return torch.device("cuda", 0)


@pytest.mark.parametrize("name", names())
def test_spgemm_matches_reference(gpu, name):
    from paper_2604_19004_b200 import spgemm
    c = Case(name)
    for o in OVR:
        C, rep = spgemm(c.A, c.B, _cfg(o, c.tiers()))
        c.check_product(C)
        want = c.meta["reports"][o]
        for k in REPORT_EXACT:
            assert getattr(rep, k) == want[k], (name, o, k, getattr(rep, k), want[k])
        for k in REPORT_FLOAT:
            got, exp = getattr(rep, k), want[k]
            if exp is None:
                assert got is None, (name, o, k)
            else:
                assert got == pytest.approx(exp, rel=1e-12), (name, o, k)


@pytest.mark.parametrize("name", [n for n in names() if n.startswith(("pair", "corpus", "enh", "tiny", "bitmap"))])
def test_stage_kernels_match_reference(gpu, name):
    import paper_2604_19004_b200._lib as L
    from paper_2604_19004_b200 import TierConfig
    from paper_2604_19004_b200.device import ptr, to_device
    from paper_2604_19004_b200.engine import _Ctx, hll_build, hll_estimate, row_stats, tiers_struct
    c = Case(name)
    ctx = _Ctx(gpu, torch.cuda.current_stream(gpu))
    A = to_device(c.A, gpu)
    B = to_device(c.B, gpu)
    products, lo, hi, totals = row_stats(ctx, A, B)
    np.testing.assert_array_equal(products.cpu().numpy(), c.d["products"])
    np.testing.assert_array_equal(lo.cpu().numpy(), c.d["span_lo"])
    np.testing.assert_array_equal(hi.cpu().numpy(), c.d["span_hi"])
    assert int(totals[0]) == int(c.d["products"].sum())
    for p in (5, 6, 7):
        regs = hll_build(ctx, B, p)
        np.testing.assert_array_equal(regs.cpu().numpy().reshape(B.nrows, 1 << p), c.d[f"regs_p{p}"])
        est = hll_estimate(ctx, A, regs, p).cpu().numpy()
        np.testing.assert_array_equal(est, c.d[f"est_p{p}"])  # bit-exact
    m = A.nrows
    ws, wsb = ctx.workspace(m)
    exact = torch.empty(m, dtype=torch.int64, device=gpu)
    L.call("sg_symbolic", m, B.ncols, ptr(A.row_ptr), ptr(A.col_idx), ptr(B.row_ptr), ptr(B.col_idx),
           ptr(products), ptr(lo), ptr(hi), ptr(exact), None, 1.0, 0, ws, wsb, ctx.sp)
    np.testing.assert_array_equal(exact.cpu().numpy(), c.d["exact"])
    t = c.tiers() or TierConfig()
    est6 = hll_estimate(ctx, A, hll_build(ctx, B, 6), 6)
    for wf, pred, code in (("symbolic", exact, 0), ("estimate", est6, 1), ("upper", products, 2)):
        kind = torch.empty(m, dtype=torch.int8, device=gpu)
        cap = torch.empty(m, dtype=torch.int64, device=gpu)
        alloc = torch.empty(m, dtype=torch.int64, device=gpu)
        L.call("sg_plan", m, code, ptr(pred), ptr(products), ptr(lo), ptr(hi), tiers_struct(t),
               ptr(kind), ptr(cap), ptr(alloc), ctx.sp)
        np.testing.assert_array_equal(kind.cpu().numpy(), c.d[f"plan_{wf}_kind"], err_msg=wf)
        np.testing.assert_array_equal(cap.cpu().numpy(), c.d[f"plan_{wf}_cap"], err_msg=wf)
        np.testing.assert_array_equal(alloc.cpu().numpy(), c.d[f"plan_{wf}_alloc"], err_msg=wf)


def test_scan_kernel(gpu):
    from paper_2604_19004_b200.engine import _Ctx, scan
    ctx = _Ctx(gpu, torch.cuda.current_stream(gpu))
    rng = np.random.default_rng(0)
    for n in (0, 1, 5, 4095, 4096, 4097, 1_000_003):
        x = rng.integers(0, 1 << 40, n)
        out = scan(ctx, torch.from_numpy(x).to(gpu)).cpu().numpy()
        np.testing.assert_array_equal(out, np.r_[0, np.cumsum(x)])


def test_identity_and_errors(gpu):
    from paper_2604_19004_b200 import (DeadlineExceeded, EngineConfig, ResourceLimitError, WorkflowOverride,
                                       identity, spgemm, validate)
    from oracle import ocean_cpu as oc
    rng = np.random.default_rng(0)
    rows = rng.integers(0, 25, 150)
    cols = rng.integers(0, 40, 150)
    b = oc.triplets_to_csr(25, 40, rows, cols, rng.uniform(0.5, 1.5, 150))
    for o in OVR:
        C, _ = spgemm(identity(25), b, _cfg(o))
        np.testing.assert_array_equal(C.row_ptr, b.row_ptr)
        np.testing.assert_array_equal(C.col_idx, b.col_idx)
        np.testing.assert_array_equal(C.values, b.values)
        assert validate(C) == []
    with pytest.raises(ValueError, match="dimension"):
        spgemm(identity(3), identity(4))
    c = Case("pair00")
    with pytest.raises(ResourceLimitError, match="symbolic"):
        spgemm(c.A, c.B, EngineConfig(workflow=WorkflowOverride.FORCE_ESTIMATE, staging_limit_bytes=16))
    with pytest.raises(DeadlineExceeded):
        spgemm(c.A, c.B, EngineConfig(), deadline=time.perf_counter() - 1.0)


def _random_pair(seed):
    """Mixed generator in the spirit of pkg/tests/matgen.py:66-95 (restated)."""
    from oracle import ocean_cpu as oc
    rng = np.random.default_rng(seed)
    kind = seed % 4
    if kind == 0:
        n, k, m = rng.integers(50, 3000, 3)
        da, db = rng.uniform(0.001, 0.03, 2)
    elif kind == 1:
        n, k, m = 2000, 500, 40_000
        da, db = 0.02, 0.004
    elif kind == 2:
        n, k, m = rng.integers(100, 1500, 3)
        da, db = rng.uniform(0.01, 0.1, 2)
    else:
        n, k, m = 300, 20_000, 300_000
        da, db = 0.002, 0.0005

    def mk(r, c, d):
        nnz = int(round(r * c * d))
        lens = np.minimum((rng.pareto(1.4, r) + 0.2) * (nnz / r), c).astype(int)
        rows = np.repeat(np.arange(r), lens)
        cols = rng.integers(0, c, len(rows))
        return oc.triplets_to_csr(r, c, rows, cols, rng.uniform(0.5, 1.5, len(rows)))
    return mk(int(n), int(k), da), mk(int(k), int(m), db)


@pytest.mark.parametrize("seed", range(12))
def test_random_skewed_pairs_vs_oracle(gpu, seed):
    from paper_2604_19004_b200 import spgemm
    from oracle import ocean_cpu as oc
    a, b = _random_pair(seed)
    ref, rrep = oc.spgemm(a, b)
    for o in OVR:
        C, rep = spgemm(a, b, _cfg(o))
        np.testing.assert_array_equal(C.row_ptr, ref.row_ptr)
        np.testing.assert_array_equal(C.col_idx, ref.col_idx)
        np.testing.assert_allclose(C.values, ref.values, rtol=1e-12, atol=0)
    _, rep = spgemm(a, b, _cfg("auto"))
    assert rep.workflow == rrep["workflow"]
    assert rep.overflow_row_count == rrep["overflow_row_count"]


def test_tiny_tiers_overflow_rerun(gpu):
    """Forced overflow with tiny tiers reruns through the fallback exactly
    (pkg/tests/test_engine.py:280-292)."""
    from paper_2604_19004_b200 import spgemm
    c = Case("tiny_tiers")
    C, rep = spgemm(c.A, c.B, _cfg("estimate", c.tiers()))
    assert rep.overflow_row_count > 0
    assert rep.overflow_row_count == c.meta["reports"]["estimate"]["overflow_row_count"]
    c.check_product(C)


def test_fp32_within_1e5(gpu):
    from paper_2604_19004_b200 import EngineConfig, spgemm
    c = Case("corpus0")
    for o in OVR:
        C, _ = spgemm(c.A, c.B, _cfg(o, dtype="f32"))
        assert C.values.dtype == np.float32
        c.check_product(C.astype(np.float64), rtol=1e-5)
    del EngineConfig


def test_config_scale_poisson_and_rmat_vs_oracle(gpu):
    """Small instances of configs 2 and 3 through every workflow vs the oracle."""
    from paper_2604_19004_b200 import matgen, spgemm
    from oracle import ocean_cpu as oc
    for a in (matgen.poisson27(16), matgen.rmat(12)):
        ref, _ = oc.spgemm(a, a)
        for o in OVR:
            C, _ = spgemm(a, a, _cfg(o))
            np.testing.assert_array_equal(C.row_ptr, ref.row_ptr)
            np.testing.assert_array_equal(C.col_idx, ref.col_idx)
            np.testing.assert_allclose(C.values, ref.values, rtol=1e-12, atol=0)


def test_window_pass_without_saved_bitmaps(gpu, monkeypatch):
    """Long rows when the saved key bitmaps do not fit (BITMAP_SAVE_SHARE = 0):
    the window kernel rebuilds keys, ranks and columns itself."""
    from paper_2604_19004_b200 import engine, matgen, spgemm
    from oracle import ocean_cpu as oc
    monkeypatch.setattr(engine, "BITMAP_SAVE_SHARE", 0.0)
    a = matgen.rmat(13)
    ref, _ = oc.spgemm(a, a)
    for o in ("symbolic", "estimate"):
        C, _ = spgemm(a, a, _cfg(o))
        np.testing.assert_array_equal(C.row_ptr, ref.row_ptr)
        np.testing.assert_array_equal(C.col_idx, ref.col_idx)
        np.testing.assert_allclose(C.values, ref.values, rtol=1e-12, atol=0)


def test_download_large_ragged(gpu):
    """sg_download (staging ring + native drains) on a ragged 300 MB tensor."""
    from paper_2604_19004_b200.device import download
    n = (300 << 20) // 8 + 12345
    t = torch.arange(n, dtype=torch.int64, device=gpu) * 3 - 7
    for thr in (1, 3, 16):
        out = download(t, thr)
        assert out.dtype == np.int64 and out.shape == (n,)
        np.testing.assert_array_equal(out[:5], [-7, -4, -1, 2, 5])
        assert int(out[-1]) == (n - 1) * 3 - 7
        assert int(out.sum()) == int(t.sum().item())


def test_download_register_failure_falls_back(gpu, monkeypatch):
    """A page-lock failure part way through a registered download finishes
    through the staged ring instead of failing (sg_io.cu download_registered)."""
    from paper_2604_19004_b200.device import download
    n = (600 << 20) // 8 + 777  # > 2 registered 256 MB chunks
    t = torch.arange(n, dtype=torch.int64, device=gpu) * 5 + 3
    for k in ("0", "1"):
        monkeypatch.setenv("SG_TEST_REGISTER_FAIL", k)
        out = download(t, 4)
        assert out.shape == (n,)
        np.testing.assert_array_equal(out[:3], [3, 8, 13])
        assert int(out[-1]) == (n - 1) * 5 + 3
        assert int(out.sum()) == int(t.sum().item())


def test_host_pool_results_recycled(gpu):
    """EngineConfig(host_pool=True): results land in pinned pool buffers that
    return to the pool when dropped and are reused by the next call."""
    import gc
    from paper_2604_19004_b200 import EngineConfig, matgen, spgemm
    from paper_2604_19004_b200.device import HOST_POOL
    from oracle import ocean_cpu as oc
    a = matgen.rmat(14)
    ref, _ = oc.spgemm(a, a)
    for _ in range(2):
        C, _ = spgemm(a, a, EngineConfig(host_pool=True))
        np.testing.assert_array_equal(C.row_ptr, ref.row_ptr)
        np.testing.assert_array_equal(C.col_idx, ref.col_idx)
        np.testing.assert_allclose(C.values, ref.values, rtol=1e-12, atol=0)
        del C
        gc.collect()
    assert HOST_POOL.free, "dropped results should return to the pool"
    HOST_POOL.release()
    assert HOST_POOL.total == 0


@pytest.mark.parametrize("assist", [1.5, 4.0, 64.0])
def test_assisted_symbolic_counts_exact(gpu, assist):
    """Assisted symbolic binning: rows sized by
    products / CR, overfull tables recounted -- counts stay exact even with an
    absurd CR (64) that overflows most tables."""
    import paper_2604_19004_b200._lib as L
    from paper_2604_19004_b200.device import ptr, to_device
    from paper_2604_19004_b200.engine import _Ctx, row_stats
    for name in ("pair05", "corpus1", "enhanced", "bitmapq"):
        c = Case(name)
        ctx = _Ctx(gpu, torch.cuda.current_stream(gpu))
        A, B = to_device(c.A, gpu), to_device(c.B, gpu)
        products, lo, hi, _ = row_stats(ctx, A, B)
        m = A.nrows
        ws, wsb = ctx.workspace(m)
        exact = torch.empty(m, dtype=torch.int64, device=gpu)
        L.call("sg_symbolic", m, B.ncols, ptr(A.row_ptr), ptr(A.col_idx), ptr(B.row_ptr), ptr(B.col_idx),
               ptr(products), ptr(lo), ptr(hi), ptr(exact), None, assist, 0, ws, wsb, ctx.sp)
        np.testing.assert_array_equal(exact.cpu().numpy(), c.d["exact"], err_msg=name)


@pytest.mark.parametrize("force", [False, True])
def test_staged_short_rows(gpu, monkeypatch, force):
    """Symbolic workflow with short rows staged instead of counted (low-CR
    gate; `force` lifts the gate so a high-CR matrix takes the path too)."""
    from paper_2604_19004_b200 import EngineConfig, engine, matgen, spgemm
    from oracle import ocean_cpu as oc
    if force:
        monkeypatch.setattr(engine, "SHORT_ROW_MAX_CR", 1e9)
        a, b = matgen.poisson27(12), None
    else:
        rng = np.random.default_rng(7)
        a = oc.triplets_to_csr(3000, 2000, np.repeat(np.arange(3000), 16), rng.integers(0, 2000, 48000),
                               rng.uniform(0.5, 1.5, 48000))
        b = oc.triplets_to_csr(2000, 900_000, np.repeat(np.arange(2000), 16), rng.integers(0, 900_000, 32000),
                               rng.uniform(0.5, 1.5, 32000))
    b = a if b is None else b
    ref, rrep = oc.spgemm(a, b)
    C, rep = spgemm(a, b, EngineConfig())
    assert rep.workflow == rrep["workflow"] == "symbolic"
    assert rep.kernel_ms["compact"] >= 0.0
    np.testing.assert_array_equal(C.row_ptr, ref.row_ptr)
    np.testing.assert_array_equal(C.col_idx, ref.col_idx)
    np.testing.assert_allclose(C.values, ref.values, rtol=1e-12, atol=0)
    assert rep.overflow_row_count == rrep["overflow_row_count"]


@pytest.mark.parametrize("variant", ["tiny_tiers", "coef1", "coef1.1"])
def test_staged_short_rows_custom_tiers(gpu, variant):
    """Staged short rows (low-CR symbolic workflow) with tiers / coef under
    which the reference plans short rows as FALLBACK or overflows them
    (tiny tiers as test_engine.py:280-292; coef < 1.25 puts a row's distinct
    count over 0.8 x its table).  C and the overflow count equal the oracle's."""
    from paper_2604_19004_b200 import EngineConfig, TierConfig, spgemm
    from oracle import ocean_cpu as oc
    rng = np.random.default_rng(11)
    a = oc.triplets_to_csr(3000, 2000, np.repeat(np.arange(3000), 16), rng.integers(0, 2000, 48000),
                           rng.uniform(0.5, 1.5, 48000))
    b = oc.triplets_to_csr(2000, 900_000, np.repeat(np.arange(2000), 16), rng.integers(0, 900_000, 32000),
                           rng.uniform(0.5, 1.5, 32000))
    if variant == "tiny_tiers":
        tiers = TierConfig(hash_capacities=(8, 16), enhanced_hash_capacity=24, dense_spans=(16, 32))
        ref, rrep = oc.spgemm(a, b, tiers=tiers)
        C, rep = spgemm(a, b, EngineConfig(tiers=tiers))
    else:
        coef = float(variant[4:])
        ref, rrep = oc.spgemm(a, b, coef=coef)
        C, rep = spgemm(a, b, EngineConfig(coef=coef))
    assert rep.workflow == rrep["workflow"] == "symbolic"
    np.testing.assert_array_equal(C.row_ptr, ref.row_ptr)
    np.testing.assert_array_equal(C.col_idx, ref.col_idx)
    np.testing.assert_allclose(C.values, ref.values, rtol=1e-12, atol=0)
    assert rep.overflow_row_count == rrep["overflow_row_count"]


def test_repeat_runs_structure_identical(gpu):
    """Same inputs, same seed: structure and report bit-identical across runs
    (test_engine.py:142-151); values agree to rtol 1e-12 -- fp64 atomics
    may reorder the last bits (known gap)."""
    from paper_2604_19004_b200 import spgemm
    c = Case("corpus1")
    C1, r1 = spgemm(c.A, c.B)
    C2, r2 = spgemm(c.A, c.B)
    np.testing.assert_array_equal(C1.row_ptr, C2.row_ptr)
    np.testing.assert_array_equal(C1.col_idx, C2.col_idx)
    np.testing.assert_allclose(C1.values, C2.values, rtol=1e-12, atol=0)
    for k in REPORT_EXACT + REPORT_FLOAT:
        assert getattr(r1, k) == getattr(r2, k), k


@pytest.mark.parametrize("name", ["pair03", "corpus1", "enhanced", "fig2"])
def test_deterministic_values_bitwise(gpu, name):
    """EngineConfig(deterministic=True): values summed in the reference's
    sequential stream order (sg_det_values) -- bit-identical across runs and
    workflows, and bit-identical to the sequential dict oracle
    (oracle.py:28-39); structure as always."""
    from paper_2604_19004_b200 import EngineConfig, WorkflowOverride, spgemm
    from oracle import ocean_cpu as oc
    c = Case(name)
    seq = oc.dict_spgemm(c.A, c.B)
    outs = []
    for o in (WorkflowOverride.AUTO, WorkflowOverride.FORCE_ESTIMATE, WorkflowOverride.FORCE_UPPER_BOUND):
        C, _ = spgemm(c.A, c.B, EngineConfig(workflow=o, deterministic=True))
        np.testing.assert_array_equal(C.row_ptr, seq.row_ptr)
        np.testing.assert_array_equal(C.col_idx, seq.col_idx)
        np.testing.assert_array_equal(C.values, seq.values)  # bitwise
        outs.append(C.values)
    for v in outs[1:]:
        assert (v == outs[0]).all()


def test_deterministic_values_rmat(gpu):
    """Deterministic mode on hub rows with windows (R-MAT 12): bitwise equal
    to the sequential oracle."""
    from paper_2604_19004_b200 import EngineConfig, matgen, spgemm
    from oracle import ocean_cpu as oc
    a = matgen.rmat(12, seed=4)
    seq = oc.dict_spgemm(a, a)
    C, _ = spgemm(a, a, EngineConfig(deterministic=True))
    np.testing.assert_array_equal(C.col_idx, seq.col_idx)
    np.testing.assert_array_equal(C.values, seq.values)
