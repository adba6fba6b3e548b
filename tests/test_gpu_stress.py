"""Randomised GPU parity sweep: shapes chosen to reach every accumulator and
code path (hub rows -> numeric windows; sparse wide spans -> block hash;
columns >= 2^23 -> the warp hash's shared-memory sort fallback; tiny column
ranges -> heavy duplicate merging; empty rows; fp32), all four workflows
against the oracle (structure exact, values rtol 1e-12)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

OVR = ("auto", "symbolic", "estimate", "upper")


def _mk(rng, r, c, lens):
    from oracle import ocean_cpu as oc
    lens = np.minimum(lens, c).astype(int)
    rows = np.repeat(np.arange(r), lens)
    cols = rng.integers(0, c, len(rows))
    return oc.triplets_to_csr(r, c, rows, cols, rng.uniform(0.5, 1.5, len(rows)))


def _case(seed):
    from paper_2604_19004_b200 import matgen
    rng = np.random.default_rng(10_000 + seed)
    kind = seed % 5
    if kind == 0:  # R-MAT: hub rows with windows
        a = matgen.rmat(int(rng.integers(10, 13)), seed=int(seed))
        return a, a
    if kind == 1:  # sparse wide spans: block-hash rows
        n, k, m = 400, 3000, 3_000_000
        a = _mk(rng, n, k, (rng.pareto(1.2, n) + 1) * 30)
        b = _mk(rng, k, m, (rng.pareto(1.5, k) + 1) * 20)
        return a, b
    if kind == 2:  # columns beyond 2^23: warp-hash sort fallback
        n, k, m = 3000, 2000, 50_000_000
        a = _mk(rng, n, k, rng.integers(0, 20, n))
        b = _mk(rng, k, m, rng.integers(0, 25, k))
        return a, b
    if kind == 3:  # tiny column range: heavy duplicate merging, empty rows
        n, k, m = 2000, 500, 64
        lens = rng.integers(0, 40, n) * (rng.random(n) < 0.7)
        a = _mk(rng, n, k, lens)
        b = _mk(rng, k, m, rng.integers(0, 30, k))
        return a, b
    n, k, m = 1500, 1500, 200_000  # mixed Pareto rows
    a = _mk(rng, n, k, (rng.pareto(1.1, n) + 0.1) * 15)
    b = _mk(rng, k, m, (rng.pareto(1.1, k) + 0.1) * 40)
    return a, b


@pytest.mark.parametrize("seed", range(40))
def test_random_shapes_all_workflows(seed):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from oracle import ocean_cpu as oc
    from paper_2604_19004_b200 import EngineConfig, WorkflowOverride, spgemm
    ov = {"auto": WorkflowOverride.AUTO, "symbolic": WorkflowOverride.FORCE_SYMBOLIC,
          "estimate": WorkflowOverride.FORCE_ESTIMATE, "upper": WorkflowOverride.FORCE_UPPER_BOUND}
    a, b = _case(seed)
    ref, rrep = oc.spgemm(a, b)
    for o in OVR:
        C, rep = spgemm(a, b, EngineConfig(workflow=ov[o]))
        np.testing.assert_array_equal(C.row_ptr, ref.row_ptr, err_msg=f"seed {seed} {o}")
        np.testing.assert_array_equal(C.col_idx, ref.col_idx, err_msg=f"seed {seed} {o}")
        np.testing.assert_allclose(C.values, ref.values, rtol=1e-12, atol=0, err_msg=f"seed {seed} {o}")
        assert rep.nnz_c == rrep["nnz_c"]
    if seed % 4 == 0:  # fp32 variant (accumulates in fp64)
        C, _ = spgemm(a, b, EngineConfig(dtype="f32"))
        np.testing.assert_array_equal(C.col_idx, ref.col_idx)
        np.testing.assert_allclose(C.values, ref.values, rtol=1e-5, atol=0)
