"""est-eval harness (reference cli.py:301-341 and
engine.py:218-226): per-register estimation error, overflow ratio and
sampled CR under FORCE_ESTIMATE, against records produced by the real
reference (tests/golden/est_eval.json, make_golden.py est_eval_cases).

Errors are reductions over rows (mean / population std), so they are checked
within rtol 1e-9 (atol 1e-12 for the zero-variance cases); counts exactly.
"""
import json
import os

import pytest

from golden_io import Case

GOLD = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "est_eval.json")))
KEYS = sorted(GOLD)


def _close(got, want):
    if want is None:
        assert got is None
    else:
        assert got == pytest.approx(want, rel=1e-9, abs=1e-12)


@pytest.mark.parametrize("key", KEYS)
def test_oracle_est_errors_match_reference(key):
    from oracle import ocean_cpu as oc
    name, m = key.split("/")
    c = Case(name)
    _, rep = oc.spgemm(c.A, c.B, workflow="estimate", registers=int(m), compute_errors=True)
    want = GOLD[key]
    assert rep["overflow_row_count"] == want["overflow_row_count"]
    assert rep["nnz_c"] == want["nnz_c"]
    for k in ("est_mean_rel_err", "est_std_rel_err", "cr_hat", "cr_true"):
        _close(rep[k], want[k])


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted({k.split("/")[0] for k in KEYS}))
def test_device_est_eval_matches_reference(name):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2604_19004_b200.est_eval import est_eval
    c = Case(name)
    recs = est_eval(c.A, c.B, op="ab", name=name)
    assert [r["registers"] for r in recs] == [32, 64, 128]
    for r in recs:
        want = GOLD[f"{name}/{r['registers']}"]
        assert r["overflow_rows"] == want["overflow_row_count"]
        assert r["overflow_ratio"] == want["overflow_row_count"] / c.A.nrows
        assert r["nnz_c"] == want["nnz_c"]
        _close(r["mean_rel_err"], want["est_mean_rel_err"])
        _close(r["std_rel_err"], want["est_std_rel_err"])
        _close(r["cr_sampled"], want["cr_hat"])
        _close(r["cr_true"], want["cr_true"])


def test_est_eval_rejects_bad_registers():
    from paper_2604_19004_b200.est_eval import est_eval
    with pytest.raises(ValueError, match="32, 64 or 128"):
        est_eval(None, registers=(16,))
