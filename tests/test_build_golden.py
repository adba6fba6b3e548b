"""Canonical CSR construction: from_triplets
(reference csr.py:52-80) and transpose (csr.py:90-97).

Goldens in tests/golden/csr_build/ were produced by the real reference
(make_golden.py build_cases).  CPU tests pin the oracle to them; the GPU
tests (sg_coo_to_csr / sg_transpose through the C ABI) must match: structure
bit-exact, values within rtol 1e-12 (duplicates are summed in input order;
the reference's add.reduceat may pair them differently), transposes exact.
"""
import glob
import os

import numpy as np
import pytest

from oracle import ocean_cpu as oc

BUILD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "csr_build")
CASES = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(BUILD, "triplets*.npz")))


def _load(name):
    return dict(np.load(os.path.join(BUILD, name + ".npz")))


def _check(got_ptr, got_col, got_val, d, pre="", rtol=1e-12):
    np.testing.assert_array_equal(np.asarray(got_ptr), d[pre + "ptr"])
    np.testing.assert_array_equal(np.asarray(got_col), d[pre + "col"])
    np.testing.assert_allclose(np.asarray(got_val), d[pre + "val"], rtol=rtol, atol=0)


@pytest.mark.parametrize("name", CASES)
def test_oracle_triplets_and_transpose_match_reference(name):
    d = _load(name)
    nr, nc = (int(x) for x in d["shape"])
    c = oc.triplets_to_csr(nr, nc, d["rows"], d["cols"], d["vals"])
    _check(c.row_ptr, c.col_idx, c.values, d)
    t = oc.transpose(c)
    np.testing.assert_array_equal(t.row_ptr, d["t_ptr"])
    np.testing.assert_array_equal(t.col_idx, d["t_col"])
    np.testing.assert_array_equal(t.values, c.values[np.argsort(c.col_idx, kind="stable")])


def test_goldens_present():
    assert len(CASES) >= 6


@pytest.fixture(scope="module")
def gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda", 0)


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_device_from_triplets_and_transpose(gpu, name):
    from paper_2604_19004_b200.build import from_triplets_device, transpose_device
    d = _load(name)
    nr, nc = (int(x) for x in d["shape"])
    c = from_triplets_device(nr, nc, d["rows"], d["cols"], d["vals"], device=gpu)
    h = c.to_host()
    _check(h.row_ptr, h.col_idx, h.values, d)
    t = transpose_device(c).to_host()
    np.testing.assert_array_equal(t.row_ptr, d["t_ptr"])
    np.testing.assert_array_equal(t.col_idx, d["t_col"])
    np.testing.assert_array_equal(t.values, h.values[np.argsort(h.col_idx, kind="stable")])


@pytest.mark.gpu
def test_device_build_errors_and_large(gpu):
    import torch
    from paper_2604_19004_b200 import matgen, multiply_mode
    from paper_2604_19004_b200.build import from_triplets_device, transpose_device
    from paper_2604_19004_b200.device import to_device
    with pytest.raises(ValueError, match="out of range"):
        from_triplets_device(3, 3, [0, 3], [0, 0], [1.0, 1.0], device=gpu)
    with pytest.raises(ValueError, match="out of range"):
        from_triplets_device(3, 3, [0, 1], [0, -1], [1.0, 1.0], device=gpu)
    with pytest.raises(ValueError, match="32-bit"):
        from_triplets_device(2 ** 31, 3, [], [], [], device=gpu)
    # transpose of a config-scale matrix equals the oracle's, exactly
    a = matgen.rmat(16)
    t = transpose_device(to_device(a, gpu)).to_host()
    ref = oc.transpose(a)
    np.testing.assert_array_equal(t.row_ptr, ref.row_ptr)
    np.testing.assert_array_equal(t.col_idx, ref.col_idx)
    np.testing.assert_array_equal(t.values, ref.values)
    # AA^T operand on the device (engine.py:113-128)
    A, At = multiply_mode(to_device(a, gpu), "aat")
    np.testing.assert_array_equal(At.col_idx.cpu().numpy(), ref.col_idx)
    # triplets from the device, shuffled, round-trip to the same CSR
    rows = np.repeat(np.arange(a.nrows), np.diff(a.row_ptr))
    perm = np.random.default_rng(0).permutation(a.nnz)
    c = from_triplets_device(a.nrows, a.ncols, torch.from_numpy(rows[perm]).to(gpu),
                             torch.from_numpy(a.col_idx[perm].astype(np.int64)).to(gpu),
                             torch.from_numpy(a.values[perm]).to(gpu), device=gpu).to_host()
    np.testing.assert_array_equal(c.row_ptr, a.row_ptr)
    np.testing.assert_array_equal(c.col_idx, a.col_idx)
    np.testing.assert_array_equal(c.values, a.values)
