"""Config-scale GPU parity (BASELINE configs at their real size).

* Poisson 27-pt 64^3 A^2 and rect 1M x 64k * 64k x 1M: the whole C against the
  real reference's fixture (structure sha256, value group sums, sampled rows)
  and, entry by entry, against the oracle port at run time.
* R-MAT scale 20 A^2 (the bench's headline config): the FULL C is computed on
  the GPU exactly as bench.py does (device-resident operands, return_device),
  then row blocks are sliced out of it and compared: the 20 products-
  stratified blocks of matgen.stratified_blocks (hub rows first) against the
  real reference's fixture, and entry by entry against the oracle port for
  the hub block, a spread of the others, and the block whose row_ptr crosses
  2^31 (int64 output offsets; C has 9.7e9 entries).

Rows are independent (reference engine.py:13-14), so a row
block of C equals the reference run on those rows of A.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import config_golden as cg  # noqa: E402

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module")
def gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2604_19004_b200 import _lib
    _lib.load()
    return torch.device("cuda", 0)


REPORT_EXACT = ("workflow", "registers", "overflow_row_count", "nnz_c", "total_products", "bitmap_query")


@pytest.mark.parametrize("name", ["poisson64", "rect"])
def test_whole_config_vs_reference(gpu, name):
    from paper_2604_19004_b200 import EngineConfig, matgen, spgemm
    from oracle import ocean_cpu as oc
    if not cg.available(name):
        pytest.fail(f"fixture {name} missing (tests/golden/make_config_golden.py)")
    meta, arrays = cg.load(name)
    a, b = matgen.make_config(name)
    c, rep = spgemm(a, b, EngineConfig())
    cg.check(c, meta, arrays)
    want = meta["report"]
    for k in REPORT_EXACT:
        assert getattr(rep, k) == want[k], (name, k, getattr(rep, k), want[k])
    assert rep.cr_hat == pytest.approx(want["cr_hat"], rel=1e-12)
    ref, _ = oc.spgemm(a, b, workers=oc.default_workers())
    cg.compare_exact(c, ref)


def _row_ptr_crossing(row_ptr_dev, bound):
    """First row r with row_ptr[r] <= bound < row_ptr[r+1] (or None)."""
    rp = row_ptr_dev
    if int(rp[-1]) <= bound:
        return None
    r = int(torch.searchsorted(rp, torch.tensor([bound], dtype=torch.int64, device=rp.device), right=True)[0]) - 1
    return max(r, 0)


def test_rmat20_blocks_from_full_c(gpu):
    from paper_2604_19004_b200 import EngineConfig, matgen, spgemm
    from paper_2604_19004_b200.device import to_device
    from oracle import ocean_cpu as oc
    if not cg.available("rmat20_blocks"):
        pytest.fail("fixture rmat20_blocks missing (tests/golden/make_config_golden.py)")
    meta, arrays = cg.load("rmat20_blocks")
    a, _ = matgen.make_config("rmat20")
    A = to_device(a, gpu)
    C, rep = spgemm(A, A, EngineConfig(return_device=True))
    assert rep.nnz_c == 9_708_383_452 and rep.total_products == 20_922_476_755
    per = matgen.row_products(a, a)
    blocks = matgen.stratified_blocks(per)
    assert [tuple(x) for x in blocks] == [(b["lo"], b["hi"]) for b in meta["blocks"]]
    # every block against the real reference's fixture
    for i, bm in enumerate(meta["blocks"]):
        cg.check(C.rows(bm["lo"], bm["hi"]), bm, arrays, prefix=f"b{i}_")
    # entry-by-entry against the oracle port: hubs, a spread, and the blocks
    # whose output offsets cross 2^31 and 2^32
    check = [blocks[i] for i in (0, 3, 7, 11, 15, 19)]
    for bound in (2 ** 31, 2 ** 32):
        r = _row_ptr_crossing(C.row_ptr, bound)
        assert r is not None
        check.append((max(0, r - 2), min(a.nrows, r + 3)))
    workers = oc.default_workers()
    for lo, hi in check:
        ref, _ = oc.spgemm(matgen.rows_slice(a, lo, hi), a, workflow="symbolic", workers=workers)
        cg.compare_exact(C.rows(lo, hi), ref)
    del C
    torch.cuda.empty_cache()
