"""CPU: the oracle port pinned to the real reference at config scale.

The config-scale fixtures (tests/golden/configs, made by the real reference
with tests/golden/make_config_golden.py) are checked against the oracle port
on the same rows: two R-MAT-20 row blocks (the hub block 0 and a mid block).
The GPU tests use the same port as their per-entry checker at this scale.
"""
import pytest

import config_golden as cg


@pytest.fixture(scope="module")
def rmat20():
    from paper_2604_19004_b200 import matgen
    return matgen.make_config("rmat20")[0]


@pytest.mark.parametrize("i", [0, 15])
def test_port_matches_reference_rmat20_block(rmat20, i):
    from paper_2604_19004_b200 import matgen
    from oracle import ocean_cpu as oc
    meta, arrays = cg.load("rmat20_blocks")
    b = meta["blocks"][i]
    c, rep = oc.spgemm(matgen.rows_slice(rmat20, b["lo"], b["hi"]), rmat20, workflow="symbolic",
                       workers=oc.default_workers())
    cg.check(c, b, arrays, prefix=f"b{i}_")


def test_block_list_matches_fixture(rmat20):
    from paper_2604_19004_b200 import matgen
    meta, _ = cg.load("rmat20_blocks")
    blocks = matgen.stratified_blocks(matgen.row_products(rmat20, rmat20))
    assert [tuple(x) for x in blocks] == [(b["lo"], b["hi"]) for b in meta["blocks"]]
    assert sum(b["products"] for b in meta["blocks"]) >= 0.02 * meta["total_products"]
