"""Seeded synthetic inputs for the five BASELINE configs.

Host-side input preparation only (never inside a timed region).  Values are
U[0.5, 1.5] and duplicates are summed, following the reference's generators
(``pkg/tests/matgen.py:3-6``) so that relative tolerances stay meaningful.
Canonicalisation follows ``from_triplets`` (``csr.py:52-80``).
"""

from __future__ import annotations

import numpy as np

from .csr import CsrMatrix, from_triplets


def erdos_renyi(n: int = 10_000, nnz: int = 80_000, seed: int = 1) -> CsrMatrix:
    """Config 1: 80k uniform (row, col) draws on n x n, seed 1."""
    rng = np.random.default_rng(seed)
    rows = rng.integers(0, n, nnz)
    cols = rng.integers(0, n, nnz)
    vals = rng.uniform(0.5, 1.5, nnz)
    return from_triplets(n, n, rows, cols, vals)


def poisson27(g: int = 64, seed: int = 2) -> CsrMatrix:
    """Config 2: 27-point stencil on a g^3 grid, idx = x*g*g + y*g + z."""
    rng = np.random.default_rng(seed)
    n = g ** 3
    x, y, z = np.meshgrid(np.arange(g), np.arange(g), np.arange(g), indexing="ij")
    x, y, z = x.ravel(), y.ravel(), z.ravel()
    src = x * g * g + y * g + z
    rows, cols = [], []
    for dx in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dz in (-1, 0, 1):
                xx, yy, zz = x + dx, y + dy, z + dz
                ok = (xx >= 0) & (xx < g) & (yy >= 0) & (yy < g) & (zz >= 0) & (zz < g)
                rows.append(src[ok])
                cols.append((xx * g * g + yy * g + zz)[ok])
    rows = np.concatenate(rows)
    cols = np.concatenate(cols)
    vals = rng.uniform(0.5, 1.5, len(rows))
    return from_triplets(n, n, rows, cols, vals)


def rmat(scale: int = 20, edge_factor: int = 16, seed: int = 3,
         abcd=(0.57, 0.19, 0.19, 0.05)) -> CsrMatrix:
    """Configs 3 / 5: R-MAT with per-bit quadrant choice, no permutation,
    self-loops kept.  row bit = u >= a+b; col bit = a <= u < a+b or u >= a+b+c."""
    a, b, c, _ = abcd
    rng = np.random.default_rng(seed)
    n = 1 << scale
    m = edge_factor * n
    rows = np.zeros(m, dtype=np.int64)
    cols = np.zeros(m, dtype=np.int64)
    for bit in range(scale):
        u = rng.random(m)
        rb = u >= a + b
        cb = ((u >= a) & (u < a + b)) | (u >= a + b + c)
        rows |= rb.astype(np.int64) << (scale - 1 - bit)
        cols |= cb.astype(np.int64) << (scale - 1 - bit)
    vals = rng.uniform(0.5, 1.5, m)
    return from_triplets(n, n, rows, cols, vals)


def rect_pair(m: int = 1_000_000, k: int = 64_000, n: int = 1_000_000,
              per_row: int = 16, seed: int = 4):
    """Config 4: A is m x k with 16 uniform columns per row, B is k x n with 16
    uniform columns per row (duplicates summed)."""
    rng = np.random.default_rng(seed)
    ar = np.repeat(np.arange(m, dtype=np.int64), per_row)
    ac = rng.integers(0, k, m * per_row)
    av = rng.uniform(0.5, 1.5, m * per_row)
    br = np.repeat(np.arange(k, dtype=np.int64), per_row)
    bc = rng.integers(0, n, k * per_row)
    bv = rng.uniform(0.5, 1.5, k * per_row)
    return from_triplets(m, k, ar, ac, av), from_triplets(k, n, br, bc, bv)


CONFIGS = {
    "er10k": "C = A*A, Erdos-Renyi 10k x 10k, ~8 nnz/row, fp64",
    "poisson64": "C = A*A, 27-point Poisson stencil on a 64^3 grid",
    "rmat20": "C = A*A, R-MAT scale 20 edge-factor 16",
    "rect": "C = A*B, A 1M x 64k, B 64k x 1M, 16 nnz/row",
    "rmat23": "C = A*A, R-MAT scale 23 edge-factor 16 (row-sharded)",
}


def make_config(name: str):
    """(A, B) for one of the BASELINE configs."""
    if name == "er10k":
        a = erdos_renyi()
        return a, a
    if name == "poisson64":
        a = poisson27()
        return a, a
    if name == "rmat20":
        a = rmat(20)
        return a, a
    if name == "rmat23":
        a = rmat(23)
        return a, a
    if name == "rect":
        return rect_pair()
    if name.startswith("rmat"):
        a = rmat(int(name[4:]))
        return a, a
    raise ValueError(f"unknown config {name!r}")


def row_products(a, b) -> np.ndarray:
    """Intermediate products per row of A·B (analysis.py:100-104), host side,
    for choosing sample blocks (input preparation, not the multiply)."""
    cum = np.r_[0, np.cumsum(np.diff(np.asarray(b.row_ptr))[np.asarray(a.col_idx)])]
    rp = np.asarray(a.row_ptr)
    return cum[rp[1:]] - cum[rp[:-1]]


def stratified_blocks(per_row: np.ndarray, nblocks: int = 20, block_frac: float = 1e-3) -> list:
    """Deterministic products-stratified row blocks of A.

    Block s starts at the row holding product number s/nblocks x total (so
    block 0 starts at row 0: the hub rows of an unpermuted R-MAT) and takes
    whole rows until it holds block_frac x total products (at least one row).
    The same list drives the CPU-reference sample (bench.py), the sampled-row
    parity check of the bench's own output, and the config-scale GPU parity
    tests (fixtures: tests/golden/make_config_golden.py).  Valid as a parity
    sample because Gustavson rows are independent (PAPER.md:153,
    engine.py:13-14)."""
    per = np.asarray(per_row, dtype=np.int64)
    m = len(per)
    cum = np.r_[0, np.cumsum(per)]
    total = int(cum[-1])
    if m == 0 or total == 0:
        return [(0, m)] if m else []
    target = max(1, int(total * block_frac))
    out = []
    for s in range(nblocks):
        start = int(np.searchsorted(cum, s * total // nblocks, side="right")) - 1
        start = max(0, min(start, m - 1))
        end = int(np.searchsorted(cum, cum[start] + target, side="left"))
        end = max(start + 1, min(end, m))
        if out and start < out[-1][1]:
            start = out[-1][1]
            if start >= m:
                break
            end = max(end, start + 1)
        out.append((start, end))
    return out


def rows_slice(a, lo: int, hi: int):
    """Host CSR of rows [lo, hi) of a (same column space)."""
    rp = np.asarray(a.row_ptr)
    s, e = int(rp[lo]), int(rp[hi])
    return CsrMatrix(hi - lo, a.ncols, rp[lo:hi + 1] - s, np.asarray(a.col_idx)[s:e], np.asarray(a.values)[s:e])
