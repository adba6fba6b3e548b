"""CPU restatement of the reference's estimation-based SpGEMM (TEST INFRASTRUCTURE).

THIS MODULE IS THE PARITY CHECKER, NOT THE PRODUCT.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline / reference arm may
import it.  The shipped path (``paper_2604_19004_b200``) never imports it and
fails loudly when its CUDA library is missing.

It restates, stage by stage, the algorithm of the reference package
``sketchgemm`` 0.1.0 (``/root/reference/pkg/src/sketchgemm``) in numpy, so that
(1) the GPU results can be checked on identical inputs without the reference
tree present (it does not exist on the GPU box) and (2) the reference's CPU
path can be timed on the GPU box's host cores (``cpu_baseline.kind = "port"``).

Parity pin: ``tests/golden/make_golden.py`` imports the real reference in the
build container and records its outputs (C, row stats, sketches, plans,
reports) for a corpus of seeded inputs; ``tests/test_oracle_golden.py`` checks
this restatement against those fixtures (structure bit-exact, values rtol
1e-12, plans / sketches / estimates exact).

Every function cites the reference file:line it follows.  Paths are relative
to ``/root/reference/pkg/src/sketchgemm/``.
"""

from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

# ---------------------------------------------------------------------------
# constants (analysis.py:26-33, accumulate.py:33-36,56-61, hll.py:23-31,
# predict.py:24, engine.py:36)

UB_AVG = 64.0
ER_MIN = 8.0
CR_MIN = 8.0
REG_ER = 48.0
SAMPLE_RATIO, SAMPLE_MIN, SAMPLE_MAX = 0.03, 600, 10_000
LOAD_LIMIT = 0.8
P_OF_M = {32: 5, 64: 6, 128: 7}
ALPHA_OF_M = {32: 0.697, 64: 0.709, 128: 0.7213 / (1 + 1.079 / 128)}

KIND_HASH, KIND_ENH, KIND_DENSE, KIND_ESC, KIND_FB = 0, 1, 2, 3, 4

_K1 = np.uint64(0x9E3779B97F4A7C15)
_K2 = np.uint64(0xBF58476D1CE4E5B9)
_K3 = np.uint64(0x94D049BB133111EB)


@dataclass
class Tiers:
    """Accumulator ladder (accumulate.py:47-61)."""

    hash_caps: tuple = (256, 512, 1024, 2048, 4096)
    enh_cap: int = 12288
    dense_spans: tuple = (1024, 2048, 4096, 8192, 16384)
    esc_max: int = 64
    coef: float = 1.5
    bitmap_threshold: float = 2.0

    @classmethod
    def of(cls, t) -> "Tiers":
        if t is None:
            return cls()
        if isinstance(t, Tiers):
            return t
        return cls(tuple(t.hash_capacities), int(t.enhanced_hash_capacity),
                   tuple(t.dense_spans), int(t.esc_max_products),
                   float(t.expansion_coef), float(t.bitmap_query_threshold))


class Csr:
    """Minimal canonical CSR holder (csr.py:24-49)."""

    def __init__(self, nrows, ncols, row_ptr, col_idx, values):
        self.nrows, self.ncols = int(nrows), int(ncols)
        self.row_ptr = np.asarray(row_ptr, dtype=np.int64)
        self.col_idx = np.asarray(col_idx, dtype=np.int32)
        self.values = np.asarray(values, dtype=np.float64)

    @property
    def nnz(self):
        return int(self.row_ptr[-1])


def as_csr(m) -> Csr:
    return m if isinstance(m, Csr) else Csr(m.nrows, m.ncols, m.row_ptr, m.col_idx, m.values)


def triplets_to_csr(nrows, ncols, rows, cols, vals) -> Csr:
    """Sort by (row, col), sum duplicates (csr.py:52-80)."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    vals = np.asarray(vals, dtype=np.float64)
    if rows.size == 0:
        return Csr(nrows, ncols, np.zeros(nrows + 1, np.int64), np.empty(0, np.int32),
                   np.empty(0, np.float64))
    key = rows * ncols + cols
    perm = np.argsort(key, kind="stable")
    key, vals = key[perm], vals[perm]
    head = np.flatnonzero(np.r_[True, key[1:] != key[:-1]])
    uk = key[head]
    ptr = np.zeros(nrows + 1, np.int64)
    ptr[1:] = np.cumsum(np.bincount(uk // ncols, minlength=nrows))
    return Csr(nrows, ncols, ptr, (uk % ncols).astype(np.int32), np.add.reduceat(vals, head))


def transpose(a: Csr) -> Csr:
    """Exact transpose (csr.py:90-97): a column-major counting sort; entries
    of one output row keep ascending source-row order."""
    a = as_csr(a)
    nnz = int(a.row_ptr[-1])
    cnt = np.bincount(np.asarray(a.col_idx[:nnz], np.int64), minlength=a.ncols)
    ptr = np.zeros(a.ncols + 1, np.int64)
    ptr[1:] = np.cumsum(cnt)
    src_row = np.repeat(np.arange(a.nrows, dtype=np.int64), np.diff(a.row_ptr))
    perm = np.argsort(np.asarray(a.col_idx[:nnz], np.int64), kind="stable")
    return Csr(a.ncols, a.nrows, ptr, src_row[perm].astype(np.int32), np.asarray(a.values)[perm])


# ---------------------------------------------------------------------------
# L1 primitives (hll.py, expand.py)

def hash64(keys) -> np.ndarray:
    """splitmix64 finaliser on uint64 (hll.py:34-49)."""
    z = np.asarray(keys, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = z + _K1
        z = (z ^ (z >> np.uint64(30))) * _K2
        z = (z ^ (z >> np.uint64(27))) * _K3
        return z ^ (z >> np.uint64(31))


def register_index_rank(keys, p: int):
    """idx = low p bits; rank = (64-p) - bit_length(h >> p) + 1 (hll.py:64-76, 52-61)."""
    h = hash64(np.atleast_1d(np.asarray(keys, dtype=np.uint64)))
    idx = (h & np.uint64((1 << p) - 1)).astype(np.int64)
    w = h >> np.uint64(p)
    # bit_length via float64 log2 is unsafe near powers of two; use frexp on halves
    hi = (w >> np.uint64(32)).astype(np.float64)
    lo = (w & np.uint64(0xFFFFFFFF)).astype(np.float64)
    bl_hi = np.frexp(hi)[1].astype(np.int64)            # 0 for 0, else bit_length
    bl_lo = np.frexp(lo)[1].astype(np.int64)
    bitlen = np.where(hi > 0, bl_hi + 32, bl_lo)
    rank = (64 - p) - bitlen + 1
    return idx, rank.astype(np.uint8)


_INV_POW2 = 2.0 ** -np.arange(64)


def hll_estimate(regs: np.ndarray) -> np.ndarray:
    """alpha*m*m / sum 2^-r with linear counting when small (hll.py:79-86)."""
    regs = np.atleast_2d(regs)
    m = regs.shape[1]
    raw = ALPHA_OF_M[m] * m * m / _INV_POW2[regs].sum(axis=1)
    zeros = (regs == 0).sum(axis=1)
    lin = np.where(zeros > 0, m * np.log(m / np.maximum(zeros, 1)), 0.0)
    return np.where((raw <= 2.5 * m) & (zeros > 0), lin, raw)


def ranges(starts, lens) -> np.ndarray:
    """Flat indices of [starts[i], starts[i]+lens[i]) (expand.py:18-26)."""
    lens = np.asarray(lens, dtype=np.int64)
    n = int(lens.sum())
    if n == 0:
        return np.empty(0, np.int64)
    base = np.repeat(np.asarray(starts, dtype=np.int64) - (np.cumsum(lens) - lens), lens)
    return base + np.arange(n, dtype=np.int64)


def expand(a: Csr, b: Csr, rows, values=True):
    """Gustavson product stream in A-row / A-nnz / B-nnz order (expand.py:29-56)."""
    st = a.row_ptr[rows]
    al = a.row_ptr[rows + 1] - st
    asel = ranges(st, al)
    loc = np.repeat(np.arange(len(rows), dtype=np.int64), al)
    k = a.col_idx[asel]
    bs = b.row_ptr[k]
    bl = b.row_ptr[k + 1] - bs
    bsel = ranges(bs, bl)
    prow = np.repeat(loc, bl)
    pcol = b.col_idx[bsel].astype(np.int64)
    if not values:
        return prow, pcol, None
    return prow, pcol, np.repeat(a.values[asel], bl) * b.values[bsel]


def reduce_cells(prow, pcol, pval, ncols):
    """Stable sort by (row, col) and sum runs (expand.py:59-78)."""
    if len(prow) == 0:
        e = np.empty(0, np.int64)
        return e, e, (None if pval is None else np.empty(0, np.float64))
    key = prow * np.int64(ncols) + pcol
    perm = np.argsort(key, kind="stable")
    key = key[perm]
    head = np.flatnonzero(np.r_[True, key[1:] != key[:-1]])
    uk = key[head]
    uval = None if pval is None else np.add.reduceat(pval[perm], head)
    return uk // ncols, uk % ncols, uval


# ---------------------------------------------------------------------------
# L2 analysis + prediction (analysis.py, predict.py)

@dataclass
class Stats:
    products: np.ndarray
    total: int
    er: float
    span_lo: np.ndarray
    span_hi: np.ndarray

    def spans(self):
        return np.where(self.products > 0, self.span_hi - self.span_lo + 1, 0)


def row_stats(a: Csr, b: Csr) -> Stats:
    """Products per row, ER, span bounds (analysis.py:96-128)."""
    bn = np.diff(b.row_ptr)
    cum = np.r_[0, np.cumsum(bn[a.col_idx])]
    products = cum[a.row_ptr[1:]] - cum[a.row_ptr[:-1]]
    total = int(products.sum())
    first = np.full(b.nrows, b.ncols, np.int64)
    last = np.full(b.nrows, -1, np.int64)
    has = bn > 0
    first[has] = b.col_idx[b.row_ptr[:-1][has]]
    last[has] = b.col_idx[b.row_ptr[1:][has] - 1]
    lo = np.full(a.nrows, b.ncols, np.int64)
    hi = np.full(a.nrows, -1, np.int64)
    ne = np.flatnonzero(np.diff(a.row_ptr) > 0)
    if len(ne):
        lo[ne] = np.minimum.reduceat(first[a.col_idx], a.row_ptr[ne])
        hi[ne] = np.maximum.reduceat(last[a.col_idx], a.row_ptr[ne])
    lo[products == 0] = b.ncols
    hi[products == 0] = -1
    return Stats(products, total, total / a.nnz if a.nnz else 0.0, lo, hi)


def b_sketches(b: Csr, p: int) -> np.ndarray:
    """u8[k, 2^p] register table, one HLL per B row (analysis.py:131-146)."""
    m = 1 << p
    regs = np.zeros((b.nrows, m), np.uint8)
    if b.nnz:
        idx, rank = register_index_rank(b.col_idx, p)
        key = np.repeat(np.arange(b.nrows, dtype=np.int64), np.diff(b.row_ptr)) * m + idx
        perm = np.argsort(key, kind="stable")
        key, rank = key[perm], rank[perm]
        head = np.flatnonzero(np.r_[True, key[1:] != key[:-1]])
        regs.reshape(-1)[key[head]] = np.maximum.reduceat(rank, head)
    return regs


def merged_estimates(a: Csr, regs: np.ndarray, rows: np.ndarray) -> np.ndarray:
    """Max-merge selected B sketches per A row, then estimate (analysis.py:149-169)."""
    lens = a.row_ptr[rows + 1] - a.row_ptr[rows]
    out = np.zeros(len(rows), np.float64)
    live = np.flatnonzero(lens > 0)
    if len(live) == 0:
        return out
    sel = ranges(a.row_ptr[rows[live]], lens[live])
    g = regs[a.col_idx[sel]]
    starts = np.r_[0, np.cumsum(lens[live])[:-1]]
    out[live] = hll_estimate(np.maximum.reduceat(g, starts, axis=0))
    return out


def sample_rows(nrows: int, ratio: float, min_n: int, max_n: int, seed: int) -> np.ndarray:
    """Sorted distinct sample rows; all rows when n >= nrows (analysis.py:182-190)."""
    n = int(np.clip(round(ratio * nrows), min(min_n, nrows), min(max_n, nrows)))
    if n >= nrows:
        return np.arange(nrows, dtype=np.int64)
    return np.sort(np.random.default_rng(seed).choice(nrows, size=n, replace=False)).astype(np.int64)


def cr_from_sample(products_sel: np.ndarray, est: np.ndarray):
    """Ratio-of-sums CR + per-row CR mean / population std (analysis.py:192-196)."""
    prods = products_sel.astype(np.float64)
    cr_hat = float(prods.sum() / max(1.0, est.sum()))
    row_cr = np.where(prods > 0, prods / np.maximum(est, 1.0), 1.0)
    return cr_hat, float(row_cr.mean()), float(row_cr.std())


def choose_registers(er: float) -> int:
    """analysis.py:199-203"""
    return 32 if er < REG_ER else 64


def choose_workflow(avg: float, er: float, cr_hat: float) -> str:
    """analysis.py:206-217"""
    if avg < UB_AVG:
        return "upper"
    if er >= ER_MIN and cr_hat >= CR_MIN:
        return "estimate"
    return "symbolic"


def exact_counts(a: Csr, b: Csr, st: Stats, span_limit: int = 16384) -> np.ndarray:
    """Symbolic pass: bitmap counts for narrow rows, sort-based otherwise (predict.py:39-84)."""
    counts = np.zeros(a.nrows, np.int64)
    spans = st.spans()
    live = st.products > 0
    narrow = np.flatnonzero(live & (spans <= span_limit))
    budget = 1 << 24
    i = 0
    while i < len(narrow):
        j, w = i, 0
        while j < len(narrow) and (w == 0 or w + spans[narrow[j]] <= budget):
            w += spans[narrow[j]]
            j += 1
        rows = narrow[i:j]
        sp = spans[rows]
        off = np.r_[0, np.cumsum(sp)]
        prow, pcol, _ = expand(a, b, rows, values=False)
        occ = np.bincount(off[prow] + pcol - st.span_lo[rows][prow], minlength=off[-1]) > 0
        c = np.r_[0, np.cumsum(occ)]
        counts[rows] = c[off[1:]] - c[off[:-1]]
        i = j
    wide = np.flatnonzero(live & (spans > span_limit))
    if len(wide):
        prow, pcol, _ = expand(a, b, wide, values=False)
        ur, _, _ = reduce_cells(prow, pcol, None, b.ncols)
        counts[wide] = np.bincount(ur, minlength=len(wide))
    return counts


def estimate_all(a: Csr, regs: np.ndarray, block_nnz: int = 1 << 22) -> np.ndarray:
    """Estimate pass over all rows in nnz-bounded blocks (predict.py:87-103)."""
    est = np.zeros(a.nrows, np.float64)
    if a.nrows == 0:
        return est
    cuts = np.searchsorted(a.row_ptr, np.arange(0, a.nnz + block_nnz, block_nnz))
    cuts[-1] = a.nrows
    for lo, hi in zip(cuts[:-1], cuts[1:]):
        if hi > lo:
            r = np.arange(lo, hi, dtype=np.int64)
            est[r] = merged_estimates(a, regs, r)
    return est


# ---------------------------------------------------------------------------
# L3 binning (accumulate.py:104-181)

def plan(pred: np.ndarray, pred_kind: str, workflow: str, st: Stats, t: Tiers):
    """(kind int8, capacity int64, alloc int64) per row, reference integer rules."""
    n = len(st.products)
    caps = np.asarray(t.hash_caps, np.int64)
    dsp = np.asarray(t.dense_spans, np.int64)
    prod = st.products
    kind = np.empty(n, np.int8)
    cap = np.zeros(n, np.int64)
    alloc = np.zeros(n, np.int64)
    if workflow == "upper":
        target = prod.astype(np.int64)
    else:
        target = np.ceil(np.asarray(pred, np.float64) * t.coef).astype(np.int64)
    target = np.maximum(target, 1)
    live = prod > 0
    span = st.spans()
    big = np.iinfo(np.int64).max
    hj = np.searchsorted(caps, target)
    hfit = hj < len(caps)
    efit = target <= t.enh_cap
    hrank = np.where(hfit, hj, np.where(efit, len(caps) - 1, big))
    is_enh = ~hfit & efit
    have_h = hfit | efit
    dj = np.searchsorted(dsp, span)
    dfit = (dj < len(dsp)) & live
    drank = np.where(dfit, dj, big)
    use_d = dfit & (~have_h | (drank < hrank) | ((drank == hrank) & ~is_enh))
    use_h = live & ~use_d & have_h
    use_f = live & ~use_d & ~use_h
    kind[use_h & ~is_enh] = KIND_HASH
    kind[use_h & is_enh] = KIND_ENH
    kind[use_d] = KIND_DENSE
    kind[use_f] = KIND_FB
    cap[use_h] = np.where(is_enh, t.enh_cap, caps[np.minimum(hj, len(caps) - 1)])[use_h]
    cap[use_d] = dsp[np.minimum(dj, len(dsp) - 1)][use_d]
    if workflow == "upper":
        esc = live & (prod < t.esc_max)
        kind[esc] = KIND_ESC
        cap[esc] = prod[esc]
        alloc[live] = prod[live]
    elif pred_kind == "exact":
        alloc[live] = np.asarray(pred, np.int64)[live]
        alloc[use_f] = prod[use_f]
    else:
        alloc[use_h] = cap[use_h]
        p2 = np.int64(1) << np.ceil(np.log2(target)).astype(np.int64)
        alloc[use_d] = np.minimum(cap[use_d], np.maximum(p2, caps[0])[use_d])
        alloc[use_f] = prod[use_f]
    kind[~live] = KIND_HASH
    cap[~live] = caps[0]
    alloc[~live] = 0
    return kind, cap, alloc


# ---------------------------------------------------------------------------
# L3 batch accumulators (accumulate.py:335-430)

def acc_hash(a, b, rows, cap, out_c, out_v, offs):
    """Hash / enhanced bins: counts, overflow at floor(0.8 cap), slot-order emission
    (accumulate.py:335-365)."""
    prow, pcol, pval = expand(a, b, rows)
    ur, uc, uv = reduce_cells(prow, pcol, pval, b.ncols)
    cnt = np.bincount(ur, minlength=len(rows)).astype(np.int64)
    ovf = cnt > (LOAD_LIMIT * cap).astype(np.int64)
    keep = ~ovf[ur]
    ur, uc, uv = ur[keep], uc[keep], uv[keep]
    tsize = np.int64(1) << np.int64(np.ceil(np.log2(np.maximum(cap, 2))))
    slot = (hash64(uc.astype(np.uint64)) & (tsize[ur] - 1).astype(np.uint64)).astype(np.int64)
    o = np.lexsort((uc, slot, ur))
    kept = np.where(ovf, 0, cnt)
    dst = ranges(offs, kept)
    out_c[dst] = uc[o].astype(np.int32)
    out_v[dst] = uv[o]
    return kept, ovf


def acc_esc(a, b, rows, out_c, out_v, offs):
    """Expand-sort-compact bin (accumulate.py:368-378)."""
    prow, pcol, pval = expand(a, b, rows)
    ur, uc, uv = reduce_cells(prow, pcol, pval, b.ncols)
    cnt = np.bincount(ur, minlength=len(rows)).astype(np.int64)
    dst = ranges(offs, cnt)
    out_c[dst] = uc.astype(np.int32)
    out_v[dst] = uv
    return cnt, np.zeros(len(rows), bool)


def acc_dense(a, b, rows, lo, width, alloc, out_c, out_v, offs, chunk=1 << 24):
    """Span-indexed scatter-add, chunked by total width (accumulate.py:381-430)."""
    n = len(rows)
    counts = np.zeros(n, np.int64)
    ovf = np.zeros(n, bool)
    i = 0
    while i < n:
        j, w = i, 0
        while j < n and (w == 0 or w + width[j] <= chunk):
            w += int(width[j])
            j += 1
        s = slice(i, j)
        seg = np.r_[0, np.cumsum(width[s])]
        prow, pcol, pval = expand(a, b, rows[s])
        pos = seg[prow] + (pcol - lo[s][prow])
        sums = np.bincount(pos, weights=pval, minlength=seg[-1])
        occ = np.flatnonzero(np.bincount(pos, minlength=seg[-1]))
        rof = np.searchsorted(seg, occ, side="right") - 1
        c = np.bincount(rof, minlength=j - i).astype(np.int64)
        o = c > alloc[s]
        keep = ~o[rof]
        occ, rof = occ[keep], rof[keep]
        kc = np.where(o, 0, c)
        dst = ranges(offs[s], kc)
        out_c[dst] = (occ - seg[rof] + lo[s][rof]).astype(np.int32)
        out_v[dst] = sums[occ]
        counts[s] = kc
        ovf[s] = o
        i = j
    return counts, ovf


# ---------------------------------------------------------------------------
# L4 orchestration (engine.py:136-368)

def spgemm(a, b, workflow: str = "auto", registers=None, tiers=None, coef=None,
           sample_ratio=SAMPLE_RATIO, sample_min=SAMPLE_MIN, sample_max=SAMPLE_MAX,
           seed: int = 0, workers: int = 1, keep_intermediates: bool = False, compute_errors: bool = False):
    """Restated ``engine.spgemm`` (engine.py:136-249).

    Returns (Csr C, report dict[, intermediates dict]).  ``workflow`` is one of
    auto / symbolic / estimate / upper (engine.py:47-51).
    """
    import time
    a, b = as_csr(a), as_csr(b)
    if a.ncols != b.nrows:
        raise ValueError(f"dimension mismatch: A is {a.nrows}x{a.ncols}, B is {b.nrows}x{b.ncols}")
    t = Tiers.of(tiers)
    t0 = time.perf_counter()
    st = row_stats(a, b)
    avg = st.total / a.nrows if a.nrows else 0.0
    t1 = time.perf_counter()
    regs_m = registers if registers is not None else choose_registers(st.er)
    regs = None
    cr = None
    if workflow == "symbolic":
        wf = "symbolic"
    elif workflow == "upper":
        wf = "upper"
    elif workflow == "auto" and avg < 64:
        wf = "upper"
    else:
        regs = b_sketches(b, P_OF_M[regs_m])
        srows = sample_rows(a.nrows, sample_ratio, sample_min, sample_max, seed)
        if a.nrows == 0:
            cr = (1.0, 1.0, 0.0)
        else:
            cr = cr_from_sample(st.products[srows], merged_estimates(a, regs, srows))
        wf = "estimate" if workflow == "estimate" else choose_workflow(avg, st.er, cr[0])
    t2 = time.perf_counter()
    if wf == "symbolic":
        pred, pk = exact_counts(a, b, st, t.dense_spans[-1]), "exact"
    elif wf == "estimate":
        pred, pk = estimate_all(a, regs), "estimated"
    else:
        pred, pk = st.products.copy(), "upper_bound"
    t3 = time.perf_counter()
    c = coef if coef is not None else (2.0 if regs_m == 32 else t.coef)
    t = Tiers(t.hash_caps, t.enh_cap, t.dense_spans, t.esc_max, c, t.bitmap_threshold)
    bitmap_query = cr is not None and max(1.0, cr[1] - 2.0 * cr[2]) >= t.bitmap_threshold
    kind, cap, alloc = plan(pred, pk, wf, st, t)

    # numeric phase into over-allocated slabs (engine.py:252-309)
    aptr = np.zeros(a.nrows + 1, np.int64)
    np.cumsum(alloc, out=aptr[1:])
    out_c = np.empty(int(aptr[-1]), np.int32)
    out_v = np.empty(int(aptr[-1]), np.float64)
    counts = np.zeros(a.nrows, np.int64)
    ovf = np.zeros(a.nrows, bool)
    spans = st.spans()

    def chunk(rows):
        k = kind[rows]
        hl = rows[((k == KIND_HASH) | (k == KIND_ENH)) & (st.products[rows] > 0)]
        if len(hl):
            counts[hl], ovf[hl] = acc_hash(a, b, hl, cap[hl], out_c, out_v, aptr[hl])
        es = rows[k == KIND_ESC]
        if len(es):
            counts[es], _ = acc_esc(a, b, es, out_c, out_v, aptr[es])
        dn = rows[k == KIND_DENSE]
        if len(dn):
            counts[dn], ovf[dn] = acc_dense(a, b, dn, st.span_lo[dn], spans[dn], alloc[dn],
                                            out_c, out_v, aptr[dn])

    parts = [p for p in np.array_split(np.arange(a.nrows, dtype=np.int64),
                                       max(1, min(workers, max(a.nrows, 1)))) if len(p)]
    if workers > 1 and len(parts) > 1:
        with ThreadPoolExecutor(max_workers=workers) as ex:
            list(ex.map(chunk, parts))
    else:
        for p in parts:
            chunk(p)
    t4 = time.perf_counter()

    # fallback phase: full-width dense rerun (engine.py:312-328)
    fb = np.flatnonzero(ovf | ((kind == KIND_FB) & (st.products > 0)))
    fptr = np.zeros(len(fb) + 1, np.int64)
    np.cumsum(st.products[fb], out=fptr[1:])
    fc = np.empty(int(fptr[-1]), np.int32)
    fv = np.empty(int(fptr[-1]), np.float64)
    if len(fb):
        counts[fb], _ = acc_dense(a, b, fb, np.zeros(len(fb), np.int64),
                                  np.full(len(fb), b.ncols, np.int64), st.products[fb],
                                  fc, fv, fptr[:-1])
    t5 = time.perf_counter()

    # sort hash rows (engine.py:331-343) then compact (engine.py:346-368)
    isfb = np.zeros(a.nrows, bool)
    isfb[fb] = True
    srt = np.flatnonzero(((kind == KIND_HASH) | (kind == KIND_ENH)) & (counts > 0) & ~isfb)
    if len(srt):
        src = ranges(aptr[srt], counts[srt])
        seq = np.repeat(np.arange(len(srt), dtype=np.int64), counts[srt])
        o = np.argsort(seq * np.int64(b.ncols) + out_c[src], kind="stable")
        out_c[src] = out_c[src][o]
        out_v[src] = out_v[src][o]
    rp = np.zeros(a.nrows + 1, np.int64)
    np.cumsum(counts, out=rp[1:])
    cc = np.empty(int(rp[-1]), np.int32)
    cv = np.empty(int(rp[-1]), np.float64)
    main = np.flatnonzero(~isfb & (counts > 0))
    if len(main):
        src = ranges(aptr[main], counts[main])
        dst = ranges(rp[main], counts[main])
        cc[dst], cv[dst] = out_c[src], out_v[src]
    if len(fb):
        src = ranges(fptr[:-1], counts[fb])
        dst = ranges(rp[fb], counts[fb])
        cc[dst], cv[dst] = fc[src], fv[src]
    t6 = time.perf_counter()
    nnz = int(rp[-1])
    report = dict(workflow=wf, registers=int(regs_m), er=st.er,
                  cr_hat=None if cr is None else cr[0],
                  cr_true=(st.total / nnz) if nnz else None,
                  analysis_ms=(t1 - t0) * 1e3, sketch_ms=(t2 - t1) * 1e3 if regs is not None else 0.0,
                  predict_ms=(t3 - t2) * 1e3, numeric_ms=(t4 - t3) * 1e3,
                  fallback_ms=(t5 - t4) * 1e3, compact_ms=(t6 - t5) * 1e3,
                  total_ms=(time.perf_counter() - t0) * 1e3,
                  overflow_row_count=int(len(fb)), nnz_c=nnz, total_products=st.total,
                  bitmap_query=bool(bitmap_query))
    # estimation error of the per-row predictions (engine.py:218-226)
    report["est_mean_rel_err"] = report["est_std_rel_err"] = None
    if compute_errors and pk == "estimated":
        truth = np.diff(rp)
        live = truth > 0
        if live.any():
            rel = np.abs(pred[live] - truth[live]) / truth[live]
            report["est_mean_rel_err"], report["est_std_rel_err"] = float(rel.mean()), float(rel.std())
        else:
            report["est_mean_rel_err"] = report["est_std_rel_err"] = 0.0
    C = Csr(a.nrows, b.ncols, rp, cc, cv)
    if keep_intermediates:
        return C, report, dict(stats=st, regs=regs, pred=pred, pred_kind=pk, kind=kind,
                               cap=cap, alloc=alloc, overflow=ovf, fb_rows=fb, counts=counts)
    return C, report


def dict_spgemm(a, b) -> Csr:
    """Slow sequential truth: per-row dict accumulation (oracle.py:16-43)."""
    a, b = as_csr(a), as_csr(b)
    rp, cc, cv = [0], [], []
    for i in range(a.nrows):
        acc: dict = {}
        for t in range(a.row_ptr[i], a.row_ptr[i + 1]):
            k, av = int(a.col_idx[t]), float(a.values[t])
            for u in range(b.row_ptr[k], b.row_ptr[k + 1]):
                c = int(b.col_idx[u])
                acc[c] = acc.get(c, 0.0) + av * float(b.values[u])
        for c in sorted(acc):
            cc.append(c)
            cv.append(acc[c])
        rp.append(len(cc))
    return Csr(a.nrows, b.ncols, rp, cc, cv)


def default_workers() -> int:
    return os.cpu_count() or 1
