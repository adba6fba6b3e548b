"""Drop-in ``spgemm(a, b, cfg, deadline) -> (C, RunReport)`` on one B200.

Same stage sequence, decisions and report as the reference engine
(``engine.py:136-249``): analysis -> [sketch + sampled CR] -> size prediction
(symbolic | HLL estimate | upper bound) -> binning -> numeric -> fallback ->
sort + compact.  Every stage runs as sm_100a kernels behind the C ABI
(``include/sgb200.h``) through ctypes; torch is used only to allocate device
buffers and to move bytes.  The only host arithmetic is what the reference's
host does on scalars: workflow choice, the seeded sample-row draw and the
10k-row sampled-CR reduction.

Memory layout differences (results are identical):
  * with an EXACT prediction (symbolic workflow) C is allocated once at its
    final size and every kernel writes its rows in place, sorted: no staging
    slab, no compaction copy;
  * otherwise the main staging slab holds only rows that the numeric phase
    accumulates (planned-FALLBACK rows are never staged, as their staged
    region is unused in the reference too); fallback rows are counted first,
    then written straight into C.
"""

from __future__ import annotations

import ctypes
import threading
import time
from dataclasses import dataclass, replace

import numpy as np
import torch
from torch.cuda import nvtx as _nvtx

from . import _lib
from .config import (DEFAULT_SAMPLE_MAX, DEFAULT_SAMPLE_MIN, PRECISION_FOR, EngineConfig,
                     PlanKind, ResourceLimitError, RunReport, TierConfig, WorkflowKind,
                     WorkflowOverride, DeadlineExceeded, select_registers, select_workflow)
from .csr import CsrMatrix
from .device import DeviceCsr, to_device, ptr

ALPHA = {32: 0.697, 64: 0.709, 128: 0.7213 / (1 + 1.079 / 128)}
_PRED_CODE = {"exact": 0, "estimated": 1, "upper_bound": 2}


def _check_deadline(deadline):
    if deadline is not None and time.perf_counter() > deadline:
        raise DeadlineExceeded("run exceeded its deadline")


def lin_table(m: int) -> np.ndarray:
    """m*ln(m/z) for z = 0..m (z = 0 unused), computed with the reference's
    own array expression (hll.py:84) so the device linear-counting branch is
    bit-identical."""
    z = np.arange(0, m + 1)
    with np.errstate(divide="ignore"):
        t = np.where(z > 0, m * np.log(m / np.maximum(z, 1)), 0.0)
    return t.astype(np.float64)


def sample_rows(nrows: int, ratio: float, min_n: int, max_n: int, seed: int) -> np.ndarray:
    """Seeded sample of distinct rows, identical draw to analysis.py:182-190."""
    n = int(np.clip(round(ratio * nrows), min(min_n, nrows), min(max_n, nrows)))
    if n >= nrows:
        return np.arange(nrows, dtype=np.int64)
    rng = np.random.default_rng(seed)
    return np.sort(rng.choice(nrows, size=n, replace=False)).astype(np.int64)


_SAMPLE_CACHE: dict = {}


def sample_rows_device(device, nrows, ratio, min_n, max_n, seed):
    """sample_rows uploaded once per (device, draw) and reused across calls."""
    key = (str(device), nrows, ratio, min_n, max_n, seed)
    t = _SAMPLE_CACHE.get(key)
    if t is None:
        if len(_SAMPLE_CACHE) >= 16:
            _SAMPLE_CACHE.pop(next(iter(_SAMPLE_CACHE)))
        t = torch.from_numpy(sample_rows(nrows, ratio, min_n, max_n, seed)).to(device)
        _SAMPLE_CACHE[key] = t
    return t


def tiers_struct(t: TierConfig) -> _lib.SgTiers:
    s = _lib.SgTiers()
    s.n_hash = len(t.hash_capacities)
    s.n_dense = len(t.dense_spans)
    for i, c in enumerate(t.hash_capacities):
        s.hash_caps[i] = int(c)
    for i, c in enumerate(t.dense_spans):
        s.dense_spans[i] = int(c)
    s.enh_cap = int(t.enhanced_hash_capacity)
    s.esc_max = int(t.esc_max_products)
    s.coef = float(t.expansion_coef)
    return s


class _Ctx:
    """Per-call device context: stream, workspace, timing."""

    def __init__(self, device, stream):
        self.device = device
        self.stream = stream
        self.sp = stream.cuda_stream
        self.ws = None
        self.ws_bytes = 0
        self._old_ws = []
        self.arena_taken = False

    def workspace(self, m):
        """Scratch for the stage calls.  A grown workspace never frees the
        previous one during the call: a caller may still hold its pointer."""
        need = int(_lib.load().sg_workspace_bytes(int(m)))
        if self.ws is None or self.ws_bytes < need:
            if self.ws is not None:
                self._old_ws.append(self.ws)
            self.ws = torch.empty(need, dtype=torch.uint8, device=self.device)
            self.ws_bytes = need
        return ptr(self.ws), self.ws_bytes

    def empty(self, n, dtype):
        try:
            return torch.empty(int(n), dtype=dtype, device=self.device)
        except torch.OutOfMemoryError as exc:
            # buffers kept from earlier calls give way first
            if _ARENA.drop_if_idle(self.device):
                torch.cuda.empty_cache()
                try:
                    return torch.empty(int(n), dtype=dtype, device=self.device)
                except torch.OutOfMemoryError:
                    pass
            raise ResourceLimitError(
                f"device allocation of {int(n)} x {dtype} failed; the symbolic workflow "
                "(workflow='symbolic') stages exact-sized rows") from exc

    def sync(self):
        self.stream.synchronize()


def row_stats(ctx: _Ctx, A: DeviceCsr, B: DeviceCsr):
    m = A.nrows
    products = ctx.empty(m, torch.int64)
    lo = ctx.empty(m, torch.int64)
    hi = ctx.empty(m, torch.int64)
    totals = ctx.empty(2, torch.int64)
    _lib.call("sg_row_stats", m, B.ncols, ptr(A.row_ptr), ptr(A.col_idx), ptr(B.row_ptr),
              ptr(B.col_idx), ptr(products), ptr(lo), ptr(hi), ptr(totals), ctx.sp)
    return products, lo, hi, totals


def hll_build(ctx: _Ctx, B: DeviceCsr, p: int):
    regs = ctx.empty(B.nrows * (1 << p), torch.uint8)
    _lib.call("sg_hll_build", B.nrows, ptr(B.row_ptr), ptr(B.col_idx), p, ptr(regs), ctx.sp)
    return regs


def hll_estimate(ctx: _Ctx, A: DeviceCsr, regs, p: int, rows=None):
    m = 1 << p
    key = ("lin", str(ctx.device), m)
    lin = _SAMPLE_CACHE.get(key)
    if lin is None:
        lin = _SAMPLE_CACHE[key] = torch.from_numpy(lin_table(m)).to(ctx.device)
    nsel = A.nrows if rows is None else int(rows.numel())
    est = ctx.empty(nsel, torch.float64)
    _lib.call("sg_hll_estimate", nsel, None if rows is None else ptr(rows), ptr(A.row_ptr),
              ptr(A.col_idx), ptr(regs), p, ptr(lin), (ALPHA[m] * m) * m, ptr(est), ctx.sp)
    return est


def scan(ctx: _Ctx, x):
    n = int(x.numel())
    out = ctx.empty(n + 1, torch.int64)
    ws, wsb = ctx.workspace(max(n, 1))
    _lib.call("sg_scan", n, ptr(x), ptr(out), ws, wsb, ctx.sp)
    return out


class Windows:
    """Numeric window tables of the long rows (sg_windows_t, include/sgb200.h)."""

    def __init__(self, off, wins, nwin, bm_off, bm_save, pre_save, total):
        self.off, self.wins, self.nwin, self.bm_off, self.total = off, wins, nwin, bm_off, total
        self.bm_save, self.pre_save = bm_save, pre_save
        self.btile_off = self.btile = None
        self._struct = None

    def struct(self):
        s = _lib.SgWindows()
        s.win_off, s.wins, s.nwin = ptr(self.off), ptr(self.wins), ptr(self.nwin)
        s.bm_off = ptr(self.bm_off) if self.bm_save is not None else None
        s.bm_save = ptr(self.bm_save) if self.bm_save is not None else None
        s.pre_save = None  # ranks live in the 16-byte saved words
        s.btile_off = ptr(self.btile_off)
        s.btile = ptr(self.btile)
        self._struct = s  # keep alive for the call
        return s

    def drop_bitmaps(self):
        """Release the saved key bitmaps (the window pass then rebuilds keys)."""
        self.bm_save = None
        self.pre_save = None


# symbolic workflow: rows with at most this many products are staged, not counted
SHORT_ROW_PRODUCTS = 1024
SHORT_ROW_MAX_CR = 1.25
# staged short rows of at most this many products use the register
# expand-sort-compress accumulator (0 = hash tables)
SHORT_ROW_ESCR = 512

# saved key bitmaps may use at most this share of the free device memory
BITMAP_SAVE_SHARE = 0.35


def windows(ctx: _Ctx, m, products, lo, hi, select, c_bytes: int = 0) -> Windows:
    """Window tables of the long rows; their key bitmaps are saved (16 B per
    64 columns) only when they fit next to `c_bytes` -- the C arrays still to
    be allocated -- so that C never has to evict them (an eviction costs the
    bitmap pass and, call after call, re-mapping tens of GB)."""
    off = ctx.empty(m + 1, torch.int64)
    bm_off = ctx.empty(m + 1, torch.int64)
    totals = (ctypes.c_int64 * 2)()
    ws, wsb = ctx.workspace(max(m, 1))
    _lib.call("sg_window_capacity", m, ptr(products), ptr(lo), ptr(hi), ptr(select), ptr(off), ptr(bm_off),
              ctypes.cast(totals, ctypes.c_void_p), ws, wsb, ctx.sp)
    total, words = int(totals[0]), int(totals[1])
    wins = torch.full((max(2 * total, 2),), -1, dtype=torch.int32, device=ctx.device)
    nwin = torch.zeros(max(m, 1), dtype=torch.int32, device=ctx.device)
    bm_save = pre_save = None
    if total and words:
        # free = device memory minus what torch has handed out (cached blocks
        # and the arena's own buffers count as free); torch's counters, not
        # cudaMemGetInfo, which costs milliseconds under expandable segments
        free = _device_total(ctx.device) - torch.cuda.memory_allocated(ctx.device)
        free += _ARENA.held_bytes(ctx.device)
        if 16 * words <= BITMAP_SAVE_SHARE * free and 16 * words + c_bytes <= 0.96 * free:
            bm_save = _ARENA.take(ctx, words)
    return Windows(off, wins, nwin, bm_off, bm_save, pre_save, total)


_TOTAL: dict = {}


def _device_total(device) -> int:
    """Device memory usable by this process (total minus a 4 GB reserve for
    the context and other processes), cached."""
    key = str(device)
    if key not in _TOTAL:
        free, total = torch.cuda.mem_get_info(device)
        _TOTAL[key] = max(0, min(total - (4 << 30), free + torch.cuda.memory_reserved(device)))
    return _TOTAL[key]


class _BitmapArena:
    """Saved-bitmap buffers kept across calls, per device.  Allocating them
    afresh (tens of GB at R-MAT-20) costs from 0.5 to 60 ms per call when the
    caching allocator has to map new memory; reusing them removes that jitter.
    A call holds the device's buffers until it returns; a concurrent call on
    the same device allocates its own (and does not keep them)."""

    HEADROOM = 1.02

    def __init__(self):
        self.lock = threading.Lock()
        self.bufs: dict = {}
        self.busy: set = set()

    def held_bytes(self, device) -> int:
        with self.lock:
            b = self.bufs.get(str(device))
        return 0 if b is None else b.numel() * 8

    def take(self, ctx, words):
        key = str(ctx.device)
        with self.lock:
            shared = key in self.busy
            cur = None if shared else self.bufs.get(key)
            if not shared:
                self.busy.add(key)
                if cur is not None and cur.numel() < 2 * words:
                    del self.bufs[key]  # too small: replace
                    cur = None
        if cur is None:
            n = words if shared else int(words * self.HEADROOM)
            try:
                cur = torch.empty(2 * n, dtype=torch.int64, device=ctx.device)  # 16 B per word
            except torch.OutOfMemoryError:
                try:
                    cur = torch.empty(2 * words, dtype=torch.int64, device=ctx.device)
                except torch.OutOfMemoryError:
                    if not shared:
                        self.release(ctx.device)
                    return None
            if not shared:
                with self.lock:
                    self.bufs[key] = cur
        if not shared:
            ctx.arena_taken = True
        return cur[:2 * words]

    def release(self, device):
        with self.lock:
            self.busy.discard(str(device))

    def drop(self, device):
        """Free the device's buffers (C needs the memory)."""
        with self.lock:
            self.bufs.pop(str(device), None)

    def drop_if_idle(self, device) -> bool:
        with self.lock:
            key = str(device)
            if key in self.busy or key not in self.bufs:
                return False
            del self.bufs[key]
            return True


_ARENA = _BitmapArena()


def release_bitmap_arena(device=None):
    """Free the saved-bitmap buffers kept across calls."""
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    _ARENA.drop(dev)


# the B tile index (sg_btile_plan) may use at most this many bytes
BTILE_BUDGET = 2 << 30


def btile(ctx: _Ctx, B: DeviceCsr, win: Windows):
    """Build the B tile index for the window pass (rows as long as fit)."""
    k = B.nrows
    scan_ = ctx.empty(k + 1, torch.int64)
    totals = (ctypes.c_int64 * 2)()
    ws, wsb = ctx.workspace(max(k, 1))
    _lib.call("sg_btile_plan", k, B.ncols, ptr(B.row_ptr), BTILE_BUDGET, ptr(scan_),
              ctypes.cast(totals, ctypes.c_void_p), ws, wsb, ctx.sp)
    if totals[0] <= 0:
        return
    off = ctx.empty(max(k, 1), torch.int64)
    tbl = ctx.empty(int(totals[0]), torch.int32)
    _lib.call("sg_btile_build", k, B.ncols, ptr(B.row_ptr), ptr(B.col_idx), ptr(scan_), ptr(off), ptr(tbl), ctx.sp)
    win.btile_off, win.btile = off, tbl


def alloc_c(ctx: _Ctx, nnz, dtype, win):
    """C's column / value arrays; if they do not fit next to the saved key
    bitmaps, the bitmaps are released (the window pass rebuilds keys)."""
    try:
        return ctx.empty(nnz, torch.int32), ctx.empty(nnz, dtype)
    except ResourceLimitError:
        if win is None or win.bm_save is None:
            raise
        win.drop_bitmaps()
        _ARENA.drop(ctx.device)
        torch.cuda.empty_cache()
        return ctx.empty(nnz, torch.int32), ctx.empty(nnz, dtype)


def select_fallback(ctx: _Ctx, m, kind, products, overflow, exclude):
    """Fallback rows (engine.py:202-203), optionally minus rows with windows."""
    rows = ctx.empty(max(m, 1), torch.int64)
    n = ctypes_int64()
    if m:
        ws, wsb = ctx.workspace(m)
        _lib.call("sg_select_fallback", m, ptr(kind), ptr(products), ptr(overflow), ptr(exclude), ptr(rows),
                  n, ws, wsb, ctx.sp)
    n = int(n.value)
    return rows[:n], n


@dataclass(frozen=True)
class Decision:
    """Workflow decision of one whole product (engine.py:147-174), made once
    on the root rank and applied by every shard (EngineConfig.decision)."""

    workflow: str          # WorkflowKind value
    registers: int
    er: float
    cr: tuple | None       # (cr_hat, mean row CR, std row CR) of the sample
    total_products: int


def decide(a, b, cfg: EngineConfig | None = None, device=None) -> Decision:
    """Analysis + sketch/sample stages of spgemm on the whole operands: the
    same row statistics, seeded sample and selection rules as the engine."""
    cfg = cfg or EngineConfig()
    device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    stream = torch.cuda.current_stream(device)
    with torch.cuda.device(device), torch.cuda.stream(stream):
        ctx = _Ctx(device, stream)
        A = to_device(a, device)
        B = A if b is a else to_device(b, device)
        products, _, _, totals = row_stats(ctx, A, B)
        total = int(totals.cpu()[0])
        m = A.nrows
        er = total / A.nnz if A.nnz else 0.0
        avg = total / m if m else 0.0
        registers = cfg.registers if cfg.registers is not None else select_registers(er)
        W = cfg.workflow
        cr = None
        if W is WorkflowOverride.FORCE_SYMBOLIC:
            wf = WorkflowKind.SYMBOLIC
        elif W is WorkflowOverride.FORCE_UPPER_BOUND or (W is WorkflowOverride.AUTO and avg < 64):
            wf = WorkflowKind.UPPER_BOUND
        else:
            p = PRECISION_FOR[registers]
            regs = hll_build(ctx, B, p)
            if m == 0:
                cr = (1.0, 1.0, 0.0)
            else:
                rows_d = sample_rows_device(device, m, cfg.sample_ratio, cfg.sample_min, cfg.sample_max, cfg.seed)
                est = hll_estimate(ctx, A, regs, p, rows_d)
                both = torch.stack((est, products[rows_d].to(torch.float64))).cpu().numpy()
                est_s, prods = both[0], both[1]
                row_cr = np.where(prods > 0, prods / np.maximum(est_s, 1.0), 1.0)
                cr = (float(prods.sum() / max(1.0, est_s.sum())), float(row_cr.mean()), float(row_cr.std()))
            wf = WorkflowKind.HLL_ESTIMATION if W is WorkflowOverride.FORCE_ESTIMATE else select_workflow(avg, er, cr[0])
        return Decision(wf.value, registers, er, cr, total)


def _dtype_code(v: torch.Tensor) -> int:
    return 0 if v.dtype == torch.float64 else 1


def spgemm(a, b, cfg: EngineConfig | None = None, deadline: float | None = None):
    """Multiply two CSR matrices on the GPU; returns (C, RunReport).

    ``a`` / ``b`` are host ``CsrMatrix`` (any object with nrows, ncols,
    row_ptr, col_idx, values) or ``DeviceCsr``.  C is a host ``CsrMatrix``
    unless ``cfg.return_device``.  Raises ValueError on a dimension mismatch
    (engine.py:145-146), ResourceLimitError when the reference staging rule
    exceeds ``staging_limit_bytes`` (engine.py:259-271), DeadlineExceeded
    between stages (engine.py:131-133).
    """
    cfg = cfg or EngineConfig()
    if a.ncols != b.nrows:
        raise ValueError(f"dimension mismatch: A is {a.nrows}x{a.ncols}, B is {b.nrows}x{b.ncols}")
    _lib.load()
    if not torch.cuda.is_available():
        from .config import CudaLibraryError
        raise CudaLibraryError("no CUDA device: the B200 path has no CPU fallback")
    device = torch.device("cuda", cfg.device if cfg.device is not None else torch.cuda.current_device())
    stream = cfg.stream if cfg.stream is not None else torch.cuda.current_stream(device)
    with torch.cuda.device(device), torch.cuda.stream(stream):
        ctx = _Ctx(device, stream)
        try:
            return _spgemm(a, b, cfg, deadline, ctx)
        finally:
            if ctx.arena_taken:
                # the call's work is complete (it ends with a stream sync on
                # success); on an error, wait before the buffers are reused
                ctx.sync()
                _ARENA.release(device)


def _spgemm(a, b, cfg, deadline, ctx: _Ctx):
    if cfg.dtype is not None:
        dtype = torch.float64 if cfg.dtype == "f64" else torch.float32
    elif isinstance(a, DeviceCsr):
        dtype = a.values.dtype
    else:
        dtype = torch.float32 if np.asarray(a.values).dtype == np.float32 else torch.float64
    kms = {}
    t0 = time.perf_counter()
    A = to_device(a, ctx.device, dtype)
    B = A if b is a else to_device(b, ctx.device, dtype)
    m, n = A.nrows, B.ncols
    kms["h2d"] = (time.perf_counter() - t0) * 1e3

    # ---- analysis (analysis.py:96-128)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(7)]
    ev[0].record(ctx.stream)
    _nvtx.range_push("spgemm:analysis")  # reference stage (engine.py:147-216)
    t0 = time.perf_counter()
    products, span_lo, span_hi, totals = row_stats(ctx, A, B)
    tot = totals.cpu().numpy()
    total_products = int(tot[0])
    nnz_a = A.nnz
    er = total_products / nnz_a if nnz_a else 0.0
    avg = total_products / m if m else 0.0
    ev[1].record(ctx.stream)
    _nvtx.range_pop()
    _nvtx.range_push("spgemm:sketch")  # reference stage (engine.py:147-216)
    _check_deadline(deadline)

    # ---- sketch + sampled CR (engine.py:157-174)
    registers = cfg.registers if cfg.registers is not None else select_registers(er)
    regs = None
    cr = None
    W = cfg.workflow
    dec = cfg.decision
    if dec is not None:
        # decided once for the whole product on the root rank (shard.py)
        registers, er = dec.registers, dec.er
        kind_wf = WorkflowKind(dec.workflow)
        cr = dec.cr
        p = PRECISION_FOR[registers]
        if kind_wf is WorkflowKind.HLL_ESTIMATION:
            regs = hll_build(ctx, B, p)
    elif W is WorkflowOverride.FORCE_SYMBOLIC:
        p = PRECISION_FOR[registers]
        kind_wf = WorkflowKind.SYMBOLIC
    elif W is WorkflowOverride.FORCE_UPPER_BOUND:
        p = PRECISION_FOR[registers]
        kind_wf = WorkflowKind.UPPER_BOUND
    elif W is WorkflowOverride.AUTO and avg < 64:
        p = PRECISION_FOR[registers]
        kind_wf = WorkflowKind.UPPER_BOUND
    else:
        p = PRECISION_FOR[registers]
        regs = hll_build(ctx, B, p)
        if m == 0:
            cr = (1.0, 1.0, 0.0)
        else:
            rows_d = sample_rows_device(ctx.device, m, cfg.sample_ratio, cfg.sample_min, cfg.sample_max,
                                        cfg.seed)
            est_d = hll_estimate(ctx, A, regs, p, rows_d)
            both = torch.stack((est_d, products[rows_d].to(torch.float64))).cpu().numpy()
            est_s, prods = both[0], both[1]
            cr_hat = float(prods.sum() / max(1.0, est_s.sum()))
            row_cr = np.where(prods > 0, prods / np.maximum(est_s, 1.0), 1.0)
            cr = (cr_hat, float(row_cr.mean()), float(row_cr.std()))
        if W is WorkflowOverride.FORCE_ESTIMATE:
            kind_wf = WorkflowKind.HLL_ESTIMATION
        else:
            kind_wf = select_workflow(avg, er, cr[0])
    ev[2].record(ctx.stream)
    _nvtx.range_pop()
    _nvtx.range_push("spgemm:predict")  # reference stage (engine.py:147-216)
    _check_deadline(deadline)

    # ---- size prediction (predict.py)
    ws, wsb = ctx.workspace(max(m, 1))
    win = None
    short = None       # symbolic: rows staged instead of counted
    pred_plan = None
    if kind_wf is WorkflowKind.SYMBOLIC:
        pred = ctx.empty(m, torch.int64)
        # C's size for the bitmap budget: products / sampled CR, else the
        # bound sum(min(products, span)) per row
        vb = 4 + (8 if dtype == torch.float64 else 4)
        if cr is not None:
            c_est = int(total_products / max(1.0, cr[0]) * 1.05)
        else:
            c_est = int(torch.minimum(products, span_hi - span_lo + 1).clamp(min=0).sum().item()) if m else 0
        win = windows(ctx, m, products, span_lo, span_hi, None, vb * c_est)
        # assisted symbolic binning with the conservative
        # sampled CR (predict.py:111-118) when the sample was taken
        assist = 1.0 if (cr is None or not cfg.assisted_symbolic) else max(1.0, cr[1] - 2.0 * cr[2])
        # short rows (<= 1024 products) skip the count pass and are accumulated
        # once into a staging slab sized by their products (the reference's
        # staging rule is checked on exact counts, so not with a staging limit)
        # -- only when the sampled compression ratio says products ~ outputs
        # (otherwise the product-sized tables cost more than the count pass)
        short_max = SHORT_ROW_PRODUCTS if (cfg.stage_short_rows and cfg.staging_limit_bytes is None
                                           and cr is not None and cr[1] <= SHORT_ROW_MAX_CR) else 0
        _lib.call("sg_symbolic", m, n, ptr(A.row_ptr), ptr(A.col_idx), ptr(B.row_ptr), ptr(B.col_idx),
                  ptr(products), ptr(span_lo), ptr(span_hi), ptr(pred), win.struct(), assist, short_max,
                  ws, wsb, ctx.sp)
        pred_kind = "exact"
        if short_max and m:
            staged = pred == -2
            if bool(staged.any()):
                short = staged
                pred_plan = torch.where(short, products, pred)
    elif kind_wf is WorkflowKind.HLL_ESTIMATION:
        pred = hll_estimate(ctx, A, regs, p)
        pred_kind = "estimated"
    else:
        pred = products
        pred_kind = "upper_bound"
    ev[3].record(ctx.stream)
    _nvtx.range_pop()
    _nvtx.range_push("spgemm:numeric")  # reference stage (engine.py:147-216)
    _check_deadline(deadline)

    # ---- binning (accumulate.plan_rows) + numeric phase (engine._numeric_phase)
    coef = cfg.coef
    if coef is None:
        coef = 2.0 if registers == 32 else cfg.tiers.expansion_coef
    tiers = replace(cfg.tiers, expansion_coef=coef)
    bitmap_query = cr is not None and max(1.0, cr[1] - 2.0 * cr[2]) >= tiers.bitmap_query_threshold
    kind = ctx.empty(m, torch.int8)
    cap = ctx.empty(m, torch.int64)
    alloc = ctx.empty(m, torch.int64)
    ts = tiers_struct(tiers)
    if pred_plan is None:
        pred_plan = pred
    _lib.call("sg_plan", m, _PRED_CODE[pred_kind], ptr(pred_plan), ptr(products), ptr(span_lo), ptr(span_hi),
              ts, ptr(kind), ptr(cap), ptr(alloc), ctx.sp)
    staging_bytes = 0
    if cfg.staging_limit_bytes is not None and m:
        staging_bytes = int(alloc.sum().item()) * 12  # engine.py:259 rule
    if cfg.staging_limit_bytes is not None and staging_bytes > cfg.staging_limit_bytes:
        raise ResourceLimitError(
            f"staged output needs {staging_bytes} bytes, over the {cfg.staging_limit_bytes} byte "
            "limit; the symbolic workflow (workflow='symbolic') stages exact-sized rows")
    counts = ctx.empty(m, torch.int64)
    overflow = torch.zeros(m, dtype=torch.uint8, device=ctx.device)
    exact = pred_kind == "exact"
    dcode = _dtype_code(A.values)
    Aargs = (ptr(A.row_ptr), ptr(A.col_idx), ptr(A.values), ptr(B.row_ptr), ptr(B.col_idx), ptr(B.values))
    st_off = st_col = st_val = counts_s = short_fb = None
    if exact and short is not None:
        # short rows: one numeric pass into a slab at their product offsets;
        # their counts complete the exact row sizes.  The staging pass uses
        # its own plan (hash kind, table of at least 1.25 x products slots:
        # the 0.8 load limit can never trip, whatever the tiers or coef), not
        # the reference plan, which is recomputed below from the exact counts.
        s_kind = torch.full_like(kind, int(PlanKind.HASH))
        s_cap = torch.clamp(products + (products + 3) // 4 + 1, min=1)
        st_off = scan(ctx, torch.where(short, products, torch.zeros_like(products)))
        st_total = int(st_off[-1].item())
        st_col, st_val = ctx.empty(st_total, torch.int32), ctx.empty(st_total, dtype)
        counts_s = ctx.empty(m, torch.int64)
        s_ovf = torch.zeros(m, dtype=torch.uint8, device=ctx.device)
        _lib.call("sg_numeric", m, n, dcode, *Aargs, ptr(s_kind), ptr(s_cap), ptr(products),
                  ptr(products), ptr(span_lo), ptr(span_hi), ptr(st_off), ptr(st_col), ptr(st_val),
                  ptr(counts_s), ptr(s_ovf), ptr((~short).to(torch.int32)), None, SHORT_ROW_ESCR,
                  ws, wsb, ctx.sp)
        del s_kind, s_cap
        if bool(s_ovf[short].any()):  # cannot happen: slots hold every product
            raise RuntimeError("internal: a staged short row overflowed its product-sized slot")
        pred = torch.where(short, counts_s, pred)
        # the reference plan (accumulate.py:104-181) on the exact counts of
        # every row; a staged row the reference would overflow (count over
        # its tier limit) or plan as FALLBACK is flagged so the report counts
        # it (engine.py:202-203, 242) -- its values are already staged
        _lib.call("sg_plan", m, _PRED_CODE[pred_kind], ptr(pred), ptr(products), ptr(span_lo), ptr(span_hi),
                  ts, ptr(kind), ptr(cap), ptr(alloc), ctx.sp)
        lim = torch.where((kind == int(PlanKind.HASH)) | (kind == int(PlanKind.ENHANCED_HASH)),
                          (cap.to(torch.float64) * 0.8).floor().to(torch.int64),
                          torch.where(kind == int(PlanKind.DENSE), alloc, torch.full_like(alloc, 1 << 62)))
        s_over = short & ((kind == int(PlanKind.FALLBACK)) | (counts_s > lim))
        overflow |= s_over.to(torch.uint8)
        short_fb = s_over
    if exact:
        row_ptr = scan(ctx, pred)
        nnz_c = int(row_ptr[-1].item()) if m else 0
        out_col, out_val = alloc_c(ctx, nnz_c, dtype, win)
        out_off = row_ptr
    else:
        main_alloc = torch.where(kind == int(PlanKind.FALLBACK), torch.zeros_like(alloc), alloc)
        out_off = scan(ctx, main_alloc)
        slab = int(out_off[-1].item()) if m else 0
        out_col = ctx.empty(slab, torch.int32)
        out_val = ctx.empty(slab, dtype)
    if m:
        skip = win.nwin if win else None
        ovf = overflow
        if short is not None:
            skip = ((win.nwin[:m] > 0) | short).to(torch.int32)
            ovf = torch.zeros(m, dtype=torch.uint8, device=ctx.device)
        _lib.call("sg_numeric", m, n, dcode, *Aargs, ptr(kind), ptr(cap), ptr(alloc),
                  ptr(products), ptr(span_lo), ptr(span_hi), ptr(out_off), ptr(out_col), ptr(out_val),
                  ptr(counts), ptr(ovf), ptr(skip), ptr(pred) if exact else None, 0, ws, wsb, ctx.sp)
        if short is not None:
            overflow |= ovf
    ev[4].record(ctx.stream)
    _nvtx.range_pop()
    _nvtx.range_push("spgemm:fallback")  # reference stage (engine.py:147-216)
    _check_deadline(deadline)

    # ---- fallback (engine._fallback_phase): overflow | planned FALLBACK rows
    fb_rows, n_fb = select_fallback(ctx, m, kind, products, overflow, None)
    fargs = (*Aargs, ptr(products), ptr(span_lo), ptr(span_hi))
    if exact:
        C_col, C_val = out_col, out_val
    elif not n_fb:
        # no fallback rows: the numeric counts are final (no windows)
        row_ptr = scan(ctx, counts)
        nnz_c = int(row_ptr[-1].item()) if m else 0
        C_col, C_val = alloc_c(ctx, nnz_c, dtype, None)
    else:
        # count the fallback rows (recording windows for long ones), size C
        sel = torch.zeros(m, dtype=torch.uint8, device=ctx.device)
        sel[fb_rows] = 1
        # C's size: the non-fallback rows' exact counts plus the fallback
        # rows' predictions (estimates / upper bounds), 5% margin
        vb = 4 + (8 if dtype == torch.float64 else 4)
        c_est = int((torch.where(sel.bool(), pred.to(torch.float64), counts.to(torch.float64)).sum().item()
                     if m else 0) * 1.05)
        win = windows(ctx, m, products, span_lo, span_hi, sel, vb * c_est)
        _lib.call("sg_fallback", 0, n_fb, ptr(fb_rows), n, dcode, *fargs, None, None, None,
                  ptr(counts), win.struct(), ws, wsb, ctx.sp)
        row_ptr = scan(ctx, counts)
        nnz_c = int(row_ptr[-1].item()) if m else 0
        C_col, C_val = alloc_c(ctx, nnz_c, dtype, win)
    if win is not None and win.total:
        btile(ctx, B, win)
        wbytes = int(_lib.load().sg_window_work_bytes(m, A.nnz, win.total))
        work = ctx.empty((wbytes + 7) // 8, torch.int64)  # window items + entry tables
        ws, wsb = ctx.workspace(max(m, 1))
        _lib.call("sg_window_numeric", m, n, dcode, *Aargs, ptr(span_lo), ptr(span_hi), win.struct(),
                  ptr(row_ptr), ptr(C_col), ptr(C_val), ptr(work), work.numel() * 8, ws, wsb, ctx.sp)
    wstats = None
    if cfg.window_stats and win is not None:
        wrow = win.nwin[:m] > 0
        rl = row_ptr[1:] - row_ptr[:-1]
        al = A.row_ptr[1:] - A.row_ptr[:-1]
        wstats = {"rows": int(wrow.sum()), "windows": win.total, "nnz_a": int(al[wrow].sum()),
                  "products": int(products[wrow].sum()), "nnz_c": int(rl[wrow].sum()),
                  "saved_bitmaps": win.bm_save is not None}
    if short_fb is not None:
        # staged rows the reference would rerun already hold their values
        excl = ((win.nwin[:m] > 0) | short_fb).to(torch.int32)
        rest, n_rest = select_fallback(ctx, m, kind, products, overflow, excl)
    elif win is None:
        rest, n_rest = fb_rows, n_fb
    else:
        rest, n_rest = select_fallback(ctx, m, kind, products, overflow, win.nwin)
    if n_rest:
        _lib.call("sg_fallback", 1, n_rest, ptr(rest), n, dcode, *fargs, ptr(row_ptr),
                  ptr(C_col), ptr(C_val), ptr(counts), None, ws, wsb, ctx.sp)
    ev[5].record(ctx.stream)
    _nvtx.range_pop()
    _nvtx.range_push("spgemm:compact")  # reference stage (engine.py:147-216)
    _check_deadline(deadline)

    # ---- post-processing: hash rows were sorted in-kernel; compact the slab
    if exact and short is not None:
        _lib.call("sg_compact", m, _dtype_code(A.values), ptr(counts_s), ptr((~short).to(torch.uint8)),
                  ptr(st_off), ptr(row_ptr), ptr(st_col), ptr(st_val), ptr(C_col), ptr(C_val), ctx.sp)
        del st_col, st_val
    if not exact and m:
        skip = torch.zeros(m, dtype=torch.uint8, device=ctx.device)
        if n_fb:
            skip[fb_rows] = 1
        _lib.call("sg_compact", m, _dtype_code(A.values), ptr(counts), ptr(skip), ptr(out_off), ptr(row_ptr),
                  ptr(out_col), ptr(out_val), ptr(C_col), ptr(C_val), ctx.sp)
        del out_col, out_val
    if m == 0:
        row_ptr = torch.zeros(1, dtype=torch.int64, device=ctx.device)
        nnz_c = 0
    if cfg.deterministic and m and nnz_c:
        # values recomputed in the reference's sequential stream order
        acc = C_val if C_val.dtype == torch.float64 else ctx.empty(nnz_c, torch.float64)
        _lib.call("sg_det_values", m, _dtype_code(A.values), *Aargs, ptr(row_ptr), ptr(C_col), ptr(C_val),
                  ptr(acc), ctx.sp)
        del acc
    ev[6].record(ctx.stream)
    _nvtx.range_pop()
    ctx.sync()
    for i, name in enumerate(("analysis", "sketch", "predict", "numeric", "fallback", "compact")):
        kms[name] = ev[i].elapsed_time(ev[i + 1])

    est_mean = est_std = None
    if cfg.compute_estimation_errors and pred_kind == "estimated":
        # engine.py:218-226 on the device (sg_est_errors)
        out3 = (ctypes.c_double * 3)()
        scratch = ctx.empty(2 * 1024 + 8, torch.float64)
        _lib.call("sg_est_errors", m, ptr(pred), ptr(row_ptr), ctypes.cast(out3, ctypes.c_void_p), ptr(scratch),
                  scratch.numel() * 8, ctx.sp)
        est_mean, est_std = float(out3[1]), float(out3[2])

    Cd = DeviceCsr(m, n, row_ptr, C_col, C_val)
    total_ms = (time.perf_counter() - t0) * 1e3
    report = RunReport(
        workflow=kind_wf.value, registers=registers, er=er,
        cr_hat=None if cr is None else cr[0],
        cr_true=(total_products / nnz_c) if nnz_c else None,
        # stage times from the CUDA events on the call's stream (the stages
        # run back to back without host synchronisation in between)
        analysis_ms=kms["analysis"], sketch_ms=kms["sketch"] if regs is not None else 0.0,
        predict_ms=kms["predict"], numeric_ms=kms["numeric"], fallback_ms=kms["fallback"],
        compact_ms=kms["compact"], total_ms=total_ms, overflow_row_count=n_fb, nnz_c=nnz_c,
        total_products=total_products, bitmap_query=bool(bitmap_query),
        est_mean_rel_err=est_mean, est_std_rel_err=est_std,
        gflops=(2.0 * total_products / (total_ms * 1e-3) / 1e9) if total_ms > 0 else None,
        kernel_ms=kms, window_stats=wstats)
    if cfg.return_device:
        return Cd, report
    from .device import HOST_POOL
    return Cd.to_host(HOST_POOL if cfg.host_pool else None), report


def ctypes_int64():
    import ctypes
    return ctypes.c_int64(0)
