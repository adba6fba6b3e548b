"""Row-sharded multi-GPU SpGEMM: one process per GPU.

Gustavson rows are independent (chunk independence is asserted
at engine.py:13-14), so C = A*B shards by rows of A with no exchange in the
data path:

  1. the root rank holds A and B; B (and A when it differs) is broadcast to
     every rank — ncclBroadcast over NVLink/NVSwitch via torch.distributed;
  2. rows of A are cut into contiguous ranges with balanced intermediate-
     product counts (the products prefix from the row-stats kernel on root);
  3. every rank runs the single-GPU pipeline (engine.spgemm) on its rows;
  4. offset exchange: all_gather of one int64 nnz per rank -> each shard's
     global row_ptr offset (the "stitch");
  5. optionally the shards are gathered to the root (NCCL send/recv) when C
     fits there; otherwise C stays distributed (R-MAT-23's C is ~2 TB).

The per-rank multiply is pluggable (``local_fn``) so the host logic — the
partition, broadcast, offset exchange and stitching — is tested on CPU with
gloo at world size 2 (tests/test_shard_gloo.py).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist


@dataclass
class Shard:
    """One rank's rows of C plus the stitching metadata."""

    row_lo: int
    row_hi: int
    nnz_offset: int          # global index of this shard's first entry
    nnz_total: int           # nnz of the whole C
    row_ptr: torch.Tensor    # local row_ptr (starts at 0)
    col_idx: torch.Tensor
    values: torch.Tensor
    report: object = None
    local: dict = None       # this rank's own counters: rows, nnz_a, products, nnz_c, batches


def balanced_cuts(products: np.ndarray, parts: int) -> list:
    """Contiguous row ranges with near-equal product sums (row r of rank i is
    in [cuts[i], cuts[i+1]))."""
    n = len(products)
    cum = np.concatenate(([0], np.cumsum(products, dtype=np.int64)))
    total = int(cum[-1])
    cuts = [0]
    for r in range(1, parts):
        cuts.append(int(np.searchsorted(cum, total * r / parts, side="left")))
    cuts.append(n)
    for i in range(1, len(cuts)):  # monotone
        cuts[i] = max(cuts[i], cuts[i - 1])
    return cuts


def _bcast_tensor(t, shape, dtype, device, src, group):
    if t is None:
        t = torch.empty(shape, dtype=dtype, device=device)
    dist.broadcast(t, src=src, group=group)
    return t


def broadcast_csr(m, device, src, group):
    """Broadcast a CSR (host or device arrays on `src`) to every rank as
    device tensors.  Returns (nrows, ncols, row_ptr, col_idx, values)."""
    rank = dist.get_rank(group)
    if rank == src:
        meta = torch.tensor([m.nrows, m.ncols, int(m.row_ptr[-1]),
                             0 if np.dtype(_np_dtype(m.values)) == np.float64 else 1],
                            dtype=torch.int64, device=device)
    else:
        meta = torch.empty(4, dtype=torch.int64, device=device)
    dist.broadcast(meta, src=src, group=group)
    nrows, ncols, nnz, dt = (int(x) for x in meta.tolist())
    vdt = torch.float64 if dt == 0 else torch.float32
    if rank == src:
        rp = _as_tensor(m.row_ptr, torch.int64, device)
        ci = _as_tensor(m.col_idx, torch.int32, device)
        vv = _as_tensor(m.values, vdt, device)
    else:
        rp = ci = vv = None
    rp = _bcast_tensor(rp, (nrows + 1,), torch.int64, device, src, group)
    ci = _bcast_tensor(ci, (nnz,), torch.int32, device, src, group)
    vv = _bcast_tensor(vv, (nnz,), vdt, device, src, group)
    return nrows, ncols, rp, ci, vv


def _np_dtype(v):
    return v.dtype if isinstance(v, np.ndarray) else {torch.float64: np.float64,
                                                      torch.float32: np.float32}[v.dtype]


def _as_tensor(x, dtype, device):
    if isinstance(x, torch.Tensor):
        return x.to(device=device, dtype=dtype).contiguous()
    return torch.from_numpy(np.ascontiguousarray(x)).to(device=device, dtype=dtype)


def row_products(a_ptr: torch.Tensor, a_col: torch.Tensor, b_ptr: torch.Tensor, b_col=None, b_ncols=None) -> np.ndarray:
    """Products per row of A (analysis.py:100-104) for partitioning, as a
    gather + cumsum over torch tensors (used on CPU test ranks; the GPU path
    uses the row-stats kernel)."""
    bn = (b_ptr[1:] - b_ptr[:-1])
    per_nz = bn[a_col.long()]
    cum = torch.cat([torch.zeros(1, dtype=torch.int64, device=per_nz.device), torch.cumsum(per_nz, 0)])
    return (cum[a_ptr[1:]] - cum[a_ptr[:-1]]).cpu().numpy()


@dataclass
class ShardPlan:
    """Everything a step needs, computed once (outside the timed loop):
    the row cuts, this rank's rows of A, the replicated B, the whole
    product's workflow decision and this rank's row batches."""

    cuts: list
    lo: int
    hi: int
    A: tuple                 # (nrows, ncols, row_ptr, col_idx, values) of the whole A (broadcast)
    B: tuple
    decision: object = None  # engine.Decision of the whole product (root), or None
    batches: list = None     # row ranges [lo_b, hi_b) covering [lo, hi)


_WF = ("symbolic", "estimate", "upper")


def _bcast_decision(dec, rank, root, group, device):
    """Broadcast an engine.Decision (or None) from root as 8 float64s."""
    t = torch.zeros(8, dtype=torch.float64, device=device)
    if rank == root and dec is not None:
        cr = dec.cr if dec.cr is not None else (0.0, 0.0, 0.0)
        t.copy_(torch.tensor([1.0, float(_WF.index(dec.workflow)), float(dec.registers), float(dec.er),
                              1.0 if dec.cr is not None else 0.0, cr[0], cr[1], cr[2]], dtype=torch.float64))
    tot = torch.tensor([dec.total_products if (rank == root and dec is not None) else 0], dtype=torch.int64,
                       device=device)
    dist.broadcast(t, src=root, group=group)
    dist.broadcast(tot, src=root, group=group)
    v = t.tolist()
    if v[0] == 0.0:
        return None
    from .engine import Decision
    return Decision(_WF[int(v[1])], int(v[2]), v[3], (v[5], v[6], v[7]) if v[4] else None, int(tot.item()))


def row_batches(per: np.ndarray, lo: int, hi: int, budget) -> list:
    """Contiguous row ranges of [lo, hi) with at most `budget` products each
    (a single row over budget is its own batch)."""
    if budget is None or hi <= lo:
        return [(lo, hi)]
    out, s, acc = [], lo, 0
    for r in range(lo, hi):
        pr = int(per[r - lo])
        if acc and acc + pr > budget:
            out.append((s, r))
            s, acc = r, 0
        acc += pr
    out.append((s, hi))
    return out


def plan_shards(a, b, group=None, root=0, device=None, products_fn=None, decide_fn=None,
                batch_products=None) -> ShardPlan:
    """Broadcast the operands from `root`, cut A's rows by balanced products,
    decide the workflow of the whole product once (decide_fn on root, e.g.
    engine.decide) and split this rank's rows into batches of at most
    `batch_products` products (C of R-MAT-23 does not fit in HBM at once)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    device = device or torch.device("cpu")
    same = rank == root and (b is a)
    flag = torch.tensor([1 if same else 0], dtype=torch.int64, device=device)
    dist.broadcast(flag, src=root, group=group)
    same = bool(flag.item())
    B = broadcast_csr(b if rank == root else None, device, root, group)
    A = B if same else broadcast_csr(a if rank == root else None, device, root, group)
    cuts_t = torch.empty(world + 1, dtype=torch.int64, device=device)
    per = None
    if rank == root:
        per = (products_fn or row_products)(A[2], A[3], B[2], B[3], B[1])
        cuts_t.copy_(torch.tensor(balanced_cuts(per, world), dtype=torch.int64))
    dist.broadcast(cuts_t, src=root, group=group)
    cuts = [int(x) for x in cuts_t.tolist()]
    dec = None
    if decide_fn is not None:
        from .device import DeviceCsr
        d = None
        if rank == root:
            Ad = DeviceCsr(A[0], A[1], A[2], A[3], A[4])
            Bd = Ad if same else DeviceCsr(B[0], B[1], B[2], B[3], B[4])
            d = decide_fn(Ad, Bd)
        dec = _bcast_decision(d, rank, root, group, device)
    lo, hi = cuts[rank], cuts[rank + 1]
    batches = [(lo, hi)]
    if batch_products is not None and hi > lo:
        s, e = int(A[2][lo].item()), int(A[2][hi].item())
        loc = (products_fn or row_products)((A[2][lo:hi + 1] - s).contiguous(), A[3][s:e].contiguous(),
                                            B[2], B[3], B[1])
        batches = row_batches(np.asarray(loc), lo, hi, batch_products)
    return ShardPlan(cuts, lo, hi, A, B, dec, batches)


def _rows(A, lo, hi):
    s, e = int(A[2][lo].item()), int(A[2][hi].item())
    return (hi - lo, A[1], (A[2][lo:hi + 1] - s).contiguous(), A[3][s:e].contiguous(), A[4][s:e].contiguous())


def _rep_get(rep, k):
    return rep[k] if isinstance(rep, dict) else getattr(rep, k)


def _rep_set(rep, k, v):
    if isinstance(rep, dict):
        rep[k] = v
    else:
        setattr(rep, k, v)


def run_shard(plan: ShardPlan, local_fn, group=None, root=0, gather=False, consume=None):
    """One row-sharded multiply with a precomputed plan.  Each batch of this
    rank's rows runs local_fn; ``consume(lo, hi, row_ptr, col_idx, values)``
    (if given) receives every batch's C and the batch is not kept (C too
    large for HBM).  Then the offset exchange (all_gather of one int64 per
    rank) places the shard in the global C, and the report counters that are
    per-row sums (nnz_c, overflow_row_count, total_products) are summed over
    ranks so the root's report describes the whole product."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    device = plan.A[2].device
    kw = {} if plan.decision is None else {"decision": plan.decision}
    parts, rep, nnz_loc = [], None, 0
    totals = torch.zeros(3, dtype=torch.int64, device=device)  # nnz_c, overflow rows, products
    for lo, hi in plan.batches:
        rp, ci, vv, r = local_fn(*_rows(plan.A, lo, hi), plan.B, **kw)
        totals += torch.tensor([int(ci.numel()), int(_rep_get(r, "overflow_row_count")),
                                int(_rep_get(r, "total_products"))], dtype=torch.int64, device=device)
        rep = r
        if consume is not None:
            consume(lo, hi, rp, ci, vv)
        else:
            parts.append((rp, ci, vv))
        nnz_loc += int(ci.numel())
    if consume is None:
        if len(parts) == 1:
            rp, ci, vv = parts[0]
        else:
            offs = np.cumsum([0] + [int(p[1].numel()) for p in parts])
            rp = torch.cat([parts[0][0][:1]] + [p[0][1:] + int(o) for p, o in zip(parts, offs[:-1])])
            ci = torch.cat([p[1] for p in parts])
            vv = torch.cat([p[2] for p in parts])
    else:
        rp = ci = vv = None
    nnz = torch.tensor([nnz_loc], dtype=torch.int64, device=device)
    all_nnz = [torch.zeros_like(nnz) for _ in range(world)]
    dist.all_gather(all_nnz, nnz, group=group)
    counts = [int(x.item()) for x in all_nnz]
    loc_totals = totals.clone()
    dist.all_reduce(totals, group=group)
    if rep is not None:
        nnz_all, ovf_all, prod_all = (int(x) for x in totals.tolist())
        _rep_set(rep, "nnz_c", nnz_all)
        _rep_set(rep, "overflow_row_count", ovf_all)
        _rep_set(rep, "total_products", prod_all)
        _rep_set(rep, "cr_true", (prod_all / nnz_all) if nnz_all else None)
    offset = int(sum(counts[:rank]))
    loc = {"rows": plan.hi - plan.lo, "nnz_a": int(plan.A[2][plan.hi].item() - plan.A[2][plan.lo].item()),
           "products": int(loc_totals[2].item()), "nnz_c": nnz_loc, "batches": len(plan.batches)}
    shard = Shard(plan.lo, plan.hi, offset, int(sum(counts)), rp, ci, vv, rep, loc)
    if not gather or consume is not None:
        return shard
    return gather_shards(shard, counts, plan.cuts, root, group, device)


def spgemm_sharded(a, b, local_fn, group=None, root=0, device=None, gather=False, products_fn=None,
                   decide_fn=None):
    """Row-sharded C = A*B over the ranks of `group`.

    ``a`` / ``b`` are needed on ``root`` only (host CsrMatrix or DeviceCsr; the
    other ranks pass None).  ``local_fn(nrows, ncols, row_ptr, col_idx,
    values, B[, decision=...]) -> (row_ptr, col_idx, values, report)``
    multiplies this rank's rows.  Returns the local ``Shard``; with
    ``gather=True`` the root's return value is the full C as a Shard covering
    all rows.  (plan_shards + run_shard, for one call.)
    """
    plan = plan_shards(a, b, group, root, device, products_fn, decide_fn)
    return run_shard(plan, local_fn, group, root, gather)


def gather_shards(shard: Shard, counts, cuts, root, group, device):
    """Stitch the shards into one CSR on `root` (NCCL/gloo point-to-point).
    gloo has no device point-to-point, so with gloo device shards travel
    through host copies."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    device = torch.device(device)
    via_host = device.type == "cuda" and dist.get_backend(group) == "gloo"

    def send(t, dst):
        dist.send(t.cpu() if via_host else t, dst=dst, group=group)

    def recv_into(t, src):
        if via_host:
            h = torch.empty(t.shape, dtype=t.dtype)
            dist.recv(h, src=src, group=group)
            t.copy_(h)
        else:
            dist.recv(t, src=src, group=group)

    if rank != root:
        if shard.col_idx.numel():
            send(shard.col_idx, root)
            send(shard.values, root)
        send(shard.row_ptr, root)
        return shard
    nrows = cuts[-1]
    total = int(sum(counts))
    col = torch.empty(total, dtype=shard.col_idx.dtype, device=device)
    val = torch.empty(total, dtype=shard.values.dtype, device=device)
    row_ptr = torch.empty(nrows + 1, dtype=torch.int64, device=device)
    off = 0
    for r in range(world):
        lo, hi = cuts[r], cuts[r + 1]
        n = counts[r]
        if r == rank:
            col[off:off + n] = shard.col_idx
            val[off:off + n] = shard.values
            rp = shard.row_ptr
        else:
            if n:
                recv_into(col[off:off + n], r)
                recv_into(val[off:off + n], r)
            rp = torch.empty(hi - lo + 1, dtype=torch.int64, device=device)
            recv_into(rp, r)
        row_ptr[lo:hi + 1] = rp + off
        off += n
    return Shard(0, nrows, 0, total, row_ptr, col, val, shard.report)


def gpu_products_fn(device):
    """products_fn for the root on a GPU: the row-stats kernel (analysis.py:96-128)."""
    from .device import DeviceCsr
    from .engine import _Ctx, row_stats

    def fn(a_ptr, a_col, b_ptr, b_col, b_ncols):
        ctx = _Ctx(device, torch.cuda.current_stream(device))
        m = a_ptr.numel() - 1
        A = DeviceCsr(m, b_ptr.numel() - 1, a_ptr, a_col, torch.empty(0, device=device))
        B = DeviceCsr(b_ptr.numel() - 1, int(b_ncols), b_ptr, b_col, torch.empty(0, device=device))
        prod, _, _, _ = row_stats(ctx, A, B)
        return prod.cpu().numpy()
    return fn


def gpu_local_fn(cfg):
    """local_fn running the single-GPU engine on this rank's device (with the
    root's decision for the whole product when the plan carries one)."""
    from .device import DeviceCsr
    from .engine import spgemm
    from dataclasses import replace

    cfg = replace(cfg, return_device=True)

    def fn(nrows, ncols_a, row_ptr, col_idx, values, B, decision=None):
        Ad = DeviceCsr(nrows, ncols_a, row_ptr, col_idx, values)
        Bd = DeviceCsr(B[0], B[1], B[2], B[3], B[4])
        c, rep = spgemm(Ad, Bd, cfg if decision is None else replace(cfg, decision=decision))
        rep.nrows_local = nrows
        return c.row_ptr, c.col_idx, c.values, rep
    return fn


def gpu_decide_fn(cfg, device):
    """decide_fn for the root: engine.decide on the whole operands."""
    from .engine import decide

    def fn(A, B):
        return decide(A, B, cfg, device)
    return fn
