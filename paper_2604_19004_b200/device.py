"""Device-resident CSR (torch CUDA tensors used purely as buffers)."""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np
import torch

from .csr import CsrMatrix


def ptr(t):
    """Raw device address for the C ABI (None for an absent tensor)."""
    if t is None:
        return None
    return t.data_ptr() if t.numel() else None


@dataclass
class DeviceCsr:
    nrows: int
    ncols: int
    row_ptr: torch.Tensor  # int64 [nrows+1]
    col_idx: torch.Tensor  # int32 [nnz]
    values: torch.Tensor   # float64 / float32 [nnz]

    @property
    def nnz(self) -> int:
        return int(self.col_idx.numel())

    def rows(self, lo: int, hi: int) -> CsrMatrix:
        """Host copy of rows [lo, hi) (row_ptr rebased to 0)."""
        rp = self.row_ptr[lo:hi + 1].cpu().numpy()
        s, e = int(rp[0]), int(rp[-1])
        return CsrMatrix(hi - lo, self.ncols, rp - s, self.col_idx[s:e].cpu().numpy(),
                         self.values[s:e].cpu().numpy())

    def to_host(self, pool: "HostPool | None" = None) -> CsrMatrix:
        return CsrMatrix(self.nrows, self.ncols, download(self.row_ptr, pool=pool),
                         download(self.col_idx, pool=pool), download(self.values, pool=pool))


_STAGE_BYTES = 64 << 20


class HostPool:
    """Recycled page-locked host buffers for results (opt-in:
    ``EngineConfig(host_pool=True)``).

    A result array is a view of an anonymous mapping pinned once by
    ``sg_host_pin`` (parallel first touch + 256 MB registrations), so the
    download is one DMA per chunk with no page faults or staging copies.  When
    the caller drops the array its buffer returns to the pool for the next
    result of the same 64 MB-rounded size.  The pool never holds more than
    ``share`` of physical memory; beyond that results fall back to fresh
    pageable arrays.  ``release()`` unpins and frees idle buffers.
    """

    GRAIN = 64 << 20

    def __init__(self, share: float = 0.6):
        import threading
        self.share = share
        self.free: dict = {}
        self.total = 0
        self.lock = threading.Lock()

    def _limit(self):
        try:
            return int(self.share * os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES"))
        except (ValueError, OSError):
            return 0

    def array(self, n: int, dtype, threads: int) -> np.ndarray | None:
        import ctypes
        import mmap
        import weakref
        from . import _lib
        itemsize = np.dtype(dtype).itemsize
        size = max(self.GRAIN, (n * itemsize + self.GRAIN - 1) // self.GRAIN * self.GRAIN)
        with self.lock:
            lst = self.free.get(size)
            blk = lst.pop() if lst else None
            if blk is None:
                if self.total + size > self._limit():
                    return None
                self.total += size
        if blk is None:
            m = mmap.mmap(-1, size, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
            try:
                m.madvise(mmap.MADV_HUGEPAGE)
            except (AttributeError, OSError):
                pass
            anchor = ctypes.c_char.from_buffer(m)
            try:
                _lib.call("sg_host_pin", ctypes.addressof(anchor), size, threads)
            except Exception:
                with self.lock:
                    self.total -= size
                del anchor
                m.close()
                return None
            blk = (m, anchor)
        arr = np.frombuffer(blk[0], dtype=dtype, count=n)
        weakref.finalize(arr, self._give_back, size, blk)
        return arr

    def _give_back(self, size, blk):
        with self.lock:
            self.free.setdefault(size, []).append(blk)

    def release(self):
        """Unpin and unmap every idle buffer."""
        import ctypes
        from . import _lib
        with self.lock:
            idle = [(size, b) for size, lst in self.free.items() for b in lst]
            self.free = {}
            self.total -= sum(size for size, _ in idle)
        while idle:
            size, (m, anchor) = idle.pop()
            _lib.call("sg_host_unpin", ctypes.addressof(anchor), size, 8)
            del anchor
            m.close()


HOST_POOL = HostPool()


def download(t: torch.Tensor, threads: int | None = None, pool: HostPool | None = None) -> np.ndarray:
    """Device -> host numpy copy.  Large tensors go through sg_download
    (libsgb200.so): pinned staging ring filled by the copy engine, drained by
    native worker threads that also take the destination's page faults in
    parallel (a single host thread is page-fault bound at ~7 GB/s)."""
    n = t.numel()
    nbytes = n * t.element_size()
    if nbytes <= (16 << 20 if pool is not None else 4 * _STAGE_BYTES):
        return t.cpu().numpy()
    from . import _lib
    np_dt = {torch.int64: np.int64, torch.int32: np.int32, torch.float64: np.float64,
             torch.float32: np.float32, torch.uint8: np.uint8, torch.int8: np.int8}[t.dtype]
    src = t if t.is_contiguous() else t.contiguous()
    nthr = threads or min(16, max(4, (os.cpu_count() or 8)))
    out = pool.array(n, np_dt, nthr) if pool is not None else None
    if out is None:
        out = np.empty(n, dtype=np_dt)
    _lib.call("sg_download", out.ctypes.data, src.data_ptr(), nbytes, nthr,
              torch.cuda.current_stream(t.device).cuda_stream)
    return out


def to_device(m, device, dtype=torch.float64, non_blocking=False) -> DeviceCsr:
    """Upload a host CSR (or pass a DeviceCsr through, casting values if needed)."""
    if isinstance(m, DeviceCsr):
        if m.values.dtype != dtype:
            return DeviceCsr(m.nrows, m.ncols, m.row_ptr, m.col_idx, m.values.to(dtype))
        return m
    rp = torch.from_numpy(np.ascontiguousarray(m.row_ptr, dtype=np.int64))
    ci = torch.from_numpy(np.ascontiguousarray(m.col_idx, dtype=np.int32))
    np_dt = np.float64 if dtype == torch.float64 else np.float32
    vv = torch.from_numpy(np.ascontiguousarray(m.values, dtype=np_dt))
    return DeviceCsr(int(m.nrows), int(m.ncols), rp.to(device, non_blocking=non_blocking),
                     ci.to(device, non_blocking=non_blocking), vv.to(device, non_blocking=non_blocking))
