"""Canonical CSR construction on the device.

``from_triplets_device`` replaces ``csr.from_triplets`` (reference
csr.py:52-80) and ``transpose_device`` replaces ``csr.transpose``
(csr.py:90-97, the AA^T operand of engine.py:113-128); both call
``sg_coo_to_csr`` / ``sg_transpose`` in libsgb200.so (include/sgb200.h).
Inputs may be numpy arrays (uploaded) or torch CUDA tensors; results are
``DeviceCsr``.  Errors follow the reference: ValueError for dimensions or nnz
beyond the 32-bit index limit, and for out-of-range coordinates.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .config import CudaLibraryError
from .csr import MAX_INDEX
from .device import DeviceCsr, ptr


def _device(device):
    if not torch.cuda.is_available():
        raise CudaLibraryError("no CUDA device: the B200 path has no CPU fallback")
    return torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())


def _as_dev(x, dtype, device):
    if isinstance(x, torch.Tensor):
        return x.to(device=device, dtype=dtype).contiguous()
    return torch.from_numpy(np.ascontiguousarray(x)).to(device=device, dtype=dtype)


def from_triplets_device(nrows: int, ncols: int, rows, cols, vals, device=None,
                         dtype: torch.dtype = torch.float64, stream=None) -> DeviceCsr:
    """Canonical device CSR from (row, col, value) triplets; duplicates are
    summed in input order (the reference's stable argsort + reduceat)."""
    if nrows >= MAX_INDEX or ncols >= MAX_INDEX:
        raise ValueError(f"matrix dimensions {nrows}x{ncols} exceed the 32-bit index limit")
    dev = _device(device)
    r = _as_dev(rows, torch.int64, dev)
    c = _as_dev(cols, torch.int64, dev)
    v = _as_dev(vals, dtype, dev)
    n = int(r.numel())
    if n >= MAX_INDEX:
        raise ValueError("nnz exceeds the 32-bit index limit")
    if c.numel() != n or v.numel() != n:
        raise ValueError("rows, cols and vals must have the same length")
    lib = _lib.load()
    stream = stream or torch.cuda.current_stream(dev)
    if stream != torch.cuda.current_stream(dev):
        stream.wait_stream(torch.cuda.current_stream(dev))  # inputs uploaded on the current stream
    # allocations are made on `stream` (so the caching allocator orders
    # their reuse after its work) and the stream is drained before the
    # workspace is dropped
    with torch.cuda.stream(stream):
        ws = torch.empty(int(lib.sg_build_workspace_bytes(n)), dtype=torch.uint8, device=dev)
        row_ptr = torch.empty(nrows + 1, dtype=torch.int64, device=dev)
        col = torch.empty(n, dtype=torch.int32, device=dev)
        val = torch.empty(n, dtype=dtype, device=dev)
    nu = ctypes.c_int64(0)
    code = 0 if dtype == torch.float64 else 1
    try:
        _lib.call("sg_coo_to_csr", nrows, ncols, n, ptr(r), ptr(c), ptr(v), code, ptr(row_ptr), ptr(col),
                  ptr(val), ctypes.byref(nu), ptr(ws), ws.numel(), stream.cuda_stream)
    except CudaLibraryError as exc:
        if "out of range" in str(exc):
            raise ValueError(str(exc)) from exc
        raise
    finally:
        stream.synchronize()
    k = int(nu.value)
    return DeviceCsr(nrows, ncols, row_ptr, col[:k], val[:k])


def transpose_device(a, device=None, stream=None) -> DeviceCsr:
    """Exact transpose of a canonical CSR (host CsrMatrix or DeviceCsr)."""
    dev = _device(device if device is not None else (a.row_ptr.device if isinstance(a, DeviceCsr) else None))
    if isinstance(a, DeviceCsr):
        rp, ci, vv = a.row_ptr, a.col_idx, a.values
    else:
        rp = _as_dev(a.row_ptr, torch.int64, dev)
        ci = _as_dev(a.col_idx, torch.int32, dev)
        vv = _as_dev(a.values, torch.float64 if np.asarray(a.values).dtype != np.float32 else torch.float32, dev)
    nnz = int(ci.numel())
    lib = _lib.load()
    stream = stream or torch.cuda.current_stream(dev)
    if stream != torch.cuda.current_stream(dev):
        stream.wait_stream(torch.cuda.current_stream(dev))  # inputs uploaded on the current stream
    with torch.cuda.stream(stream):
        ws = torch.empty(int(lib.sg_build_workspace_bytes(nnz)), dtype=torch.uint8, device=dev)
        t_ptr = torch.empty(a.ncols + 1, dtype=torch.int64, device=dev)
        t_col = torch.empty(nnz, dtype=torch.int32, device=dev)
        t_val = torch.empty(nnz, dtype=vv.dtype, device=dev)
    try:
        _lib.call("sg_transpose", a.nrows, a.ncols, ptr(rp), ptr(ci), ptr(vv),
                  0 if vv.dtype == torch.float64 else 1,
                  ptr(t_ptr), ptr(t_col), ptr(t_val), ptr(ws), ws.numel(), stream.cuda_stream)
    finally:
        stream.synchronize()  # the workspace is released on return
    return DeviceCsr(a.ncols, a.nrows, t_ptr, t_col, t_val)
