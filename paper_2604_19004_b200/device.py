"""Device-resident CSR (torch CUDA tensors used purely as buffers)."""

from __future__ import annotations

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

    def to_host(self) -> CsrMatrix:
        return CsrMatrix(self.nrows, self.ncols, download(self.row_ptr), download(self.col_idx),
                         download(self.values))


_STAGE_BYTES = 64 << 20
_NSTAGE = 4


def download(t: torch.Tensor) -> np.ndarray:
    """Device -> host numpy copy.  Large tensors go through a ring of pinned
    64 MB staging buffers: the copy engine fills buffer i+1 while host
    threads move buffer i into the (freshly page-faulted) destination, so
    PCIe and host page faults overlap instead of serialising."""
    n = t.numel()
    nbytes = n * t.element_size()
    if nbytes <= 4 * _STAGE_BYTES:
        return t.cpu().numpy()
    from concurrent.futures import ThreadPoolExecutor
    np_dt = {torch.int64: np.int64, torch.int32: np.int32, torch.float64: np.float64,
             torch.float32: np.float32, torch.uint8: np.uint8, torch.int8: np.int8}[t.dtype]
    out = np.empty(n, dtype=np_dt)
    src = t.view(torch.uint8) if t.is_contiguous() else t.contiguous().view(torch.uint8)
    dst = out.view(np.uint8)
    stages = [torch.empty(_STAGE_BYTES, dtype=torch.uint8, pin_memory=True) for _ in range(_NSTAGE)]
    events = [torch.cuda.Event() for _ in range(_NSTAGE)]
    stream = torch.cuda.Stream(device=t.device)
    stream.wait_stream(torch.cuda.current_stream(t.device))
    chunks = [(o, min(_STAGE_BYTES, nbytes - o)) for o in range(0, nbytes, _STAGE_BYTES)]
    pending = [None] * _NSTAGE

    def drain(i, o, ln):
        events[i].synchronize()
        dst[o:o + ln] = stages[i][:ln].numpy()

    with ThreadPoolExecutor(max_workers=_NSTAGE) as pool:
        for k, (o, ln) in enumerate(chunks):
            i = k % _NSTAGE
            if pending[i] is not None:
                pending[i].result()
            with torch.cuda.stream(stream):
                stages[i][:ln].copy_(src[o:o + ln], non_blocking=True)
                events[i].record(stream)
            pending[i] = pool.submit(drain, i, o, ln)
        for f in pending:
            if f is not None:
                f.result()
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
