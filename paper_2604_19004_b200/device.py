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

    def to_host(self, pinned_out=None) -> CsrMatrix:
        return CsrMatrix(self.nrows, self.ncols, self.row_ptr.cpu().numpy(),
                         self.col_idx.cpu().numpy(), self.values.cpu().numpy())


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
