"""Host CSR container, the reference's interface type (``csr.py:24-87``).

A ``CsrMatrix`` is canonical: ``row_ptr`` int64 (nrows + 1), ``col_idx`` int32
strictly increasing within each row, ``values`` float64 (or float32 for the
fp32 variant of the north star).  ``from_triplets`` sorts and sums duplicates;
it is host-side input preparation, not part of the multiply.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

MAX_INDEX = 2 ** 31  # int32 column indices (csr.py:17)


@dataclass
class CsrMatrix:
    nrows: int
    ncols: int
    row_ptr: np.ndarray  # int64, nrows + 1
    col_idx: np.ndarray  # int32, nnz
    values: np.ndarray   # float64 (or float32), nnz

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    def row(self, i: int):
        lo, hi = self.row_ptr[i], self.row_ptr[i + 1]
        return self.col_idx[lo:hi], self.values[lo:hi]

    def row_nnz(self) -> np.ndarray:
        return np.diff(self.row_ptr)

    def to_dense(self) -> np.ndarray:
        out = np.zeros((self.nrows, self.ncols), dtype=self.values.dtype)
        out[np.repeat(np.arange(self.nrows), self.row_nnz()), self.col_idx] = self.values
        return out

    def astype(self, dtype) -> "CsrMatrix":
        return CsrMatrix(self.nrows, self.ncols, self.row_ptr, self.col_idx,
                         self.values.astype(dtype))


def from_triplets(nrows: int, ncols: int, rows, cols, vals) -> CsrMatrix:
    """Canonical CSR from (row, col, value) triplets; duplicates summed."""
    if nrows >= MAX_INDEX or ncols >= MAX_INDEX:
        raise ValueError(f"matrix dimensions {nrows}x{ncols} exceed the 32-bit index limit")
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    vals = np.asarray(vals, dtype=np.float64)
    if len(rows) >= MAX_INDEX:
        raise ValueError("nnz exceeds the 32-bit index limit")
    if len(rows) == 0:
        return CsrMatrix(nrows, ncols, np.zeros(nrows + 1, np.int64),
                         np.empty(0, np.int32), np.empty(0, np.float64))
    key = rows * ncols + cols
    perm = np.argsort(key, kind="stable")
    key = key[perm]
    vals = vals[perm]
    head = np.flatnonzero(np.r_[True, key[1:] != key[:-1]])
    uk = key[head]
    ptr = np.zeros(nrows + 1, np.int64)
    np.cumsum(np.bincount(uk // ncols, minlength=nrows), out=ptr[1:])
    return CsrMatrix(nrows, ncols, ptr, (uk % ncols).astype(np.int32),
                     np.add.reduceat(vals, head))


def identity(n: int) -> CsrMatrix:
    return CsrMatrix(n, n, np.arange(n + 1, dtype=np.int64),
                     np.arange(n, dtype=np.int32), np.ones(n, dtype=np.float64))


def transpose(a: CsrMatrix) -> CsrMatrix:
    """Exact transpose (csr.py:90-97); used by the AA^T mode only."""
    rows = np.repeat(np.arange(a.nrows, dtype=np.int64), a.row_nnz())
    order = np.argsort(a.col_idx, kind="stable")
    ptr = np.zeros(a.ncols + 1, np.int64)
    np.cumsum(np.bincount(a.col_idx, minlength=a.ncols), out=ptr[1:])
    return CsrMatrix(a.ncols, a.nrows, ptr, rows[order].astype(np.int32), a.values[order])


def validate(a: CsrMatrix) -> list:
    """Canonical-form checks (csr.py:100-133), condensed to one message per class."""
    out = []
    ptr = np.asarray(a.row_ptr)
    if len(ptr) != a.nrows + 1:
        return [f"row_ptr length {len(ptr)} != nrows + 1"]
    if ptr[0] != 0:
        out.append("row_ptr[0] != 0")
    if np.any(np.diff(ptr) < 0):
        out.append("row_ptr not non-decreasing")
    if out:
        return out
    if ptr[-1] != len(a.col_idx) or len(a.values) != len(a.col_idx):
        return ["nnz mismatch between row_ptr, col_idx and values"]
    if len(a.col_idx) and (a.col_idx.min() < 0 or a.col_idx.max() >= a.ncols):
        out.append("column out of range")
    if len(a.col_idx) > 1:
        bad = np.flatnonzero(np.diff(a.col_idx.astype(np.int64)) <= 0) + 1
        if len(bad) and not np.all(np.isin(bad, ptr[1:-1])):
            out.append("duplicate/unsorted column within a row")
    return out
