"""B200-native estimation-based SpGEMM (Ocean, arXiv 2604.19004).

Drop-in for the reference package ``sketchgemm``'s multiply path: the same
``spgemm(a, b, cfg=None, deadline=None) -> (CsrMatrix, RunReport)`` entry
point, CSR interface, configuration, report and exceptions
(reference ``__init__.py:9-45``), computed by hand-written sm_100a kernels in
``libsgb200.so`` (C ABI: ``include/sgb200.h``).  There is no CPU fallback.
"""

from .config import (CR_THRESHOLD, ER_THRESHOLD, HASH_LOAD_LIMIT, REGISTER_ER_THRESHOLD,
                     UPPER_BOUND_AVG_PRODUCTS, CudaLibraryError, DeadlineExceeded, EngineConfig,
                     PlanKind, ResourceLimitError, RunReport, TierConfig, WorkflowKind,
                     WorkflowOverride, cr_variance_bound, select_registers, select_workflow)
from .csr import CsrMatrix, from_triplets, identity, transpose, validate

__version__ = "0.1.0"


def spgemm(a, b, cfg=None, deadline=None):
    """C = A @ B on the GPU; see engine.spgemm."""
    from .engine import spgemm as _spgemm
    return _spgemm(a, b, cfg, deadline)


def multiply_mode(a, mode, b=None):
    """Operand resolution for aa / aat / ab (reference engine.py:113-128)."""
    mode = mode.lower()
    if mode == "aa":
        if a.nrows != a.ncols:
            raise ValueError(f"AA requires a square matrix, got {a.nrows}x{a.ncols}")
        return a, a
    if mode == "aat":
        from .device import DeviceCsr
        if isinstance(a, DeviceCsr):
            from .build import transpose_device
            return a, transpose_device(a)
        return a, transpose(a)
    if mode == "ab":
        if b is None:
            raise ValueError("AB mode requires a second matrix")
        if a.ncols != b.nrows:
            raise ValueError(f"dimension mismatch: A is {a.nrows}x{a.ncols}, B is {b.nrows}x{b.ncols}")
        return a, b
    raise ValueError(f"unknown mode '{mode}' (expected aa, aat or ab)")


__all__ = [
    "CsrMatrix", "from_triplets", "identity", "transpose", "validate",
    "EngineConfig", "WorkflowOverride", "WorkflowKind", "RunReport", "TierConfig", "PlanKind",
    "ResourceLimitError", "DeadlineExceeded", "CudaLibraryError",
    "select_registers", "select_workflow", "cr_variance_bound",
    "spgemm", "multiply_mode", "from_triplets_device", "transpose_device",
]


def from_triplets_device(*args, **kwargs):
    """Canonical CSR from triplets on the GPU; see build.from_triplets_device."""
    from .build import from_triplets_device as f
    return f(*args, **kwargs)


def transpose_device(*args, **kwargs):
    """Exact transpose on the GPU; see build.transpose_device."""
    from .build import transpose_device as f
    return f(*args, **kwargs)
