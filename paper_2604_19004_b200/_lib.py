"""ctypes binding of libsgb200.so (the C ABI declared in include/sgb200.h).

The library is built in-tree by ``__graft_entry__.build()`` (``make -C
paper_2604_19004_b200/csrc``).  There is no fallback: if the library or a CUDA
device is missing, every entry point raises ``CudaLibraryError``.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from .config import CudaLibraryError

LIB_PATH = os.environ.get("SGB200_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libsgb200.so")

_lock = threading.Lock()
_lib = None

I64, I32, SZ, P, D = C.c_int64, C.c_int, C.c_size_t, C.c_void_p, C.c_double


class SgWindows(C.Structure):
    _fields_ = [("win_off", C.c_void_p), ("wins", C.c_void_p), ("nwin", C.c_void_p),
                ("bm_off", C.c_void_p), ("bm_save", C.c_void_p), ("pre_save", C.c_void_p),
                ("btile_off", C.c_void_p), ("btile", C.c_void_p)]


class SgTiers(C.Structure):
    _fields_ = [("n_hash", C.c_int32), ("n_dense", C.c_int32),
                ("hash_caps", C.c_int64 * 8), ("dense_spans", C.c_int64 * 8),
                ("enh_cap", C.c_int64), ("esc_max", C.c_int64), ("coef", C.c_double)]


# name -> (restype, argtypes); mirrors include/sgb200.h one to one
SIGNATURES = {
    "sg_abi_version": (I32, []),
    "sg_last_error": (C.c_char_p, []),
    "sg_launch_count": (C.c_ulonglong, []),
    "sg_kernel_timer": (I32, [I32]),
    "sg_build_workspace_bytes": (SZ, [I64]),
    "sg_coo_to_csr": (I32, [I64, I64, I64, P, P, P, I32, P, P, P, P, P, SZ, P]),
    "sg_transpose": (I32, [I64, I64, P, P, P, I32, P, P, P, P, SZ, P]),
    "sg_download": (I32, [P, P, SZ, I32, P]),
    "sg_est_errors": (I32, [I64, P, P, P, P, SZ, P]),
    "sg_host_pin": (I32, [P, SZ, I32]),
    "sg_host_unpin": (I32, [P, SZ, I32]),
    "sg_kernel_time": (I32, [C.c_char_p, P, P]),
    "sg_workspace_bytes": (SZ, [I64]),
    "sg_row_stats": (I32, [I64, I64, P, P, P, P, P, P, P, P, P]),
    "sg_hll_build": (I32, [I64, P, P, I32, P, P]),
    "sg_hll_estimate": (I32, [I64, P, P, P, P, I32, P, D, P, P]),
    "sg_window_capacity": (I32, [I64, P, P, P, P, P, P, P, P, SZ, P]),
    "sg_symbolic": (I32, [I64, I64, P, P, P, P, P, P, P, P, C.POINTER(SgWindows), D, I64, P, SZ, P]),
    "sg_window_numeric": (I32, [I64, I64, I32, P, P, P, P, P, P, P, P, C.POINTER(SgWindows), P, P, P, P,
                                I64, P, SZ, P]),
    "sg_btile_plan": (I32, [I64, I64, P, I64, P, P, P, SZ, P]),
    "sg_window_work_bytes": (I64, [I64, I64, I64]),
    "sg_det_values": (I32, [I64, I32, P, P, P, P, P, P, P, P, P, P, P]),
    "sg_btile_build": (I32, [I64, I64, P, P, P, P, P, P]),
    "sg_plan": (I32, [I64, I32, P, P, P, P, C.POINTER(SgTiers), P, P, P, P]),
    "sg_scan": (I32, [I64, P, P, P, SZ, P]),
    "sg_numeric": (I32, [I64, I64, I32, P, P, P, P, P, P, P, P, P, P, P, P, P, P, P, P, P, P, P, I64, P, SZ, P]),
    "sg_select_fallback": (I32, [I64, P, P, P, P, P, C.POINTER(C.c_int64), P, SZ, P]),
    "sg_fallback": (I32, [I32, I64, P, I64, I32, P, P, P, P, P, P, P, P, P, P, P, P, P,
                          C.POINTER(SgWindows), P, SZ, P]),
    "sg_compact": (I32, [I64, I32, P, P, P, P, P, P, P, P, P]),
}


def load():
    """Return the loaded library (cached); raise CudaLibraryError if unusable."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise CudaLibraryError(
                f"{LIB_PATH} is missing: run __graft_entry__.build() (make -C "
                "paper_2604_19004_b200/csrc); there is no CPU fallback")
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.sg_abi_version() != 1:
            raise CudaLibraryError("libsgb200.so ABI version mismatch")
        _lib = lib
    return _lib


def call(name, *args):
    """Invoke an entry point and raise on a non-zero status."""
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc != 0:
        msg = lib.sg_last_error().decode(errors="replace")
        raise CudaLibraryError(f"{name} failed (status {rc}): {msg}")
    return rc


def exported_symbols():
    return list(SIGNATURES)
