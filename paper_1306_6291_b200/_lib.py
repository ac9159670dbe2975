"""ctypes binding of the C ABI in include/symdiag_b200.h.

The library (paper_1306_6291_b200/lib/libsymdiag_b200.so) is the product:
there is no CPU fallback.  Any call without the library or without a CUDA
device raises `CudaUnavailable`.
"""

from __future__ import annotations

import ctypes
import threading
from pathlib import Path

import os

# SD_LIB_PATH: a variant build of the same library (tools/ experiments only)
LIB_PATH = Path(os.environ.get("SD_LIB_PATH") or
                Path(__file__).resolve().parent / "lib" / "libsymdiag_b200.so")

SD_OK, SD_EINVAL, SD_ECUDA, SD_ENOMEM = 0, 1, 2, 3
REPORT_STRIDE = 24

# every exported symbol of include/symdiag_b200.h with its ctypes signature
_P, _I64, _I = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
SIGNATURES = {
    "sd_eig2_f64": [_P, _I64, _P, _P, _P, _P],
    "sd_eig3_f64": [_P, _I64, _P, _P, _P, _P],
    "sd_eig3_f32": [_P, _I64, _P, _P, _P, _P],
    "sd_eig3_report_f64": [_P, _I64, _P, _P, _P, _P, _P, _P],
    "sd_eig2_report_f64": [_P, _I64, _P, _P, _P, _P, _P],
    "sd_char_coeffs_f64": [_P, _I64, _P, _P, _P],
    "sd_compute_pq_f64": [_P, _I64, _P, _P, _P],
    "sd_eigenvalues3_f64": [_P, _P, _I64, _P, _P],
    "sd_pq_expanded_f64": [_P, _I64, _P, _P, _P],
    "sd_compute_v_f64": [_P, _P, _I64, _P, _P, _P],
    "sd_compute_w_f64": [_P, _P, _P, _I64, _P, _P, _P],
    "sd_resolve_signs_f64": [_P, _P, _P, _I64, _P, _P, _P, _P],
    "sd_degenerate_double_f64": [_P, _P, _I64, _P, _P, _P, _P],
    "sd_f_vectors_f64": [_P, _I64, _P, _P],
    "sd_g_vectors_f64": [_P, _I64, _P, _P],
    "sd_compose_rotation_f64": [_P, _I64, _P, _P],
    "sd_jacobi_f64": [_I, _P, _I64, ctypes.c_double, _P, _P, _P, _P, _P, _P],
    "sd_residuals_f64": [_I, _P, _P, _P, _I64, _P, _P],
    "sd_cubic_roots_f64": [_P, _I64, _P, _P, _P],
    "sd_glibc_pow_f64": [_P, _P, _I64, _P, _P],
    "sd_crlibm_f64": [_I, _P, _P, _I64, _P, _P],
    "sd_plan_create": [_I, _I64, ctypes.POINTER(_P)],
    "sd_eig3_report_f64_host": [_P, _P, _I64, _P, _P, _P, _P, _P],
    "sd_eig2_report_f64_host": [_P, _P, _I64, _P, _P, _P, _P],
    "sd_jsonl_parse": [_P, _I64, _I64, _I, _P, _P, _P, _P],
    "sd_jsonl_format": [_I64, _P, _P, _P, _P, _P, _P, _P, _P, _I, _P, _I64, _P],
    "sd_plan_destroy": [_P],
    "sd_eig3_f64_host": [_P, _P, _I64, _P, _P, _P],
    "sd_eig3_f32_host": [_P, _P, _I64, _P, _P, _P],
    "sd_eig2_f64_host": [_P, _P, _I64, _P, _P, _P],
    "sd_eig3_literal_f64": [_P, _I64, _P, _P, _P, _P],
    "sd_eig3_classify_f64": [_P, _I64, _P, _P, _P, _P],
    "sd_probe_dfma": [_I, _I, _P, ctypes.POINTER(ctypes.c_double), _P],
    "sd_last_error": [],
    "sd_version": [],
    "sd_launch_count": [],
}
RESTYPES = {"sd_last_error": ctypes.c_char_p, "sd_version": ctypes.c_char_p,
            "sd_launch_count": ctypes.c_int64, "sd_jsonl_parse": ctypes.c_int64,
            "sd_jsonl_format": ctypes.c_int64}


class CudaUnavailable(RuntimeError):
    """The CUDA library or a CUDA device is missing; there is no CPU path."""


class SymdiagError(RuntimeError):
    """A C-ABI call returned an error code (argument or CUDA launch error)."""


_lock = threading.Lock()
_lib = None


def load(build_if_missing: bool = True):
    """Load (building in-tree first if needed) and type the library."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists() and build_if_missing:
            from . import build_ext
            build_ext.build()
        if not LIB_PATH.exists():
            raise CudaUnavailable(f"{LIB_PATH} missing: run __graft_entry__.build()")
        try:
            L = ctypes.CDLL(str(LIB_PATH))
        except OSError as e:  # e.g. libcudart missing
            raise CudaUnavailable(f"cannot load {LIB_PATH}: {e}") from e
        for name, args in SIGNATURES.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = RESTYPES.get(name, ctypes.c_int)
        _lib = L
        return L


def call(name: str, *args):
    rc = getattr(load(), name)(*args)
    if rc != SD_OK:
        msg = load().sd_last_error().decode(errors="replace")
        raise SymdiagError(f"{name} returned {rc}: {msg}")


def launch_count() -> int:
    return int(load().sd_launch_count())


def require_cuda():
    """Fail loudly when no CUDA device is visible (no CPU fallback)."""
    import torch
    if not torch.cuda.is_available():
        raise CudaUnavailable("symdiag_b200 needs a CUDA device (B200); none is visible")
    load()
