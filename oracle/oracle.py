"""ctypes front end of the CPU ORACLE (test infrastructure, NOT product code).

Loads oracle/build/libsymdiag_oracle.so (built from symdiag_oracle.c by
oracle/Makefile, or by __graft_entry__.build()).  Every function takes and
returns numpy arrays in the packed layouts of include/symdiag_b200.h.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this module.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
# SD_ORACLE_LIB selects another build of the same source (tools only, e.g.
# build/libsymdiag_oracle_cr.so: the correctly rounded libm variant)
LIB_PATH = Path(os.environ.get("SD_ORACLE_LIB", HERE / "build" / "libsymdiag_oracle.so"))
REPORT_STRIDE = 24

_lib = None


def build(force: bool = False) -> Path:
    if force or not LIB_PATH.exists():
        subprocess.run(["make", "-C", str(HERE)], check=True,
                       stdout=subprocess.PIPE, stderr=subprocess.STDOUT)
    return LIB_PATH


CR_LIB_PATH = HERE / "build" / "libsymdiag_oracle_cr.so"
_libs = {}


def lib(path=None):
    """The oracle library (glibc libm); `path` = another build of the same
    source, e.g. CR_LIB_PATH (the correctly rounded libm variant)."""
    global _lib
    if path is not None:
        if path not in _libs:
            if not Path(path).exists():
                build(force=True)
            _libs[path] = _bind(ctypes.CDLL(str(path)))
        return _libs[path]
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        _lib = _bind(ctypes.CDLL(str(LIB_PATH)))
    return _lib


def _bind(L):
    if True:
        P = ctypes.c_void_p
        I64 = ctypes.c_int64
        L.sdo_eig3.argtypes = [P, I64, P, P, P, P, P, ctypes.c_int]
        L.sdo_eig3_f32.argtypes = [P, I64, P, P, P, ctypes.c_int]
        L.sdo_eig2.argtypes = [P, I64, P, P, P, P, ctypes.c_int]
        L.sdo_char_coeffs.argtypes = [P, I64, P, P]
        L.sdo_compute_pq.argtypes = [P, I64, P, P]
        L.sdo_eigenvalues3.argtypes = [P, P, I64, P]
        L.sdo_pq_expanded.argtypes = [P, I64, P, P]
        L.sdo_compute_vw.argtypes = [P, P, I64, P, P]
        L.sdo_compute_w.argtypes = [P, P, P, I64, P, P]
        L.sdo_resolve_signs.argtypes = [P, P, P, I64, P, P, P]
        L.sdo_degenerate_double.argtypes = [P, P, I64, P, P, P]
        L.sdo_g_vectors.argtypes = [P, I64, P]
        L.sdo_compose_rotation.argtypes = [P, I64, P]
        L.sdo_jacobi.argtypes = [ctypes.c_int, P, I64, ctypes.c_double, P, P, P, P, P,
                                 ctypes.c_int]
        L.sdo_residuals.argtypes = [ctypes.c_int, P, P, P, I64, P]
        L.sdo_set_nudge.argtypes = [ctypes.c_int, ctypes.c_uint64]
        L.sdo_py_hypot.argtypes = [ctypes.c_double, ctypes.c_double]
        L.sdo_py_hypot.restype = ctypes.c_double
    return L


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def _c(a, dtype=np.float64, width=None):
    a = np.ascontiguousarray(a, dtype=dtype)
    if width is not None:
        a = a.reshape(-1, width)
    return a


def default_threads() -> int:
    return len(os.sched_getaffinity(0))


def eig3(A, nthreads: int = 1, report: bool = False, d: bool = False, cr: bool = False):
    """diagonalize3 over packed A[n,6] -> dict(lam, ang, status[, report, d]).
    cr=True: the build with correctly rounded sin/cos/acos/asin/atan2/hypot
    (oracle/cr_variant.c) -- the libm of the device's literal solver."""
    A = _c(A, width=6)
    n = A.shape[0]
    out = dict(lam=np.empty((n, 3)), ang=np.empty((n, 3)),
               status=np.empty(n, np.uint8))
    out["report"] = np.empty((n, REPORT_STRIDE)) if report else None
    out["d"] = np.empty((n, 9)) if d else None
    lib(CR_LIB_PATH if cr else None).sdo_eig3(
        _p(A), n, _p(out["lam"]), _p(out["ang"]), _p(out["status"]),
        _p(out["report"]), _p(out["d"]), nthreads)
    return out


def eig3_f32(A, nthreads: int = 1):
    A = _c(A, np.float32, 6)
    n = A.shape[0]
    out = dict(lam=np.empty((n, 3), np.float32), ang=np.empty((n, 3), np.float32),
               status=np.empty(n, np.uint8))
    lib().sdo_eig3_f32(_p(A), n, _p(out["lam"]), _p(out["ang"]),
                       _p(out["status"]), nthreads)
    return out


def eig2(A, nthreads: int = 1, d: bool = False):
    A = _c(A, width=3)
    n = A.shape[0]
    out = dict(lam=np.empty((n, 2)), phi=np.empty(n), status=np.empty(n, np.uint8))
    out["d"] = np.empty((n, 4)) if d else None
    lib().sdo_eig2(_p(A), n, _p(out["lam"]), _p(out["phi"]), _p(out["status"]),
                   _p(out["d"]), nthreads)
    return out


def char_coeffs(A):
    A = _c(A, width=6)
    out, st = np.empty((A.shape[0], 3)), np.empty(A.shape[0], np.uint8)
    lib().sdo_char_coeffs(_p(A), A.shape[0], _p(out), _p(st))
    return out, st


def compute_pq(bcd):
    bcd = _c(bcd, width=3)
    n = bcd.shape[0]
    out, st = np.empty((n, 3)), np.empty(n, np.uint8)
    lib().sdo_compute_pq(_p(bcd), n, _p(out), _p(st))
    return out, st


def eigenvalues3(bcd, pqd):
    bcd, pqd = _c(bcd, width=3), _c(pqd, width=3)
    out = np.empty((bcd.shape[0], 3))
    lib().sdo_eigenvalues3(_p(bcd), _p(pqd), bcd.shape[0], _p(out))
    return out


def pq_expanded(A):
    A = _c(A, width=6)
    out, st = np.empty((A.shape[0], 2)), np.empty(A.shape[0], np.uint8)
    lib().sdo_pq_expanded(_p(A), A.shape[0], _p(out), _p(st))
    return out, st


def compute_vw(A, lam):
    A, lam = _c(A, width=6), _c(lam, width=3)
    n = A.shape[0]
    out, st = np.empty((n, 2)), np.empty(n, np.uint8)
    lib().sdo_compute_vw(_p(A), _p(lam), n, _p(out), _p(st))
    return out, st


def compute_w(A, lam, v):
    A, lam = _c(A, width=6), _c(lam, width=3)
    v = np.ascontiguousarray(v, dtype=np.float64).reshape(-1)
    n = A.shape[0]
    out, st = np.empty(n), np.empty(n, np.uint8)
    lib().sdo_compute_w(_p(A), _p(lam), _p(v), n, _p(out), _p(st))
    return out, st


def resolve_signs(A, lam, vw):
    A, lam, vw = _c(A, width=6), _c(lam, width=3), _c(vw, width=2)
    n = A.shape[0]
    ang, st = np.empty((n, 3)), np.empty(n, np.uint8)
    rep = np.empty((n, REPORT_STRIDE))
    lib().sdo_resolve_signs(_p(A), _p(lam), _p(vw), n, _p(ang), _p(st), _p(rep))
    return ang, st, rep


def degenerate_double(A, lam2):
    A, lam2 = _c(A, width=6), _c(lam2, width=2)
    n = A.shape[0]
    ang, st = np.empty((n, 3)), np.empty(n, np.uint8)
    rep = np.empty((n, REPORT_STRIDE))
    lib().sdo_degenerate_double(_p(A), _p(lam2), n, _p(ang), _p(st), _p(rep))
    return ang, st, rep


def g_vectors(inp):
    inp = _c(inp, width=7)
    out = np.empty((inp.shape[0], 4))
    lib().sdo_g_vectors(_p(inp), inp.shape[0], _p(out))
    return out


def compose_rotation(ang):
    ang = _c(ang, width=3)
    out = np.empty((ang.shape[0], 9))
    lib().sdo_compose_rotation(_p(ang), ang.shape[0], _p(out))
    return out


def jacobi(A, dim: int = 3, tol: float = 1e-13, nthreads: int = 1):
    """jacobi_eigen (oracle.py:45-84) over packed rows -> dict(evals, evecs
    [n, dim*dim] row-major, sweeps, offdiag, status (0, 1 NoConvergence, 8))."""
    w = 3 if dim == 2 else 6
    A = _c(A, width=w)
    n = A.shape[0]
    out = dict(evals=np.empty((n, dim)), evecs=np.empty((n, dim * dim)),
               sweeps=np.empty(n, np.int32), offdiag=np.empty(n), status=np.empty(n, np.uint8))
    lib().sdo_jacobi(dim, _p(A), n, tol, _p(out["evals"]), _p(out["evecs"]), _p(out["sweeps"]),
                     _p(out["offdiag"]), _p(out["status"]), nthreads)
    return out


def residuals(A, lam, d, dim: int = 3):
    """residuals (oracle.py:144-161) -> [n, dim + 2] = (recon_rel, ortho,
    eigvec_res...)."""
    w = 3 if dim == 2 else 6
    A, lam, d = _c(A, width=w), _c(lam, width=dim), _c(d, width=dim * dim)
    out = np.empty((A.shape[0], dim + 2))
    lib().sdo_residuals(dim, _p(A), _p(lam), _p(d), A.shape[0], _p(out))
    return out


def eig3_nudged(A, mode: int, seed: int = 0, nthreads: int = 1, report: bool = False):
    """eig3 with every libm result of the hot path moved by one ulp (mode 1
    up, 2 down, 3 random direction per call, seeded) — the reference's own
    sensitivity to 1-ulp libm differences."""
    lib().sdo_set_nudge(mode, seed)
    try:
        return eig3(A, nthreads=nthreads, report=report)
    finally:
        lib().sdo_set_nudge(0, 0)


def py_hypot(x: float, y: float) -> float:
    return lib().sdo_py_hypot(x, y)
