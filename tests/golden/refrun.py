"""Run the UNMODIFIED reference (`symdiag`, imported in place from
/root/reference/pkg/src) over packed arrays and return its results in the
packed layouts of include/symdiag_b200.h.

Used only in this container: by make_golden.py to freeze the golden
fixtures, and by tests/test_oracle_pin.py's live leg when /root/reference
exists.  Nothing on the GPU box imports it.
"""

from __future__ import annotations

import math
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"

# status codes (include/symdiag_b200.h)
GENERIC, ALREADY_DIAGONAL_2D, DOUBLE_ROOT, TRIPLE_ROOT = 0, 1, 2, 3
STAGE_DEGENERATE, STAGE_BOTH_F_ZERO = 6, 7
NONFINITE, P_NEGATIVE, ACOS_SLACK, DOMAIN, NOT_DOUBLE, ZERO_VEC, MATH_DOMAIN, OVERFLOW = (
    8, 9, 10, 11, 12, 13, 14, 15)
S2_NEG, S3_NEG, NEAR_TIE, POLISHED = 0x10, 0x20, 0x40, 0x80
REPORT_STRIDE = 24


def available() -> bool:
    return os.path.isdir(REF_SRC)


def _import():
    os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
    sys.dont_write_bytecode = True
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import symdiag  # noqa: F401
    from symdiag import eig3, core
    return symdiag, eig3, core


def exc_code(e: BaseException) -> int:
    symdiag, eig3, core = _import()
    if isinstance(e, core.NonFiniteInput):
        return NONFINITE
    if isinstance(e, eig3.DomainExcursion):
        return DOMAIN
    if isinstance(e, eig3.NotDoubleRoot):
        return NOT_DOUBLE
    if isinstance(e, core.AngleOfZeroVector):
        return ZERO_VEC
    if isinstance(e, eig3.DegenerateEigenvalues):
        return STAGE_DEGENERATE
    if isinstance(e, eig3.BothFVectorsZero):
        return STAGE_BOTH_F_ZERO
    if isinstance(e, OverflowError):
        return OVERFLOW
    if isinstance(e, ValueError):
        msg = str(e)
        if msg.startswith("p = ") and "negative" in msg:
            return P_NEGATIVE
        if msg.startswith("arccos argument"):
            return ACOS_SLACK
        if "math domain error" in msg:
            return MATH_DOMAIN
    raise e


_BRANCH = None


def _branch_code(branch):
    global _BRANCH
    if _BRANCH is None:
        _, _, core = _import()
        _BRANCH = {core.Branch.GENERIC: GENERIC,
                   core.Branch.ALREADY_DIAGONAL_2D: ALREADY_DIAGONAL_2D,
                   core.Branch.DOUBLE_ROOT: DOUBLE_ROOT,
                   core.Branch.TRIPLE_ROOT: TRIPLE_ROOT}
    return _BRANCH[branch]


def sym3_from_packed(symdiag, row):
    a11, a12, a13, a22, a23, a33 = (float(x) for x in row)
    return symdiag.SymMat3(a11=a11, a22=a22, a33=a33, a12=a12, a13=a13, a23=a23)


def run_eig3(A: np.ndarray, with_d: bool = False):
    """diagonalize3 per row -> dict(lam, ang, status, report[, d])."""
    symdiag, eig3, core = _import()
    A = np.asarray(A, dtype=np.float64).reshape(-1, 6)
    n = A.shape[0]
    lam = np.full((n, 3), np.nan)
    ang = np.full((n, 3), np.nan)
    status = np.zeros(n, np.uint8)
    report = np.full((n, REPORT_STRIDE), np.nan)
    dmat = np.full((n, 9), np.nan)

    # observe the polish decision without changing behaviour
    state = {}
    orig_res = eig3._reconstruction_residual
    orig_pol = eig3._polish_angles

    def res_hook(a, d, lambdas):
        r = orig_res(a, d, lambdas)
        state.setdefault("first_res", r)
        return r

    def pol_hook(a_arr, lambdas, angles, scale):
        out = orig_pol(a_arr, lambdas, angles, scale)
        state["polish"] = (out[1], scale)
        return out

    eig3._reconstruction_residual = res_hook
    eig3._polish_angles = pol_hook
    try:
        for i in range(n):
            state.clear()
            try:
                m = sym3_from_packed(symdiag, A[i])
                dec = eig3.diagonalize3(m)
            except Exception as e:  # noqa: BLE001 — mapped to status codes
                status[i] = exc_code(e)
                report[i, 3] = 0.0
                continue
            lam[i] = dec.lambdas
            ang[i] = dec.angles.as_tuple()
            st = _branch_code(dec.branch)
            s2, s3 = dec.report.selected_signs
            if s2 < 0:
                st |= S2_NEG
            if s3 < 0:
                st |= S3_NEG
            if dec.report.near_tie:
                st |= NEAR_TIE
            if "polish" in state:
                abs_res, scale = state["polish"]
                if abs_res / scale < state["first_res"]:
                    st |= POLISHED
            status[i] = st
            rep = dec.report
            report[i, 0] = rep.f1_norm
            report[i, 1] = rep.f2_norm
            report[i, 2] = rep.recon_residual
            report[i, 3] = len(rep.phi1_candidates)
            for k, c in enumerate(rep.phi1_candidates):
                report[i, 4 + 5 * k: 9 + 5 * k] = c
            if with_d:
                dmat[i] = np.asarray(dec.d).reshape(9)
    finally:
        eig3._reconstruction_residual = orig_res
        eig3._polish_angles = orig_pol
    out = dict(lam=lam, ang=ang, status=status, report=report)
    if with_d:
        out["d"] = dmat
    return out


def run_eig2(A: np.ndarray, with_d: bool = False):
    symdiag, _, _ = _import()
    A = np.asarray(A, dtype=np.float64).reshape(-1, 3)
    n = A.shape[0]
    lam = np.full((n, 2), np.nan)
    phi = np.full(n, np.nan)
    status = np.zeros(n, np.uint8)
    dmat = np.full((n, 4), np.nan)
    for i in range(n):
        a11, a12, a22 = (float(x) for x in A[i])
        try:
            dec = symdiag.diagonalize2(symdiag.SymMat2(a11=a11, a22=a22, a12=a12))
        except Exception as e:  # noqa: BLE001
            status[i] = exc_code(e)
            continue
        lam[i] = (dec.lambda1, dec.lambda2)
        phi[i] = dec.phi
        dmat[i] = np.asarray(dec.d).reshape(4)
    out = dict(lam=lam, phi=phi, status=status)
    if with_d:
        out["d"] = dmat
    return out


def run_referees(A: np.ndarray, dim: int):
    """oracle.py referees: jacobi_eigen per row, and for 3x3 also
    cubic_roots_reference on char_coeffs and residuals of diagonalize3."""
    symdiag, eig3, core = _import()
    from symdiag import oracle as RO
    w = 3 if dim == 2 else 6
    A = np.asarray(A, dtype=np.float64).reshape(-1, w)
    n = A.shape[0]
    evals = np.full((n, dim), np.nan)
    evecs = np.full((n, dim * dim), np.nan)
    sweeps = np.zeros(n, np.int32)
    offdiag = np.full(n, np.nan)
    jstatus = np.zeros(n, np.uint8)
    roots = np.full((n, 3), np.nan)
    rstatus = np.zeros(n, np.uint8)
    resid = np.full((n, dim + 2), np.nan)
    for i in range(n):
        try:
            if dim == 2:
                m = symdiag.SymMat2(a11=float(A[i, 0]), a22=float(A[i, 2]), a12=float(A[i, 1]))
            else:
                m = sym3_from_packed(symdiag, A[i])
        except core.NonFiniteInput:
            jstatus[i] = rstatus[i] = NONFINITE
            continue
        try:
            r = RO.jacobi_eigen(m)
            evals[i], evecs[i] = r.eigenvalues, r.eigenvectors.reshape(-1)
            sweeps[i], offdiag[i] = r.sweeps, r.offdiag_final
        except RO.NoConvergence:
            jstatus[i] = 1
        if dim == 3:
            try:
                roots[i] = RO.cubic_roots_reference(eig3.char_coeffs(m))
            except RO.ComplexRootsDetected:
                rstatus[i] = 1
            except (OverflowError, ValueError):
                rstatus[i] = 2
            try:
                dec = eig3.diagonalize3(m)
                rr = RO.residuals(m, dec)
                resid[i] = [rr[0], rr[1], *rr[2]]
            except Exception:  # noqa: BLE001 — rows the solver rejects
                pass
        else:
            try:
                dec = symdiag.diagonalize2(m)
                rr = RO.residuals(m, dec)
                resid[i] = [rr[0], rr[1], *rr[2]]
            except Exception:  # noqa: BLE001 — rows the solver rejects
                pass
    return dict(evals=evals, evecs=evecs, sweeps=sweeps, offdiag=offdiag, jstatus=jstatus,
                roots=roots, rstatus=rstatus, resid=resid)


def run_stages(A: np.ndarray):
    """Stage-level reference outputs: char_coeffs, compute_pq, eigenvalues3,
    pq_expanded, compute_v/compute_w (with exception codes)."""
    symdiag, eig3, core = _import()
    A = np.asarray(A, dtype=np.float64).reshape(-1, 6)
    n = A.shape[0]
    bcd = np.full((n, 3), np.nan)
    cc_status = np.zeros(n, np.uint8)
    pqe_status = np.zeros(n, np.uint8)
    pqd = np.full((n, 3), np.nan)
    pq_status = np.zeros(n, np.uint8)
    lam = np.full((n, 3), np.nan)
    pqe = np.full((n, 2), np.nan)
    vw = np.full((n, 2), np.nan)
    vw_status = np.zeros(n, np.uint8)
    for i in range(n):
        try:
            m = sym3_from_packed(symdiag, A[i])
        except Exception as e:  # noqa: BLE001
            cc_status[i] = pqe_status[i] = pq_status[i] = vw_status[i] = exc_code(e)
            continue
        try:
            pqe[i] = eig3.pq_expanded(m)
        except Exception as e:  # noqa: BLE001
            pqe_status[i] = exc_code(e)
        try:
            c = eig3.char_coeffs(m)
        except Exception as e:  # noqa: BLE001
            cc_status[i] = pq_status[i] = vw_status[i] = exc_code(e)
            continue
        bcd[i] = (c.b, c.c, c.d)
        try:
            pq = eig3.compute_pq(c)
        except Exception as e:  # noqa: BLE001
            pq_status[i] = exc_code(e)
            continue
        pqd[i] = (pq.p, pq.q, math.nan if pq.delta is None else pq.delta)
        lams = eig3.eigenvalues3(c, pq)
        lam[i] = lams
        try:
            v = eig3.compute_v(m, lams)
            w = eig3.compute_w(m, lams, v)
            vw[i] = (v, w)
        except Exception as e:  # noqa: BLE001
            vw_status[i] = exc_code(e)
    return dict(bcd=bcd, cc_status=cc_status, pqd=pqd, pq_status=pq_status,
                lam=lam, pqe=pqe, pqe_status=pqe_status, vw=vw,
                vw_status=vw_status)


def _angles_record(i, angles, report, ang, status, rep):
    ang[i] = angles.as_tuple()
    s2, s3 = report.selected_signs
    st = 0
    if s2 < 0:
        st |= S2_NEG
    if s3 < 0:
        st |= S3_NEG
    if report.near_tie:
        st |= NEAR_TIE
    status[i] = st
    rep[i, 0] = report.f1_norm
    rep[i, 1] = report.f2_norm
    rep[i, 3] = len(report.phi1_candidates)
    for k, c in enumerate(report.phi1_candidates):
        rep[i, 4 + 5 * k: 9 + 5 * k] = c


def run_sign_stages(A: np.ndarray, lam: np.ndarray, vw: np.ndarray):
    """resolve_signs (eig3.py:269-386) on the rows whose (lam, v, w) are
    given (finite vw), and degenerate_double (eig3.py:389-454) on
    (lam, lam3) = _double_root_lambdas(lam) (eig3.py:492-501) for every row
    with finite lam.  Angles, status (sign / near-tie flags or the
    exception's code), report rows (f-norms, candidate tuples; the residual
    slot stays NaN, these stages do not compute it)."""
    symdiag, eig3, core = _import()
    A = np.asarray(A, dtype=np.float64).reshape(-1, 6)
    n = A.shape[0]
    out = {}
    for tag in ("rs", "dd"):
        out[f"{tag}_ang"] = np.full((n, 3), np.nan)
        out[f"{tag}_status"] = np.full(n, 255, np.uint8)  # 255: stage not run on this row
        out[f"{tag}_report"] = np.full((n, REPORT_STRIDE), np.nan)
        out[f"{tag}_report"][:, 3] = 0.0
    lam2 = np.full((n, 2), np.nan)
    for i in range(n):
        if not np.all(np.isfinite(lam[i])):
            continue
        m = sym3_from_packed(symdiag, A[i])
        lams = tuple(float(x) for x in lam[i])
        if np.all(np.isfinite(vw[i])):
            try:
                angles, report = eig3.resolve_signs(m, lams, float(vw[i, 0]), float(vw[i, 1]))
                _angles_record(i, angles, report, out["rs_ang"], out["rs_status"], out["rs_report"])
            except Exception as e:  # noqa: BLE001 — mapped to status codes
                out["rs_status"][i] = exc_code(e)
        lam2[i] = eig3._double_root_lambdas(lams)
        try:
            angles, report = eig3.degenerate_double(m, float(lam2[i, 0]), float(lam2[i, 1]))
            _angles_record(i, angles, report, out["dd_ang"], out["dd_status"], out["dd_report"])
        except Exception as e:  # noqa: BLE001
            out["dd_status"][i] = exc_code(e)
    out["lam2"] = lam2
    return out
