"""Drop-in `symdiag.eig3` API (/root/reference/pkg/src/symdiag/eig3.py).

Same names, signatures, return types and exceptions as the reference; every
computation is one launch of the B200 kernels (batched.py) with n = 1.
For throughput, call `batched.diagonalize3_batched` on millions of rows.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib, batched, status as S
from .core import Angles3, Branch, EigenDecomp3, SolveReport, SymMat3

F_ZERO_EPS = 1e-14      # eig3.py:34
DEGENERATE_EPS = 1e-12  # eig3.py:36
V_ZERO_EPS = 1e-12      # eig3.py:38
CLAMP_SLACK = 1e-9      # eig3.py:41
TIE_EPS = 1e-12         # eig3.py:43
NEAR_TIE_EPS = 1e-6     # eig3.py:45


class DegenerateEigenvalues(ValueError):
    """An eigenvalue gap needed by the generic branch is numerically zero."""


class BothFVectorsZero(ValueError):
    """f1 = f2 = 0: the matrix is diagonal with two equal diagonal entries."""


class NotDoubleRoot(ValueError):
    """degenerate_double was called with all three eigenvalues equal."""


class DomainExcursion(ValueError):
    """A squared cosine left [0, 1] beyond slack."""


@dataclass(frozen=True)
class CubicCoeffs:
    """l^3 - b l^2 + c l + d = 0 (eig3.py:65-75)."""

    b: float
    c: float
    d: float

    def scale(self):
        return max(1.0, math.sqrt(max(self.b * self.b - 2.0 * self.c, 0.0)))


@dataclass(frozen=True)
class PQ:
    """p, q and the arccos angle delta (None near p = 0) (eig3.py:78-84)."""

    p: float
    q: float
    delta: float | None = None


_BRANCH = {S.GENERIC: Branch.GENERIC, S.ALREADY_DIAGONAL_2D: Branch.ALREADY_DIAGONAL_2D,
           S.DOUBLE_ROOT: Branch.DOUBLE_ROOT, S.TRIPLE_ROOT: Branch.TRIPLE_ROOT}


def _dev():
    _lib.require_cuda()
    return torch.device("cuda", torch.cuda.current_device())


def _t(rows, width):
    return torch.tensor(np.asarray(rows, dtype=np.float64).reshape(-1, width),
                        dtype=torch.float64, device=_dev())


def _a(a: SymMat3):
    return _t([a.packed()], 6)


def _check(st, where):
    c = int(st) & S.CODE_MASK
    if c >= S.STAGE_DEGENERATE_EIGENVALUES:
        S.raise_for(c, where)


def _report_from_row(st: int, rep: np.ndarray) -> SolveReport:
    nc = int(rep[3]) if not math.isnan(rep[3]) else 0
    cands = tuple((int(rep[4 + 5 * k]), int(rep[5 + 5 * k]), float(rep[6 + 5 * k]),
                   float(rep[7 + 5 * k]), float(rep[8 + 5 * k])) for k in range(nc))
    s2 = -1 if st & S.FLAG_S2_NEG else 1
    s3 = -1 if st & S.FLAG_S3_NEG else 1
    return SolveReport(selected_signs=(s2, s3), phi1_candidates=cands,
                       f1_norm=float(rep[0]), f2_norm=float(rep[1]),
                       recon_residual=float(rep[2]), near_tie=bool(st & S.FLAG_NEAR_TIE))


def char_coeffs(a: SymMat3) -> CubicCoeffs:
    bcd, st = batched.char_coeffs_batched(_a(a))
    _check(st[0].item(), "char_coeffs")
    b, c, d = bcd[0].tolist()
    return CubicCoeffs(b=b, c=c, d=d)


def pq_expanded(a: SymMat3) -> tuple:
    pq, st = batched.pq_expanded_batched(_a(a))
    _check(st[0].item(), "pq_expanded")
    return tuple(pq[0].tolist())


def compute_pq(coeffs: CubicCoeffs) -> PQ:
    pqd, st = batched.compute_pq_batched(_t([(coeffs.b, coeffs.c, coeffs.d)], 3))
    _check(st[0].item(), "compute_pq")
    p, q, delta = pqd[0].tolist()
    return PQ(p=p, q=q, delta=None if math.isnan(delta) else delta)


def eigenvalues3(coeffs: CubicCoeffs, pq: PQ) -> tuple:
    delta = math.nan if pq.delta is None else pq.delta
    lam = batched.eigenvalues3_batched(_t([(coeffs.b, coeffs.c, coeffs.d)], 3),
                                       _t([(pq.p, pq.q, delta)], 3))
    return tuple(lam[0].tolist())


def compute_v(a: SymMat3, lambdas) -> float:
    v, st = batched.compute_v_batched(_a(a), _t([tuple(lambdas)], 3))
    _check(st[0].item(), "compute_v")
    return v[0].item()


def compute_w(a: SymMat3, lambdas, v) -> float:
    w, st = batched.compute_w_batched(_a(a), _t([tuple(lambdas)], 3), _t([v], 1))
    _check(st[0].item(), "compute_w")
    return w[0].item()


def f_vectors(a: SymMat3):
    f = batched.f_vectors_batched(_a(a))[0].tolist()
    return np.array(f[:2]), np.array(f[2:])


def g_vectors(lambdas, phi2, phi3, v, w):
    l1, l2, l3 = lambdas
    g = batched.g_vectors_batched(_t([(l1, l2, l3, phi2, phi3, v, w)], 7))[0].tolist()
    return np.array(g[:2]), np.array(g[2:])


def _angles_report(ang, st, rep, where):
    st = int(st[0].item())
    _check(st, where)
    return Angles3(*ang[0].tolist()), _report_from_row(st, rep[0].cpu().numpy())


def resolve_signs(a: SymMat3, lambdas, v, w):
    ang, st, rep = batched.resolve_signs_batched(_a(a), _t([tuple(lambdas)], 3), _t([(v, w)], 2))
    angles, report = _angles_report(ang, st, rep, "resolve_signs")
    return angles, SolveReport(selected_signs=report.selected_signs,
                               phi1_candidates=report.phi1_candidates,
                               f1_norm=report.f1_norm, f2_norm=report.f2_norm,
                               near_tie=report.near_tie)


def degenerate_double(a: SymMat3, lam, lam3):
    ang, st, rep = batched.degenerate_double_batched(_a(a), _t([(lam, lam3)], 2))
    angles, report = _angles_report(ang, st, rep, "degenerate_double")
    return angles, SolveReport(selected_signs=report.selected_signs,
                               phi1_candidates=report.phi1_candidates,
                               f1_norm=report.f1_norm, f2_norm=report.f2_norm,
                               near_tie=report.near_tie)


def diagonalize3(a: SymMat3) -> EigenDecomp3:
    """diagonalize3 (eig3.py:509-565) through the fused B200 kernel."""
    st, lam, ang, rep, d = batched.eig3_report_scalar(a.packed())  # one synchronous C call
    c = st & S.CODE_MASK
    if c >= S.ERR_FIRST:
        S.raise_for(c, "diagonalize3")
    l1, l2, l3 = lam
    return EigenDecomp3(lambda1=l1, lambda2=l2, lambda3=l3, angles=Angles3(*ang),
                        d=np.array(d).reshape(3, 3), branch=_BRANCH[c],
                        report=_report_from_row(st, rep))


def euler_angles(dec: EigenDecomp3) -> Angles3:
    """The Euler angles are the fixed-axis triple itself (eig3.py:568-576)."""
    return dec.angles
