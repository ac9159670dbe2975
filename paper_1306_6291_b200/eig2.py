"""Drop-in `symdiag.eig2` API (/root/reference/pkg/src/symdiag/eig2.py),
computed by the B200 2x2 kernel (n = 1 launches; use
batched.diagonalize2_batched for throughput)."""

from __future__ import annotations

import numpy as np

from . import batched, status as S
from .core import EigenDecomp2, SymMat2

DEGENERACY_EPS = 1e-14  # eig2.py:14


def _run(a: SymMat2, with_d=False):
    """One synchronous host-buffer call (sd_eig2_report_f64_host)."""
    st, lam, phi, d = batched.eig2_report_scalar(a.packed())
    if (st & S.CODE_MASK) >= S.ERR_FIRST:
        S.raise_for(st, "diagonalize2")
    return lam, phi, d


def eigenvalues2(a: SymMat2):
    """(lambda1, lambda2), lambda1 on the sign(a11 - a22) branch (eig2.py:22-26)."""
    l1, l2 = _run(a)[0]
    return l1, l2


def rotation_angle2(a: SymMat2):
    """Eigenvector angle in (-pi/2, pi/2] (eig2.py:29-41)."""
    return _run(a)[1]


def diagonalize2(a: SymMat2) -> EigenDecomp2:
    """A = D diag(l1, l2) D^T (eig2.py:44-48)."""
    lam, phi, d = _run(a, with_d=True)
    l1, l2 = lam
    return EigenDecomp2(lambda1=l1, lambda2=l2, phi=phi, d=np.array(d).reshape(2, 2))
