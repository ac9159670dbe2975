"""Drop-in `symdiag.oracle` names (/root/reference/pkg/src/symdiag/oracle.py),
computed by the GPU referee kernels (sd_jacobi.cuh): cyclic Jacobi,
bracketed cubic roots and decomposition residuals.  They share no code with
the closed-form solver, which is what makes them referees.

Scalar calls are n = 1 launches; use `batched.jacobi_batched`,
`batched.residuals_batched`, `batched.cubic_roots_batched` for throughput.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib, batched
from .core import SymMat2, SymMat3

MAX_SWEEPS = 100              # oracle.py:18
DOUBLE_ROOT_POLY_EPS = 1e-11  # oracle.py:20


class NoConvergence(RuntimeError):
    """Jacobi failed to converge (oracle.py:23-24)."""


class ComplexRootsDetected(ValueError):
    """The cubic is not real-rooted (oracle.py:27-29)."""


@dataclass(frozen=True)
class JacobiResult:
    eigenvalues: np.ndarray
    eigenvectors: np.ndarray
    sweeps: int
    offdiag_final: float


def _dev():
    _lib.require_cuda()
    return torch.device("cuda", torch.cuda.current_device())


def _packed(a):
    """SymMat2 / SymMat3 / symmetric ndarray -> (dim, packed row)."""
    if isinstance(a, SymMat2):
        return 2, a.packed()
    if isinstance(a, SymMat3):
        return 3, a.packed()
    m = np.asarray(a, dtype=float)
    if m.shape == (2, 2):
        return 2, (m[0, 0], m[0, 1], m[1, 1])
    if m.shape == (3, 3):
        return 3, (m[0, 0], m[0, 1], m[0, 2], m[1, 1], m[1, 2], m[2, 2])
    raise ValueError("expected a 2x2 or 3x3 symmetric matrix")


def jacobi_eigen(a, tol=1e-13) -> JacobiResult:
    """Cyclic-by-row Jacobi (oracle.py:45-84) on the GPU."""
    if tol <= 0.0:
        raise ValueError("tol must be positive")
    dim, row = _packed(a)
    A = torch.tensor([row], dtype=torch.float64, device=_dev())
    r = batched.jacobi_batched(A, dim=dim, tol=tol)
    st = int(r.status[0].item())
    if st == 1:
        raise NoConvergence(f"no convergence after {MAX_SWEEPS} sweeps")
    if st != 0:
        from .core import NonFiniteInput
        raise NonFiniteInput("non-finite matrix entry")
    return JacobiResult(eigenvalues=r.evals[0].cpu().numpy(),
                        eigenvectors=r.evecs[0].cpu().numpy(),
                        sweeps=int(r.sweeps[0].item()),
                        offdiag_final=float(r.offdiag[0].item()))


def cubic_roots_reference(coeffs):
    """Three real roots of l^3 - b l^2 + c l + d (oracle.py:87-133)."""
    bcd = torch.tensor([[coeffs.b, coeffs.c, coeffs.d]], dtype=torch.float64, device=_dev())
    roots, st = batched.cubic_roots_batched(bcd)
    if int(st[0].item()):
        raise ComplexRootsDetected("cubic has complex roots")
    return tuple(roots[0].tolist())


def reconstruct(d, lambdas):
    """D diag(lambdas) D^T for a decomposition candidate (oracle.py:136-141)."""
    d = np.asarray(d, dtype=float)
    if float(np.linalg.norm(d.T @ d - np.eye(d.shape[0]))) > 1e-10:
        raise ValueError("d is not orthogonal within 1e-10")
    return d @ np.diag(lambdas) @ d.T


def residuals(a, dec):
    """(recon_rel, ortho, [eigvec_res...]) of a decomposition (oracle.py:144-161)."""
    dim, row = _packed(a)
    lam = (dec.lambda1, dec.lambda2, dec.lambda3) if dim == 3 else (dec.lambda1, dec.lambda2)
    dev = _dev()
    out = batched.residuals_batched(
        torch.tensor([row], dtype=torch.float64, device=dev),
        torch.tensor([lam], dtype=torch.float64, device=dev),
        torch.as_tensor(np.asarray(dec.d, dtype=float).reshape(1, dim * dim)).to(dev),
        dim=dim)[0].tolist()
    return out[0], out[1], out[2:]
