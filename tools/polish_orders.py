#!/usr/bin/env python3
"""Find/verify the operation orders of numpy's small linear algebra on this
host (numpy 2.3 + scipy-openblas 0.3.30, Haswell kernels), used by the
reference's polish and residuals (eig3.py:463-489, oracle.py:144-161):

  j.T @ j  (9x3)       -> syrk: per entry a k-ascending FMA chain
  j.T @ r  (9-vector)  -> dgemv_n, 3-row / lda==3 tail: t += fma(a_k, x_k,
                          a_{k+1} x_{k+1}) per column pair in blocks of four,
                          then t = fma(a_8, x_8, t)
  m @ v    (3x3, 2x2)  -> dgemv_t small-m tail: fma(a2, x2, fma(a0, x0, a1 x1))
  np.linalg.solve 3x3  -> OpenBLAS getf2 + getrs (see oracle/symdiag_oracle.c
                          solve3)

Each candidate is compiled from the C below and compared with numpy on
random inputs; prints the match counts.  The oracle restates the winning
orders; tests/test_oracle_pin.py then pins the oracle's polished rows and
residuals bit for bit against the reference's own golden outputs.
"""
import ctypes
import subprocess
import tempfile
from pathlib import Path

import numpy as np

SRC = r"""
#include <math.h>
#include <float.h>
void syrk(const double* J, double* o) {
  for (int i = 0; i < 3; i++) for (int j = 0; j < 3; j++) {
    double s = J[i] * J[j];
    for (int k = 1; k < 9; k++) s = fma(J[3*k+i], J[3*k+j], s);
    o[3*i+j] = s; } }
void jtr(const double* J, const double* r, double* o) {
  for (int i = 0; i < 3; i++) { double t = 0.0; int k = 0;
    for (; k + 4 <= 9; k += 4) for (int h = 0; h < 4; h += 2)
      t = t + fma(J[3*(k+h)+i], r[k+h], J[3*(k+h+1)+i] * r[k+h+1]);
    for (; k < 9; k++) t = fma(J[3*k+i], r[k], t);
    o[i] = t; } }
void mv3(const double* m, const double* v, double* o) {
  for (int j = 0; j < 3; j++) { const double* a = m + 3*j;
    o[j] = fma(a[2], v[2], fma(a[0], v[0], a[1]*v[1])); } }
void solve(const double* M, const double* v, double* x) {
  double a[9]; for (int i = 0; i < 3; i++) for (int j = 0; j < 3; j++) a[i+3*j] = M[3*i+j];
  int ipiv[3];
  for (int j = 0; j < 3; j++) { double* b = a + 3*j;
    for (int i = 0; i < j; i++) { int jp = ipiv[i]; if (jp != i) { double t = b[i]; b[i] = b[jp]; b[jp] = t; } }
    for (int i = 1; i < j; i++) { double t = 0.0; for (int k = 0; k < i; k++) t = fma(b[k], a[i+3*k], t); b[i] = b[i] - t; }
    for (int r = j; r < 3; r++) { double t = 0.0; for (int k = 0; k < j; k++) t = fma(a[r+3*k], b[k], t); b[r] = fma(-1.0, t, b[r]); }
    int jp = j; double best = fabs(b[j]);
    for (int r = j+1; r < 3; r++) if (fabs(b[r]) > best) { best = fabs(b[r]); jp = r; }
    ipiv[j] = jp; double piv = b[jp];
    if (piv != 0.0) {
      if (jp != j) for (int k = 0; k <= j; k++) { double t = a[j+3*k]; a[j+3*k] = a[jp+3*k]; a[jp+3*k] = t; }
      if (fabs(piv) >= DBL_MIN) { double rp = 1.0 / piv; for (int r = j+1; r < 3; r++) b[r] *= rp; }
      else for (int r = j+1; r < 3; r++) b[r] /= piv; } }
  double y[3] = {v[0], v[1], v[2]};
  for (int i = 0; i < 3; i++) { int jp = ipiv[i]; if (jp != i) { double t = y[i]; y[i] = y[jp]; y[jp] = t; } }
  for (int i = 0; i < 3; i++) for (int k = i+1; k < 3; k++) y[k] = fma(-y[i], a[k+3*i], y[k]);
  for (int i = 2; i >= 0; i--) { y[i] = y[i] / a[i+3*i]; for (int k = 0; k < i; k++) y[k] = fma(-y[i], a[k+3*i], y[k]); }
  x[0] = y[0]; x[1] = y[1]; x[2] = y[2]; }
"""


def main(n=5000, seed=0):
    d = Path(tempfile.mkdtemp())
    (d / "c.c").write_text(SRC)
    subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-shared", "-fPIC", "-o", str(d / "c.so"),
                    str(d / "c.c"), "-lm"], check=True)
    L = ctypes.CDLL(str(d / "c.so"))
    p = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    rng = np.random.default_rng(seed)
    ok = dict(syrk=0, jtr=0, mv3=0, solve=0)
    for t in range(n):
        J = np.ascontiguousarray(rng.standard_normal((9, 3)) * 10.0 ** rng.integers(-3, 3))
        r = rng.standard_normal(9)
        o = np.empty(9); L.syrk(p(J), p(o)); ok["syrk"] += np.array_equal(o.reshape(3, 3), J.T @ J)
        o = np.empty(3); L.jtr(p(J), p(r), p(o)); ok["jtr"] += np.array_equal(o, J.T @ r)
        m, dd = rng.standard_normal((3, 3)), rng.standard_normal((3, 3))
        v = np.ascontiguousarray(dd[:, 1])
        o = np.empty(3); L.mv3(p(np.ascontiguousarray(m)), p(v), p(o)); ok["mv3"] += np.array_equal(o, m @ dd[:, 1])
        M = J.T @ J + 1e-14 * np.eye(3) if t % 2 else rng.standard_normal((3, 3))
        o = np.empty(3); L.solve(p(np.ascontiguousarray(M)), p(r[:3].copy()), p(o))
        ok["solve"] += np.array_equal(o, np.linalg.solve(M, r[:3]))
    print({k: f"{v}/{n}" for k, v in ok.items()})
    return ok


if __name__ == "__main__":
    main()
