// sd_jacobi.cuh — batched independent referees on the GPU:
// cyclic Jacobi (jacobi_eigen, oracle.py:45-84) and the decomposition
// residuals (residuals, oracle.py:144-161).
//
// Both follow numpy's evaluation order: every n x n matmul is the
// k-ascending FMA chain OpenBLAS produces (including the zero and unit
// entries of the rotation, so signed zeros and roundings agree), np.sum of
// the 9 squares is numpy's pairwise sum, math.hypot is CPython's.  The
// only intended difference from the reference is `x**2` in _offdiag_sq
// (numpy scalar power = glibc pow) evaluated as x*x.
#pragma once

#include "sd_math.cuh"

namespace sd {

template <int N>
__device__ __forceinline__ void mmn(const double* a, const double* b, double* c) {
#pragma unroll
  for (int i = 0; i < N; i++)
#pragma unroll
    for (int j = 0; j < N; j++) {
      double s = a[N * i] * b[j];
#pragma unroll
      for (int k = 1; k < N; k++) s = fma(a[N * i + k], b[N * k + j], s);
      c[N * i + j] = s;
    }
}

template <int N>
__device__ __forceinline__ double np_sum_sq(const double* m) {
  double a[N * N];
#pragma unroll
  for (int k = 0; k < N * N; k++) a[k] = m[k] * m[k];
  if (N * N < 8) {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < N * N; k++) s += a[k];
    return s;
  }
  double r = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
#pragma unroll
  for (int k = 8; k < N * N; k++) r += a[k];
  return r;
}

template <int N>
__device__ __forceinline__ double offdiag_sq(const double* m) {
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < N; i++)
#pragma unroll
    for (int j = i + 1; j < N; j++) s = s + m[N * i + j] * m[N * i + j];
  return s;
}

// one Jacobi rotation on (p, q): m = J^T m J, v = v J (oracle.py:67-81)
template <int N, int P, int Q>
__device__ __forceinline__ void jacobi_rotate(double* m, double* v) {
  const double apq = m[N * P + Q];
  if (apq == 0.0) return;
  const double theta = 0.5 * (m[N * Q + Q] - m[N * P + P]) / apq;
  const double t = copysign(1.0, theta) / (fabs(theta) + py_hypot(theta, 1.0));
  const double c = 1.0 / py_hypot(t, 1.0);
  const double s = t * c;
  double j[N * N], jt[N * N], t1[N * N];
#pragma unroll
  for (int k = 0; k < N * N; k++) j[k] = (k % (N + 1) == 0) ? 1.0 : 0.0;
  j[N * P + P] = c;
  j[N * Q + Q] = c;
  j[N * P + Q] = s;
  j[N * Q + P] = -s;
#pragma unroll
  for (int a = 0; a < N; a++)
#pragma unroll
    for (int b = 0; b < N; b++) jt[N * a + b] = j[N * b + a];
  mmn<N>(jt, m, t1);
  mmn<N>(t1, j, m);
  mmn<N>(v, j, t1);
#pragma unroll
  for (int k = 0; k < N * N; k++) v[k] = t1[k];
}

constexpr int kJacobiMaxSweeps = 100;  // oracle.py:18

// jacobi_eigen for one full symmetric matrix; returns 0, or 1 (NoConvergence)
template <int N>
__device__ __forceinline__ int jacobi(double* m, double tol, double* v, int& sweeps,
                                      double& offdiag) {
#pragma unroll
  for (int k = 0; k < N * N; k++) v[k] = (k % (N + 1) == 0) ? 1.0 : 0.0;
  const double thresh = tol * tol * pmax(1.0, np_sum_sq<N>(m));
  sweeps = 0;
  int rc = 0;
  while (offdiag_sq<N>(m) > thresh) {
    if (sweeps >= kJacobiMaxSweeps) {
      rc = 1;
      break;
    }
    if (N == 2) {
      jacobi_rotate<N, 0, 1>(m, v);
    } else {
      jacobi_rotate<N, 0, 1>(m, v);
      jacobi_rotate<N, 0, N - 1>(m, v);
      jacobi_rotate<N, N - 2, N - 1>(m, v);
    }
    sweeps++;
  }
  offdiag = sqrt(offdiag_sq<N>(m));
  return rc;
}

// residuals (oracle.py:144-161): out = (recon_rel, ortho, eigvec_res[N])
template <int N>
__device__ __forceinline__ void residuals(const double* m, const double* lam, const double* d,
                                          double* out) {
  double fro2;
  if (N == 2)
    fro2 = m[0] * m[0] + m[3] * m[3] + 2.0 * (m[1] * m[1]);
  else
    fro2 = m[0] * m[0] + m[4] * m[4] + m[8] * m[8] +
           2.0 * (m[1] * m[1] + m[2] * m[2] + m[5] * m[5]);
  const double scale = pmax(1.0, sqrt(fro2));
  double dg[N * N], t1[N * N], dt[N * N], rec[N * N];
#pragma unroll
  for (int k = 0; k < N * N; k++) dg[k] = 0.0;
#pragma unroll
  for (int k = 0; k < N; k++) dg[N * k + k] = lam[k];
#pragma unroll
  for (int a = 0; a < N; a++)
#pragma unroll
    for (int b = 0; b < N; b++) dt[N * a + b] = d[N * b + a];
  mmn<N>(d, dg, t1);
  mmn<N>(t1, dt, rec);
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < N * N; k++) {
    const double x = rec[k] - m[k];
    s = fma(x, x, s);
  }
  out[0] = sqrt(s) / scale;
  mmn<N>(dt, d, t1);
  s = 0.0;
#pragma unroll
  for (int k = 0; k < N * N; k++) {
    const double y = t1[k] - ((k % (N + 1) == 0) ? 1.0 : 0.0);
    s = fma(y, y, s);
  }
  out[1] = sqrt(s);
#pragma unroll
  for (int c = 0; c < N; c++) {
    double r2 = 0.0;
#pragma unroll
    for (int r = 0; r < N; r++) {
      double mv = m[N * r] * d[c];
#pragma unroll
      for (int k = 1; k < N; k++) mv = fma(m[N * r + k], d[N * k + c], mv);
      const double y = mv - lam[c] * d[N * r + c];
      r2 = fma(y, y, r2);
    }
    out[2 + c] = sqrt(r2) / scale;
  }
}

// cubic_roots_reference (oracle.py:87-133): the three real roots of
// l^3 - b l^2 + c l + d by bracketing at the critical points (b +- sqrt p)/3.
// The reference refines each bracket with scipy brentq (xtol 1e-15,
// rtol 4 eps); here each bracket is bisected to adjacent doubles (at most
// 1100 steps, ~60 in practice), which lands within the same tolerance.
// Returns 0, or 1 = ComplexRootsDetected (oracle.py:102-105, :116-117).
__device__ __forceinline__ double cubic_poly(double b, double c, double d, double x) {
  return ((x - b) * x + c) * x + d;  // oracle.py:97-98
}

__device__ __forceinline__ double bisect_root(double b, double c, double d, double lo,
                                              double hi) {
  double flo = cubic_poly(b, c, d, lo);
  const double fhi = cubic_poly(b, c, d, hi);
  if (flo == 0.0) return lo;
  if (fhi == 0.0) return hi;
  for (int it = 0; it < 1100; it++) {
    const double mid = lo + 0.5 * (hi - lo);
    if (!(mid > lo && mid < hi)) break;  // adjacent doubles
    const double fm = cubic_poly(b, c, d, mid);
    if (fm == 0.0) return mid;
    if ((fm < 0.0) == (flo < 0.0)) {
      lo = mid;
      flo = fm;
    } else {
      hi = mid;
    }
  }
  return (fabs(cubic_poly(b, c, d, lo)) <= fabs(cubic_poly(b, c, d, hi))) ? lo : hi;
}

__device__ __forceinline__ int cubic_roots(double b, double c, double d, double r[3]) {
  const double s = pmax(1.0, sqrt(pmax(b * b - 2.0 * c, 0.0)));  // CubicCoeffs.scale
  double p = b * b - 3.0 * c;
  if (p < -1e-12 * s * s) return 1;
  p = pmax(p, 0.0);
  const double t = 1e-12 * s;
  if (p <= 9.0 * (t * t)) {
    r[0] = r[1] = r[2] = b / 3.0;
    return 0;
  }
  const double sp = sqrt(p);
  const double x_lo = (b - sp) / 3.0;  // local maximum
  const double x_hi = (b + sp) / 3.0;  // local minimum
  const double f_lo = cubic_poly(b, c, d, x_lo);
  const double f_hi = cubic_poly(b, c, d, x_hi);
  const double ptol = 1e-11 * (s * s * s);
  if (f_lo < -ptol || f_hi > ptol) return 1;
  const double margin = pmax(1e-8 * s, 1e-8 * sp);
  const double lo = (b - 2.0 * sp) / 3.0 - margin;
  const double hi = (b + 2.0 * sp) / 3.0 + margin;
  if (fabs(f_lo) <= ptol) {  // double root at the local maximum
    r[0] = r[1] = x_lo;
    r[2] = bisect_root(b, c, d, x_hi, hi);
    return 0;
  }
  if (fabs(f_hi) <= ptol) {
    r[0] = bisect_root(b, c, d, lo, x_lo);
    r[1] = r[2] = x_hi;
    return 0;
  }
  r[0] = bisect_root(b, c, d, lo, x_lo);
  r[1] = bisect_root(b, c, d, x_lo, x_hi);
  r[2] = bisect_root(b, c, d, x_hi, hi);
  return 0;
}

}  // namespace sd
