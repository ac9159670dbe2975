// sd_eig3.cuh — device-side 3x3 closed-form diagonalization (arXiv 1306.6291)
// with the reference's branch, sign, ordering and exception semantics
// (/root/reference/pkg/src/symdiag/eig3.py, cited as eig3.py:line).
//
// One thread owns one matrix; everything lives in registers.  The functions
// below are the stage functions of the reference, each usable on its own
// (the stage-level C-ABI entry points launch them directly) and fused by
// diagonalize3() into the single-pass hot kernel.
#pragma once

#include "sd_math.cuh"

namespace sd {

constexpr double F_ZERO_EPS = 1e-14;     // eig3.py:34
constexpr double DEGENERATE_EPS = 1e-12; // eig3.py:36
constexpr double V_ZERO_EPS = 1e-12;     // eig3.py:38
constexpr double CLAMP_SLACK = 1e-9;     // eig3.py:41
constexpr double TIE_EPS = 1e-12;        // eig3.py:43
constexpr double NEAR_TIE_EPS = 1e-6;    // eig3.py:45

struct Sym3 {
  double a11, a22, a33, a12, a13, a23;
};

// packed (a11, a12, a13, a22, a23, a33)
__device__ __forceinline__ Sym3 unpack3(const double* p) {
  Sym3 a;
  a.a11 = p[0];
  a.a12 = p[1];
  a.a13 = p[2];
  a.a22 = p[3];
  a.a23 = p[4];
  a.a33 = p[5];
  return a;
}

__device__ __forceinline__ bool finite3(const Sym3& a) {
  return is_finite(a.a11) && is_finite(a.a22) && is_finite(a.a33) && is_finite(a.a12) &&
         is_finite(a.a13) && is_finite(a.a23);
}

// SymMat3.fro_norm / scale (core.py:107-112)
__device__ __forceinline__ double sym3_scale(Err& e, const Sym3& a) {
  double f = py_sqrt(e, pow2(e, a.a11) + pow2(e, a.a22) + pow2(e, a.a33) +
                            2.0 * (pow2(e, a.a12) + pow2(e, a.a13) + pow2(e, a.a23)));
  return pmax(1.0, f);
}

// char_coeffs (eig3.py:102-109), Python's left-to-right association
__device__ __forceinline__ void char_coeffs(Err& e, const Sym3& a, double& b, double& c,
                                            double& d) {
  b = a.a11 + a.a22 + a.a33;
  c = a.a11 * a.a22 + a.a11 * a.a33 + a.a22 * a.a33 - pow2(e, a.a12) - pow2(e, a.a13) -
      pow2(e, a.a23);
  d = a.a11 * pow2(e, a.a23) + a.a22 * pow2(e, a.a13) + a.a33 * pow2(e, a.a12) -
      a.a11 * a.a22 * a.a33 - 2.0 * a.a12 * a.a13 * a.a23;
}

// pq_expanded (eig3.py:112-126)
__device__ __forceinline__ void pq_expanded(Err& e, const Sym3& a, double& p, double& q) {
  double off2 = pow2(e, a.a12) + pow2(e, a.a13) + pow2(e, a.a23);
  p = 0.5 * (pow2(e, a.a11 - a.a22) + pow2(e, a.a11 - a.a33) + pow2(e, a.a22 - a.a33)) +
      3.0 * off2;
  q = 18.0 * (a.a11 * a.a22 * a.a33 + 3.0 * a.a12 * a.a13 * a.a23) +
      2.0 * (pow3(e, a.a11) + pow3(e, a.a22) + pow3(e, a.a33)) +
      9.0 * (a.a11 + a.a22 + a.a33) * off2 -
      3.0 * (a.a11 + a.a22) * (a.a11 + a.a33) * (a.a22 + a.a33) -
      27.0 * (a.a11 * pow2(e, a.a23) + a.a22 * pow2(e, a.a13) + a.a33 * pow2(e, a.a12));
}

// compute_pq (eig3.py:129-156); has_delta == false encodes delta=None.
// Thresholds: CubicCoeffs.scale (eig3.py:73-75), triple_root_threshold
// (eig3.py:87-89), discriminant_threshold (eig3.py:92-99).
__device__ __forceinline__ void compute_pq(Err& e, double b, double c, double d, double& p,
                                           double& q, double& delta, bool& has_delta) {
  double s = pmax(1.0, py_sqrt(e, pmax(b * b - 2.0 * c, 0.0)));
  p = b * b - 3.0 * c;
  q = 2.0 * pow3(e, b) - 9.0 * b * c - 27.0 * d;
  has_delta = false;
  delta = qnan();
  if (p < 0.0) {
    if (p < -1e-12 * pmax(1.0, b * b + fabs(c))) {
      e.raise(SD_ERR_P_NEGATIVE);
      return;
    }
    p = 0.0;
  }
  double t = 1e-12 * s;
  if (p <= 9.0 * pow2(e, t)) return;
  double p3 = pow3(e, p);
  if (4.0 * p3 - q * q <= 1e-12 * pow6(e, s)) {
    has_delta = true;
    delta = (q >= 0.0) ? 0.0 : kPi;
    return;
  }
  double arg = q / (2.0 * py_sqrt(e, p3));
  if (fabs(arg) > 1.0) {
    if (fabs(arg) > 1.0 + CLAMP_SLACK) {
      e.raise(SD_ERR_ACOS_SLACK);
      return;
    }
    arg = (arg > 0.0) ? 1.0 : -1.0;
  }
  has_delta = true;
  delta = py_acos(e, arg);
}

// eigenvalues3 (eig3.py:159-174): lambda1 >= lambda3 >= lambda2
__device__ __forceinline__ void eigenvalues3(Err& e, double b, double p, double delta,
                                             bool has_delta, double l[3]) {
  if (!has_delta) {
    double lam = b / 3.0;
    l[0] = l[1] = l[2] = lam;
    return;
  }
  double sp2 = 2.0 * py_sqrt(e, p);
  double third = delta / 3.0;
  const double two_pi_3 = 2.0 * kPi / 3.0;
  l[0] = (b + sp2 * py_cos(e, third)) / 3.0;
  l[1] = (b + sp2 * py_cos(e, third + two_pi_3)) / 3.0;
  l[2] = (b + sp2 * py_cos(e, third - two_pi_3)) / 3.0;
}

// _clamp_unit (eig3.py:177-180)
__device__ __forceinline__ double clamp_unit(Err& e, double x, double slack) {
  if (x < -slack || x > 1.0 + slack) {
    e.raise(SD_ERR_DOMAIN_EXCURSION);
    return qnan();
  }
  return pmin(pmax(x, 0.0), 1.0);
}

__device__ __forceinline__ double lam_tol(const double l[3]) {
  double m = pmax(1.0, fabs(l[0]));
  m = pmax(m, fabs(l[1]));
  m = pmax(m, fabs(l[2]));
  return DEGENERATE_EPS * m;
}

// compute_v (eig3.py:183-195)
__device__ __forceinline__ double compute_v(Err& e, const Sym3& a, const double l[3]) {
  double tol = lam_tol(l);
  if (fabs(l[1] - l[2]) <= tol || fabs(l[2] - l[0]) <= tol) {
    e.raise(SD_STAGE_DEGENERATE_EIGENVALUES);
    return qnan();
  }
  double num = pow2(e, a.a12) + pow2(e, a.a13) + (a.a11 - l[2]) * (a.a11 + l[2] - l[0] - l[1]);
  return clamp_unit(e, num / ((l[1] - l[2]) * (l[2] - l[0])), CLAMP_SLACK);
}

// compute_w (eig3.py:198-206)
__device__ __forceinline__ double compute_w(Err& e, const Sym3& a, const double l[3], double v) {
  if (v <= V_ZERO_EPS) return 1.0;
  double tol = lam_tol(l);
  if (fabs(l[0] - l[1]) <= tol) {
    e.raise(SD_STAGE_DEGENERATE_EIGENVALUES);
    return qnan();
  }
  return clamp_unit(e, (a.a11 - l[2] + (l[2] - l[1]) * v) / ((l[0] - l[1]) * v), CLAMP_SLACK);
}

// _rotated_angle (eig3.py:228-230): angle of R(-psi) g
__device__ __forceinline__ double rotated_angle(Err& e, double cp, double sp, double gx,
                                                double gy) {
  return angle_of(e, cp * gx + sp * gy, -sp * gx + cp * gy);
}

// _phi1_candidates (eig3.py:233-245)
__device__ __forceinline__ void phi1_candidates(Err& e, double n1, double n2, double tol_f,
                                                double c1x, double c1y, double c2x, double c2y,
                                                double g1x, double g1y, double g2x, double g2y,
                                                double& p11, double& p12) {
  p11 = (n1 > tol_f && (g1x != 0.0 || g1y != 0.0)) ? rotated_angle(e, c1x, c1y, g1x, g1y)
                                                    : qnan();
  p12 = (n2 > tol_f && (g2x != 0.0 || g2y != 0.0)) ? 0.5 * rotated_angle(e, c2x, c2y, g2x, g2y)
                                                    : qnan();
}

// Result of the angle stage (resolve_signs / degenerate_double).
template <bool kReport>
struct AngleOut {
  double phi[3];
  int s2 = 1, s3 = 1;
  bool near_tie = false;
  double n1 = 0.0, n2 = 0.0;
  int ncand = 0;
  double cand[kReport ? 4 : 1][5];
};

// candidate selection (eig3.py:313-324, :433-442): first scored combo within
// TIE_EPS of the minimum; near_tie if the best other one is within
// (TIE_EPS, NEAR_TIE_EPS]; combo 0 if none is scored.
template <int N>
__device__ __forceinline__ int select_candidate(const double diff[N], bool& near_tie) {
  double best = 0.0;
  bool any = false;
#pragma unroll
  for (int k = 0; k < N; k++)
    if (!is_nan(diff[k])) {
      if (!any || diff[k] < best) best = diff[k];
      any = true;
    }
  near_tie = false;
  if (!any) return 0;
  int sel = -1;
#pragma unroll
  for (int k = N - 1; k >= 0; k--)
    if (!is_nan(diff[k]) && diff[k] <= best + TIE_EPS) sel = k;
  bool have_other = false;
  double mo = 0.0;
#pragma unroll
  for (int k = 0; k < N; k++)
    if (k != sel && !is_nan(diff[k])) {
      if (!have_other || diff[k] < mo) mo = diff[k];
      have_other = true;
    }
  if (have_other) {
    double gap = mo - diff[sel];
    near_tie = (TIE_EPS < gap) && (gap <= NEAR_TIE_EPS);
  }
  return sel;
}

// _assemble_angles (eig3.py:248-266) + Angles3 normalisation (core.py:115-132)
template <bool kReport>
__device__ __forceinline__ void assemble_angles(Err& e, double n1, double n2, double p11,
                                                double p12, int s2, int s3, double phi2_mag,
                                                double phi3_mag, AngleOut<kReport>& out) {
  double phi1;
  if (is_nan(p11))
    phi1 = is_nan(p12) ? 0.0 : p12;
  else if (is_nan(p12))
    phi1 = p11;
  else
    phi1 = (n1 >= n2) ? p11 : p12;
  if (!is_nan(p11) && (p11 > 0.5 * kPi || p11 <= -0.5 * kPi)) {
    s2 = -s2;
    s3 = -s3;
  }
  double a2 = (double)s2 * phi2_mag, a3 = (double)s3 * phi3_mag;
  if (!is_finite(phi1) || !is_finite(a2) || !is_finite(a3)) e.raise(SD_ERR_NONFINITE_INPUT);
  out.phi[0] = wrap_half_pi(e, phi1);
  out.phi[1] = wrap_half_pi(e, a2);
  out.phi[2] = wrap_half_pi(e, a3);
  out.s2 = s2;
  out.s3 = s3;
}

// resolve_signs (eig3.py:269-386).  `scale` = SymMat3.scale() (the caller
// has it already; eig3.py:279 recomputes the same value).
template <bool kReport>
__device__ __forceinline__ void resolve_signs(Err& e, const Sym3& a, double scale,
                                              const double l[3], double v, double w,
                                              AngleOut<kReport>& out) {
  double tol_f = F_ZERO_EPS * scale;
  double f1x = a.a12, f1y = -a.a13;
  double f2x = a.a22 - a.a33, f2y = -2.0 * a.a23;
  double n1 = py_hypot(f1x, f1y);
  double n2 = py_hypot(f2x, f2y);
  out.n1 = n1;
  out.n2 = n2;
  if (n1 <= tol_f && n2 <= tol_f) {
    e.raise(SD_STAGE_BOTH_F_ZERO);
    return;
  }
  double phi2_mag = py_acos(e, py_sqrt(e, clamp_unit(e, v, CLAMP_SLACK)));
  double phi3_mag = py_acos(e, py_sqrt(e, clamp_unit(e, w, CLAMP_SLACK)));
  if (e.code) return;
  double c1x = 1.0, c1y = 0.0, c2x = 1.0, c2y = 0.0;
  if (n1 > tol_f) {
    c1x = f1x / n1;
    c1y = f1y / n1;
  }
  if (n2 > tol_f) {
    c2x = f2x / n2;
    c2y = f2y / n2;
  }
  const double l1 = l[0], l2 = l[1], l3 = l[2];
  double c2, s2m, s3x2;
  py_sincos(e, phi2_mag, &s2m, &c2);
  s3x2 = py_sin(e, 2.0 * phi3_mag);
  double s2x2 = 2.0 * s2m * c2;
  double g1y_mag = 0.5 * ((l1 - l2) * w + l2 - l3) * s2x2;
  double g1x_mag = 0.5 * (l1 - l2) * c2 * s3x2;
  double g2x = (l1 - l2) * (1.0 + (v - 2.0) * w) + (l2 - l3) * v;
  double g2y_mag = (l1 - l2) * s2m * s3x2;

  // the four sign combinations (+,+), (+,-), (-,+), (-,-) (eig3.py:302-311)
  double p11k[4], p12k[4], diff[4];
  const bool both = n1 > tol_f && n2 > tol_f;
#pragma unroll
  for (int k = 0; k < 4; k++) {
    const double s2 = (k < 2) ? 1.0 : -1.0;
    const double s3 = (k & 1) ? -1.0 : 1.0;
    phi1_candidates(e, n1, n2, tol_f, c1x, c1y, c2x, c2y, s3 * g1x_mag, s2 * g1y_mag, g2x,
                    (s2 * s3) * g2y_mag, p11k[k], p12k[k]);
    diff[k] = both ? wrapped_diff(e, p11k[k], p12k[k]) : qnan();
  }
  if (e.code) return;
  bool near_tie;
  int sel = select_candidate<4>(diff, near_tie);
  out.near_tie = near_tie;
  if (kReport) {
    out.ncand = 4;
#pragma unroll
    for (int k = 0; k < 4; k++) {
      out.cand[k][0] = (k < 2) ? 1.0 : -1.0;
      out.cand[k][1] = (k & 1) ? -1.0 : 1.0;
      out.cand[k][2] = p11k[k];
      out.cand[k][3] = p12k[k];
      out.cand[k][4] = diff[k];
    }
  }
  int s2 = (sel < 2) ? 1 : -1;
  int s3 = (sel & 1) ? -1 : 1;
  double p11 = p11k[0], p12 = p12k[0];
#pragma unroll
  for (int k = 1; k < 4; k++)
    if (sel == k) {
      p11 = p11k[k];
      p12 = p12k[k];
    }

  // refinement (eig3.py:328-379)
  if (n1 > tol_f) {
    const double gap12 = l1 - l2;
    const double gap23 = l2 - l3;
    for (int it = 0; it < 2; it++) {
      double phi1_est = (is_nan(p11) || (n2 > n1 && !is_nan(p12))) ? p12 : p11;
      if (is_nan(phi1_est)) break;
      double s1, c1, s1d, c1d;
      py_sincos(e, phi1_est, &s1, &c1);
      py_sincos(e, 2.0 * phi1_est, &s1d, &c1d);
      double hx = c1 * f1x - s1 * f1y;
      double hy = s1 * f1x + c1 * f1y;
      double h2x = c1d * f2x - s1d * f2y;
      double h2y = s1d * f2x + c1d * f2y;
      if (phi3_mag < 0.125 * kPi || phi3_mag > 0.375 * kPi) {
        double den_a = fabs(0.5 * gap12 * c2);
        double den_b = fabs(gap12 * s2m);
        const double inf = __longlong_as_double(0x7ff0000000000000LL);
        double k_a = (den_a > 0.0) ? fabs(hy) / (2.0 * den_a) : inf;
        double k_b = (n2 > tol_f && den_b > 0.0) ? fabs(h2x) / den_b : inf;
        double est = inf;
        if (k_a <= pmin(k_b, 0.5))
          est = hx / (0.5 * gap12 * c2);
        else if (k_b <= 0.5)
          est = h2y / (gap12 * s2m);
        if (is_finite(est)) {
          double half = 0.5 * py_asin(e, pmin(fabs(est), 1.0));
          phi3_mag = (phi3_mag <= 0.25 * kPi) ? half : 0.5 * kPi - half;
          w = pow2(e, py_cos(e, phi3_mag));
        }
      }
      if (phi2_mag < 0.125 * kPi || phi2_mag > 0.375 * kPi) {
        double den = 0.5 * (gap12 * w + gap23);
        if (fabs(den) > 0.0 && fabs(hx) / (2.0 * fabs(den)) <= 0.5) {
          double half = 0.5 * py_asin(e, pmin(fabs(hy / den), 1.0));
          phi2_mag = (phi2_mag <= 0.25 * kPi) ? half : 0.5 * kPi - half;
          v = pow2(e, py_cos(e, phi2_mag));
        }
      }
      py_sincos(e, phi2_mag, &s2m, &c2);
      s3x2 = py_sin(e, 2.0 * phi3_mag);
      s2x2 = 2.0 * s2m * c2;
      double g1x = (double)s3 * 0.5 * gap12 * c2 * s3x2;
      double g1y = (double)s2 * 0.5 * (gap12 * w + gap23) * s2x2;
      double g2xx = gap12 * (1.0 + (v - 2.0) * w) + gap23 * v;
      double g2y = (double)(s2 * s3) * gap12 * s2m * s3x2;
      phi1_candidates(e, n1, n2, tol_f, c1x, c1y, c2x, c2y, g1x, g1y, g2xx, g2y, p11, p12);
    }
  }
  if (e.code) return;
  assemble_angles(e, n1, n2, p11, p12, s2, s3, phi2_mag, phi3_mag, out);
}

// degenerate_double (eig3.py:389-454)
template <bool kReport>
__device__ __forceinline__ void degenerate_double(Err& e, const Sym3& a, double scale,
                                                  double lam, double lam3,
                                                  AngleOut<kReport>& out) {
  if (fabs(lam - lam3) <= DEGENERATE_EPS * scale) {
    e.raise(SD_ERR_NOT_DOUBLE_ROOT);
    return;
  }
  double s = clamp_unit(e, (a.a11 - lam3) / (lam - lam3), 1e-5);
  if (e.code) return;
  double phi2_mag = py_acos(e, py_sqrt(e, s));
  double tol_f = F_ZERO_EPS * scale;
  double f1x = a.a12, f1y = -a.a13;
  double f2x = a.a22 - a.a33, f2y = -2.0 * a.a23;
  double n1 = py_hypot(f1x, f1y);
  double n2 = py_hypot(f2x, f2y);
  out.n1 = n1;
  out.n2 = n2;
  if (phi2_mag < 0.125 * kPi || phi2_mag > 0.375 * kPi) {
    double sin2 = pmin(2.0 * n1 / fabs(lam - lam3), 1.0);
    double half = 0.5 * py_asin(e, sin2);
    phi2_mag = (phi2_mag <= 0.25 * kPi) ? half : 0.5 * kPi - half;
    s = pow2(e, py_cos(e, phi2_mag));
  }
  double c1x = 1.0, c1y = 0.0, c2x = 1.0, c2y = 0.0;
  if (n1 > tol_f) {
    c1x = f1x / n1;
    c1y = f1y / n1;
  }
  if (n2 > tol_f) {
    c2x = f2x / n2;
    c2y = f2y / n2;
  }
  double g1y_mag = 0.5 * (lam - lam3) * py_sin(e, 2.0 * phi2_mag);
  double g2x = (lam - lam3) * s;
  double p11k[2], p12k[2], diff[2];
  const bool both = n1 > tol_f && n2 > tol_f;
#pragma unroll
  for (int k = 0; k < 2; k++) {
    const double s2 = k == 0 ? 1.0 : -1.0;
    phi1_candidates(e, n1, n2, tol_f, c1x, c1y, c2x, c2y, 0.0, s2 * g1y_mag, g2x, 0.0, p11k[k],
                    p12k[k]);
    diff[k] = both ? wrapped_diff(e, p11k[k], p12k[k]) : qnan();
  }
  if (e.code) return;
  bool near_tie;
  int sel = select_candidate<2>(diff, near_tie);
  out.near_tie = near_tie;
  if (kReport) {
    out.ncand = 2;
#pragma unroll
    for (int k = 0; k < 2; k++) {
      out.cand[k][0] = k == 0 ? 1.0 : -1.0;
      out.cand[k][1] = 1.0;
      out.cand[k][2] = p11k[k];
      out.cand[k][3] = p12k[k];
      out.cand[k][4] = diff[k];
    }
  }
  const int s2 = sel == 0 ? 1 : -1;
  if (n1 <= tol_f && n2 <= tol_f) {
    out.phi[0] = 0.0;
    out.phi[1] = wrap_half_pi(e, (double)s2 * phi2_mag);
    out.phi[2] = 0.0;
    out.s2 = s2;
    out.s3 = 1;
  } else {
    assemble_angles(e, n1, n2, sel == 0 ? p11k[0] : p11k[1], sel == 0 ? p12k[0] : p12k[1], s2,
                    1, phi2_mag, 0.0, out);
  }
}

// _double_root_lambdas (eig3.py:492-501)
__device__ __forceinline__ void double_root_lambdas(double l[3]) {
  double g0 = fabs(l[0] - l[1]), g1 = fabs(l[0] - l[2]), g2 = fabs(l[1] - l[2]);
  double m = g0;
  if (g1 < m) m = g1;
  if (g2 < m) m = g2;
  double lam, lam3;
  if (g0 == m) {
    lam = 0.5 * (l[0] + l[1]);
    lam3 = l[2];
  } else if (g1 == m) {
    lam = 0.5 * (l[0] + l[2]);
    lam3 = l[1];
  } else {
    lam = 0.5 * (l[1] + l[2]);
    lam3 = l[0];
  }
  l[0] = l[1] = lam;
  l[2] = lam3;
}

// ---- compose_rotation, residual, polish (core.py:229-235, eig3.py:458-506)
// numpy's 3x3 matmul (OpenBLAS) accumulates k-ascending with FMA; the same
// chains are used here so the 1e-12 polish gate sees the same residual.
__device__ __forceinline__ void mm3(const double* a, const double* b, double* c) {
#pragma unroll
  for (int i = 0; i < 3; i++)
#pragma unroll
    for (int j = 0; j < 3; j++)
      c[3 * i + j] = fma(a[3 * i + 2], b[6 + j], fma(a[3 * i + 1], b[3 + j], a[3 * i] * b[j]));
}

// D = rot3x(p1) rot3y(p2) rot3z(p3), evaluated as numpy does ((Rx Ry) Rz)
// kLit = false: libdevice's sincos instead of the literal solver's
// correctly rounded one (the polish pass's gate, whose outcome the parity
// rules check through the residual, not bit for bit)
template <bool kLit = true>
__device__ __forceinline__ void compose_rotation(Err& e, const double phi[3], double d[9]) {
  double s1, c1, s2, c2, s3, c3;
  if (kLit) {
    py_sincos(e, phi[0], &s1, &c1);
    py_sincos(e, phi[1], &s2, &c2);
    py_sincos(e, phi[2], &s3, &c3);
  } else {
    sincos(phi[0], &s1, &c1);
    sincos(phi[1], &s2, &c2);
    sincos(phi[2], &s3, &c3);
  }
  const double rx[9] = {1.0, 0.0, 0.0, 0.0, c1, -s1, 0.0, s1, c1};
  const double ry[9] = {c2, 0.0, s2, 0.0, 1.0, 0.0, -s2, 0.0, c2};
  const double rz[9] = {c3, -s3, 0.0, s3, c3, 0.0, 0.0, 0.0, 1.0};
  double t[9];
  mm3(rx, ry, t);
  mm3(t, rz, d);
}

// ||(D diag(lam)) D^T - A||_F (np.linalg.norm = sequential FMA dot)
__device__ __forceinline__ double abs_residual(const double d[9], const double lam[3],
                                               const Sym3& a) {
  double dl[9], dt[9], r[9];
#pragma unroll
  for (int i = 0; i < 3; i++)
#pragma unroll
    for (int j = 0; j < 3; j++) {
      dl[3 * i + j] = d[3 * i + j] * lam[j];
      dt[3 * i + j] = d[3 * j + i];
    }
  mm3(dl, dt, r);
  const double am[9] = {a.a11, a.a12, a.a13, a.a12, a.a22, a.a23, a.a13, a.a23, a.a33};
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 9; k++) {
    double x = r[k] - am[k];
    s = fma(x, x, s);
  }
  return sqrt(s);
}

// numpy's j.T @ r for j[9][3] (OpenBLAS 0.3.30 dgemv_n, 3-row lda==3 tail:
// column pairs in blocks of four, then the last column), bit for bit as
// oracle/symdiag_oracle.c jt_resid (tools/polish_orders.py)
__device__ __forceinline__ void jt_resid_ob(const double J[9][3], const double r[9], double out[3]) {
#pragma unroll
  for (int i = 0; i < 3; i++) {
    double t = 0.0;
#pragma unroll
    for (int k = 0; k < 8; k += 2) t = t + fma(J[k][i], r[k], J[k + 1][i] * r[k + 1]);
    out[i] = fma(J[8][i], r[8], t);
  }
}

// np.linalg.solve for 3x3, one right-hand side: OpenBLAS's dgesv (getf2:
// left-looking LU, reciprocal-scaled multipliers; getrs: laswp + column
// axpys + divisions), bit for bit as oracle/symdiag_oracle.c solve3
__device__ __forceinline__ void solve3_ob(const double m[9], const double rhs[3], double x[3]) {
  double a[9];  // column-major
#pragma unroll
  for (int i = 0; i < 3; i++)
#pragma unroll
    for (int j = 0; j < 3; j++) a[i + 3 * j] = m[3 * i + j];
  int ipiv[3];
#pragma unroll
  for (int j = 0; j < 3; j++) {
    double* b = a + 3 * j;
#pragma unroll
    for (int i = 0; i < j; i++) {
      const int jp = ipiv[i];
      if (jp != i) {
        const double t = b[i];
        b[i] = b[jp];
        b[jp] = t;
      }
    }
#pragma unroll
    for (int i = 1; i < j; i++) {
      double t = 0.0;
#pragma unroll
      for (int k = 0; k < i; k++) t = fma(b[k], a[i + 3 * k], t);
      b[i] = b[i] - t;
    }
#pragma unroll
    for (int r = j; r < 3; r++) {
      double t = 0.0;
#pragma unroll
      for (int k = 0; k < j; k++) t = fma(a[r + 3 * k], b[k], t);
      b[r] = fma(-1.0, t, b[r]);
    }
    int jp = j;
    double best = fabs(b[j]);
#pragma unroll
    for (int r = j + 1; r < 3; r++)
      if (fabs(b[r]) > best) {
        best = fabs(b[r]);
        jp = r;
      }
    ipiv[j] = jp;
    const double piv = b[jp];
    if (piv != 0.0) {
      if (jp != j)
#pragma unroll
        for (int k = 0; k <= j; k++) {
          const double t = a[j + 3 * k];
          a[j + 3 * k] = a[jp + 3 * k];
          a[jp + 3 * k] = t;
        }
      if (fabs(piv) >= 0x1p-1022) {
        const double rp = 1.0 / piv;
#pragma unroll
        for (int r = j + 1; r < 3; r++) b[r] = b[r] * rp;
      } else {
#pragma unroll
        for (int r = j + 1; r < 3; r++) b[r] = b[r] / piv;
      }
    }
  }
  double y[3] = {rhs[0], rhs[1], rhs[2]};
#pragma unroll
  for (int i = 0; i < 3; i++) {
    const int jp = ipiv[i];
    if (jp != i) {
      const double t = y[i];
      y[i] = y[jp];
      y[jp] = t;
    }
  }
#pragma unroll
  for (int i = 0; i < 3; i++)
#pragma unroll
    for (int k = i + 1; k < 3; k++) y[k] = fma(-y[i], a[k + 3 * i], y[k]);
#pragma unroll
  for (int i = 2; i >= 0; i--) {
    y[i] = y[i] / a[i + 3 * i];
#pragma unroll
    for (int k = 0; k < i; k++) y[k] = fma(-y[i], a[k + 3 * i], y[k]);
  }
  x[0] = y[0];
  x[1] = y[1];
  x[2] = y[2];
}

// _polish_angles (eig3.py:463-489): two damped Gauss-Newton steps on the
// angles, keeping the best.  Rare (0.02% of N(0,1), ~10% of the degenerate
// config), so it is kept out of line to spare the hot path's registers.
__device__ __noinline__ double polish_angles(const Sym3& a, const double* lam, double* phis,
                                             double scale) {
  Err e;
  double d[9], rec[9];
  const double am[9] = {a.a11, a.a12, a.a13, a.a12, a.a22, a.a23, a.a13, a.a23, a.a33};
  auto recon = [&](const double* dd, double* r) {
    double dl[9], dt[9];
#pragma unroll
    for (int i = 0; i < 3; i++)
#pragma unroll
      for (int j = 0; j < 3; j++) {
        dl[3 * i + j] = dd[3 * i + j] * lam[j];
        dt[3 * i + j] = dd[3 * j + i];
      }
    mm3(dl, dt, r);
  };
  auto fro = [&](const double* r) {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 9; k++) {
      double x = r[k] - am[k];
      s = fma(x, x, s);
    }
    return sqrt(s);
  };
  compose_rotation(e, phis, d);
  recon(d, rec);
  double best = fro(rec);
  double bp0 = phis[0], bp1 = phis[1], bp2 = phis[2];
  const double damp = 1e-14 * scale * scale;
  double cur[3] = {phis[0], phis[1], phis[2]};
  const double G1[9] = {0, 0, 0, 0, 0, -1, 0, 1, 0};
  const double G2[9] = {0, 0, 1, 0, 0, 0, -1, 0, 0};
  const double G3[9] = {0, -1, 0, 1, 0, 0, 0, 0, 0};
#pragma unroll 1
  for (int it = 0; it < 2; it++) {
    double s1, c1, s2, c2;
    lit_sincos(cur[0], &s1, &c1);
    lit_sincos(cur[1], &s2, &c2);
    const double r1[9] = {1.0, 0.0, 0.0, 0.0, c1, -s1, 0.0, s1, c1};
    const double ry[9] = {c2, 0.0, s2, 0.0, 1.0, 0.0, -s2, 0.0, c2};
    double r12[9], r1t[9], r12t[9], t[9], g2[9], g3[9];
    mm3(r1, ry, r12);
#pragma unroll
    for (int i = 0; i < 3; i++)
#pragma unroll
      for (int j = 0; j < 3; j++) {
        r1t[3 * i + j] = r1[3 * j + i];
        r12t[3 * i + j] = r12[3 * j + i];
      }
    mm3(r1, G2, t);
    mm3(t, r1t, g2);
    mm3(r12, G3, t);
    mm3(t, r12t, g3);
    double J[9][3];
#pragma unroll
    for (int c = 0; c < 3; c++) {
      const double* g = c == 0 ? G1 : (c == 1 ? g2 : g3);
      double gr[9], rg[9];
      mm3(g, rec, gr);
      mm3(rec, g, rg);
#pragma unroll
      for (int k = 0; k < 9; k++) J[k][c] = gr[k] - rg[k];
    }
    double jtj[9], jtr[3], x[3];
#pragma unroll
    for (int i = 0; i < 3; i++)
#pragma unroll
      for (int j = 0; j < 3; j++) {
        double s = J[0][i] * J[0][j];
#pragma unroll
        for (int k = 1; k < 9; k++) s = fma(J[k][i], J[k][j], s);
        jtj[3 * i + j] = s + (i == j ? damp : 0.0);
      }
    double resid[9];
#pragma unroll
    for (int k = 0; k < 9; k++) resid[k] = rec[k] - am[k];
    jt_resid_ob(J, resid, jtr);
    solve3_ob(jtj, jtr, x);
#pragma unroll
    for (int i = 0; i < 3; i++) cur[i] = cur[i] - x[i];
    compose_rotation(e, cur, d);
    recon(d, rec);
    double res = fro(rec);
    if (res < best) {
      best = res;
      bp0 = cur[0];
      bp1 = cur[1];
      bp2 = cur[2];
    }
  }
  phis[0] = bp0;
  phis[1] = bp1;
  phis[2] = bp2;
  return best;
}

// The tail of diagonalize3 (eig3.py:553-561) for a row whose closed-form
// (lam, phi) are known: literal residual, polish if above the gate, accept
// if better.  Returns true when the polished angles were accepted (phi
// updated).  Non-finite polished angles set phi[0] = NaN (NonFiniteInput is
// raised by Angles3 whether or not the polish is accepted, core.py:127).
__device__ __noinline__ bool polish_rows_literal(const Sym3& a, const double lam[3],
                                                 double phi[3]) {
  Err e;
  const double scale = sym3_scale(e, a);
  double d[9];
  compose_rotation(e, phi, d);
  const double recon_res = abs_residual(d, lam, a) / scale;
  if (!(recon_res > 1e-12)) return false;
  double phis[3] = {phi[0], phi[1], phi[2]};
  const double abs_res = polish_angles(a, lam, phis, scale);
  if (!is_finite(phis[0]) || !is_finite(phis[1]) || !is_finite(phis[2])) {
    phi[0] = qnan();
    return false;
  }
  if (abs_res / scale < recon_res) {
#pragma unroll
    for (int i = 0; i < 3; i++) phi[i] = wrap_half_pi(e, phis[i]);
    return true;
  }
  return false;
}

// ---- diagonalize3 (eig3.py:509-565) ---------------------------------------
template <bool kReport>
struct Result3 {
  double lam[3];
  double phi[3];
  uint8_t status;
  double recon;
  AngleOut<kReport> ar;
  double d[kReport ? 9 : 1];
};

template <bool kReport>
__device__ __forceinline__ void diagonalize3(const Sym3& a, Result3<kReport>& r) {
  Err e;
  AngleOut<kReport>& ar = r.ar;
  r.recon = qnan();
  int code = SD_CODE_GENERIC;
  if (!finite3(a)) {
    e.raise(SD_ERR_NONFINITE_INPUT);
  }
  double b = 0.0, c = 0.0, dd = 0.0, p = 0.0, q = 0.0, delta = 0.0;
  bool has_delta = false;
  double scale = 1.0;
  if (!e.code) char_coeffs(e, a, b, c, dd);
  if (!e.code) compute_pq(e, b, c, dd, p, q, delta, has_delta);
  if (!e.code) scale = sym3_scale(e, a);
  double lam[3] = {0.0, 0.0, 0.0};
  if (!e.code) {
    if (!has_delta) {
      // TripleRoot (eig3.py:521-528); report norms via np.hypot = libm hypot
      lam[0] = lam[1] = lam[2] = b / 3.0;
      ar.phi[0] = ar.phi[1] = ar.phi[2] = 0.0;
      if (kReport) {
        ar.n1 = lit_hypot(a.a12, -a.a13);
        ar.n2 = lit_hypot(a.a22 - a.a33, -2.0 * a.a23);
      }
      code = SD_CODE_TRIPLE_ROOT;
    } else {
      eigenvalues3(e, b, p, delta, has_delta, lam);
      double disc = 4.0 * pow3(e, p) - q * q;
      double thr = e.code ? 0.0 : 1e-12 * pow6(e, scale);
      if (!e.code && disc <= thr) {
        double_root_lambdas(lam);
        degenerate_double(e, a, scale, lam[0], lam[2], ar);
        code = SD_CODE_DOUBLE_ROOT;
      } else if (!e.code) {
        // generic try-block (eig3.py:538-551)
        Err t;
        double v = compute_v(t, a, lam);
        double w = 0.0;
        if (!t.code) w = compute_w(t, a, lam, v);
        if (!t.code) resolve_signs(t, a, scale, lam, v, w, ar);
        if (!t.code) {
          code = (ar.n1 <= F_ZERO_EPS * scale || ar.n2 <= F_ZERO_EPS * scale)
                     ? SD_CODE_ALREADY_DIAGONAL_2D
                     : SD_CODE_GENERIC;
        } else if (t.code == SD_STAGE_BOTH_F_ZERO || t.code == SD_STAGE_DEGENERATE_EIGENVALUES ||
                   t.code == SD_ERR_DOMAIN_EXCURSION) {
          double_root_lambdas(lam);
          ar = AngleOut<kReport>();
          degenerate_double(e, a, scale, lam[0], lam[2], ar);
          code = SD_CODE_DOUBLE_ROOT;
        } else {
          e.raise(t.code);  // not in the except tuple: propagates
        }
      }
    }
  }
  bool polished = false;
  double d[9];
  if (!e.code) {
    compose_rotation(e, ar.phi, d);
    double recon_res = abs_residual(d, lam, a) / scale;
    if (recon_res > 1e-12) {
      double phis[3] = {ar.phi[0], ar.phi[1], ar.phi[2]};
      double abs_res = polish_angles(a, lam, phis, scale);
      double wrapped[3];
#pragma unroll
      for (int i = 0; i < 3; i++)
        if (!is_finite(phis[i])) e.raise(SD_ERR_NONFINITE_INPUT);
#pragma unroll
      for (int i = 0; i < 3; i++) wrapped[i] = wrap_half_pi(e, phis[i]);
      if (!e.code && abs_res / scale < recon_res) {
#pragma unroll
        for (int i = 0; i < 3; i++) ar.phi[i] = wrapped[i];
        recon_res = abs_res / scale;
        if (kReport) compose_rotation(e, ar.phi, d);
        polished = true;
      }
    }
    r.recon = recon_res;
  }
  if (e.code) {
#pragma unroll
    for (int i = 0; i < 3; i++) r.lam[i] = r.phi[i] = qnan();
    r.status = (uint8_t)e.code;
    if (kReport) {
      ar.ncand = 0;
#pragma unroll
      for (int i = 0; i < 9; i++) r.d[i] = qnan();
    }
    return;
  }
#pragma unroll
  for (int i = 0; i < 3; i++) {
    r.lam[i] = lam[i];
    r.phi[i] = ar.phi[i];
  }
  if (kReport) {
#pragma unroll
    for (int i = 0; i < 9; i++) r.d[i] = d[i];
  }
  uint8_t st = (uint8_t)code;
  if (ar.s2 < 0) st |= SD_FLAG_S2_NEG;
  if (ar.s3 < 0) st |= SD_FLAG_S3_NEG;
  if (ar.near_tie) st |= SD_FLAG_NEAR_TIE;
  if (polished) st |= SD_FLAG_POLISHED;
  r.status = st;
}

}  // namespace sd
