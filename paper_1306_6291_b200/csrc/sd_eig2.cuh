// sd_eig2.cuh — device-side 2x2 closed-form diagonalization
// (/root/reference/pkg/src/symdiag/eig2.py, cited as eig2.py:line).
#pragma once

#include "sd_math.cuh"

namespace sd {

constexpr double DEGENERACY_EPS_2 = 1e-14;  // eig2.py:14

// diagonalize2 (eig2.py:44-48) = eigenvalues2 (eig2.py:22-26) +
// rotation_angle2 (eig2.py:29-41); _sign(0) = +1 (eig2.py:17-19).
__device__ __forceinline__ uint8_t diagonalize2(double a11, double a12, double a22, double& l1,
                                                double& l2, double& phi) {
  if (!(is_finite(a11) && is_finite(a12) && is_finite(a22))) {
    l1 = l2 = phi = qnan();
    return SD_ERR_NONFINITE_INPUT;  // SymMat2 construction (core.py:62-63)
  }
  Err e;
  const double dd = a11 - a22;
  const double t = a11 + a22;
  const double sg = (dd < 0.0) ? -1.0 : 1.0;
  const double r = sg * py_hypot(dd, 2.0 * a12);
  // SymMat2.scale (core.py:68-73) gates the phi = 0 special case only
  // (eig2.py:37-39): eps = 1e-14 max(1, ||A||_F).  Its sqrt is needed only
  // when both |a11 - a22| and |a12| could be below eps, i.e. below
  // 1e-14 * sqrt(F) * (1 + 2^-40) — otherwise the gate is decided without it.
  const double fro2 = pow2(e, a11) + pow2(e, a22) + 2.0 * pow2(e, a12);
  const double m = pmax(fabs(dd), fabs(a12));
  bool zero_angle = false;
  if (m * m <= 1.0000000001e-28 * pmax(1.0, fro2) || m <= DEGENERACY_EPS_2) {
    const double eps = DEGENERACY_EPS_2 * pmax(1.0, py_sqrt(e, fro2));
    zero_angle = fabs(dd) <= eps && fabs(a12) <= eps;
  }
  double ph = 0.0;
  if (!zero_angle) {
    // wrap_half_pi of a value already in [-pi/2, pi/2]: remainder(x, pi) == x
    // exactly there, so only the -pi/2 -> pi/2 and -0 -> +0 rules remain
    ph = 0.5 * atan2(2.0 * a12 * sg, dd * sg);
    if (ph <= -0.5 * kPi) ph = 0.5 * kPi;
    if (ph == 0.0) ph = 0.0;
  }
  if (e.code) {
    l1 = l2 = phi = qnan();
    return (uint8_t)e.code;
  }
  l1 = 0.5 * (t + r);
  l2 = 0.5 * (t - r);
  phi = ph;
  return SD_CODE_GENERIC;
}

__device__ __noinline__ uint8_t diagonalize2_literal(double a11, double a12, double a22,
                                                     double& l1, double& l2, double& phi) {
  return diagonalize2(a11, a12, a22, l1, l2, phi);
}

// ---- fast 2x2 path -----------------------------------------------------------
// Same outputs as diagonalize2 above on every row it accepts, with the FP64
// work cut from ~135 to ~50 pipe instructions per row (the 2x2 kernel was
// FP64-pipe-bound, ncu 60% pipe busy at 2.6 IPC):
//  * range and gate decisions on integer exponent fields (ALU pipe);
//  * math.hypot: the same scaled operands as CPython's vector_norm, their
//    squares summed exactly (double-double), sqrt via rsqrt.approx + one
//    cubic Newton step and one FMA correction of the double-double residual.
//    Result = the correctly rounded hypot of the scaled operands except
//    within ~2^-60 ulp of a rounding midpoint; CPython's result is the same
//    value under the same condition (its differential correction), so lambda
//    stays bit-identical to the reference outside those measure-zero cases;
//  * 0.5*atan2(y, x) with x = |a11 - a22| >= 0 (eig2.py:41): the half-angle
//    identity tan(theta/2) = b / (a + hypot(a, b)) on the octant-reduced
//    pair (a, b) = (max, min) of (x, |y|) gives |phi| = atan(w) or
//    pi/4 - atan(w) with w in [0, tan(pi/8)], reusing the hypot just
//    computed: one reciprocal and a degree-10 minimax polynomial in w^2
//    (tools/fit_atan.py, 0.61 ulp) instead of libdevice's division, 20-term
//    polynomial and quadrant fix-ups.  |phi| <= pi/4, so wrap_half_pi
//    (core.py:37-47) reduces to -0 -> +0.
// Rows it declines (non-finite or |a_ij| >= 2^500, hypot operands below
// 2^-1021, or a possible phi = 0 gate hit) return false for the literal path.
#ifndef SD_EIG2_LITERAL
#define SD_EIG2_LITERAL 0
#endif

__device__ __forceinline__ double rsqrt_approx(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}
__device__ __forceinline__ double rcp_approx(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}
__device__ __forceinline__ uint64_t dbits(double x) { return (uint64_t)__double_as_longlong(x); }
// |x| as bits on the integer pipe (a plain mask is turned back into an
// FP64-pipe DADD |x| by the compiler)
__device__ __forceinline__ uint64_t abs_bits(double x) {
  uint64_t r;
  asm("and.b64 %0, %1, 0x7fffffffffffffff;" : "=l"(r) : "l"(dbits(x)));
  return r;
}
__device__ __forceinline__ double bdouble(uint64_t b) { return __longlong_as_double((long long)b); }

// atan(w) = w + w s P(s), s = w^2, w in [0, tan(pi/8)]: minimax P of degree
// 10 (tools/fit_atan.py: |P - f| <= 3.0e-17, atan within 0.61 ulp)
__device__ __forceinline__ double atan_oct(double w) {
  const double s = w * w;
  double p = -0.019228204970831376;
  p = fma(p, s, 0.03927572279035204);
  p = fma(p, s, -0.050870579623365775);
  p = fma(p, s, 0.05858473913774763);
  p = fma(p, s, -0.06664551143049129);
  p = fma(p, s, 0.07692186192120325);
  p = fma(p, s, -0.09090904716299451);
  p = fma(p, s, 0.11111111018911234);
  p = fma(p, s, -0.14285714284715656);
  p = fma(p, s, 0.19999999999995777);
  p = fma(p, s, -0.3333333333333333);
  return fma(w * s, p, w);
}

// SD_EIG2_NULL (diagnostics, tools/eig2_variants.py): 1 = no arithmetic
// (the kernel's memory time alone), 2 = eigenvalues only (no angle)
#ifndef SD_EIG2_NULL
#define SD_EIG2_NULL 0
#endif
__device__ __forceinline__ bool diagonalize2_fast(double a11, double a12, double a22, double& l1,
                                                  double& l2, double& phi) {
#if SD_EIG2_NULL == 1
  l1 = a11;
  l2 = a22;
  phi = a12;
  return true;
#endif
  // Branch-free: the range tests only set `ok` (a declined row computes
  // garbage that the caller discards), so several rows' chains interleave.
  const uint32_t h11 = (uint32_t)__double2hiint(a11) & 0x7fffffffu;
  const uint32_t h12 = (uint32_t)__double2hiint(a12) & 0x7fffffffu;
  const uint32_t h22 = (uint32_t)__double2hiint(a22) & 0x7fffffffu;
  const uint32_t hmax = max(max(h11, h12), h22);
  bool ok = hmax < 0x5f300000u;  // finite, |a| < 2^500 (no square overflows)
  const double dd = a11 - a22;
  const double t = a11 + a22;
  const double y = a12 + a12;  // 2.0 * a12, exact
  const uint64_t bd = dbits(dd);
  const uint64_t X = abs_bits(dd), AY = abs_bits(y);
  const bool neg = X != bd && X != 0;  // dd < 0.0
  const uint64_t mx = max(X, AY), mn = min(X, AY);
  ok &= mx >= 0x0020000000000000ull;  // hypot's subnormal / zero cases
  // phi = 0 gate (eig2.py:37-39): certainly not taken when
  // max(|dd|, |a12|) >= 2^-44 * 2^e(max(1, max|a|)) > 2.0002e-14 max(1, ||A||_F)
  const uint64_t m = max(X, abs_bits(a12));
  ok &= (uint32_t)(m >> 52) + 44u >= (max(hmax, 0x3ff00000u) >> 20);

  // hypot(dd, 2 a12) on CPython's scaled operands P >= q (scale = 2^-e)
  const uint32_t ex = (uint32_t)(mx >> 52) & 0x7ffu;  // biased; 2^(ex-1022) > mx >= 2^(ex-1023)
  const double scale = bdouble((uint64_t)((2045u - ex) & 0x7ffu) << 52);
  const double inv = bdouble((uint64_t)((ex + 1u) & 0x7ffu) << 52);
  const double P = bdouble(mx) * scale, q = bdouble(mn) * scale;
  const double hp = P * P, lp = fma(P, P, -hp);
  const double hq = q * q, lq = fma(q, q, -hq);
  const double s = hp + hq;
  const double lo = (lp + lq) + (hq - (s - hp));  // s + lo = P^2 + q^2 (to 2^-105)
  const double y0 = rsqrt_approx(s);            // s in [0.25, 2)
  const double e1 = fma(-(s * y0), y0, 1.0);
  const double y1 = fma(y0 * e1, fma(e1, 0.375, 0.5), y0);
  const double h0 = s * y1;
  const double h = fma(fma(-h0, h0, s) + lo, 0.5 * y1, h0);
  const double R = h * inv;
  const double r = neg ? -R : R;
  l1 = 0.5 * (t + r);
  l2 = 0.5 * (t - r);

#if SD_EIG2_NULL == 2
  phi = q;
  return ok;
#endif
  // phi = 0.5 atan2(2 a12 sg, |dd|), sg = sign(dd)
  const double D = P + h;  // in [1, 1 + 2^0.5]
  const double r0 = rcp_approx(D);
  double e = fma(-D, r0, 1.0);
  e = fma(e, e, e);
  const double rd = fma(r0, e, r0);
  const double w0 = q * rd;
  const double w = fma(rd, fma(-D, w0, q), w0);
  const double at = atan_oct(w);
  const double a = (AY > X) ? (0.7853981633974483 - at) + 3.061616997868383e-17 : at;  // pi/4 - at
  const bool ysign = (dbits(y) >> 63) != 0;
  phi = (a == 0.0) ? 0.0 : ((ysign != neg) ? -a : a);
  return ok;
}

}  // namespace sd
