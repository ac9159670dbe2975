// sd_math.cuh — fp64 device arithmetic with the reference's (CPython +
// glibc) semantics, for sm_100a.
//
// The whole library is compiled with -fmad=false: like CPython, no a*b+c is
// ever contracted into an FMA unless written as fma() explicitly (SURVEY F4:
// one contraction in p = b*b - 3c flips 20% of near-triple branches).
//
// What is reproduced exactly, and how:
//   x**2, x**3, x**6 -> glibc 2.39's pow restated bit for bit
//                    (sd_glibc_pow.h); the fast path evaluates correctly
//                    rounded powers and bounds their one-ulp difference
//   math.hypot    -> CPython 3.12 vector_norm algorithm (exact restatement)
//   math.remainder-> CUDA remainder (exact, as glibc)
//   math.sqrt     -> IEEE sqrt (correctly rounded, as glibc)
//   sin/cos/acos/asin/atan2, numpy hypot -> correctly rounded
//                    (sd_crlibm.h): glibc's own value except where glibc
//                    misrounds (0.03-0.25% of arguments, ~0.51 ulp); the
//                    fast path uses its own cheaper functions and bounds
//                    or defers every decision they could move
// CPython's exception rules for math.* / ** are mirrored as status codes.
#pragma once

#include <cstdint>

#include "../../include/symdiag_b200.h"
#include "sd_crlibm.h"
#include "sd_glibc_pow.h"

// SD_LIT_CRLIBM (on): the literal solver's sin/cos/acos/asin/atan2 and
// numpy's hypot are correctly rounded (sd_crlibm.h) instead of libdevice's
// 1-2 ulp versions, so its values and last-bit decisions are glibc's
// wherever glibc is correctly rounded
#ifndef SD_LIT_CRLIBM
#define SD_LIT_CRLIBM 1
#endif

namespace sd {

constexpr double kPi = 3.141592653589793;  // math.pi

// First error wins, as in Python where the first raise unwinds.
struct Err {
  int code = 0;
  __device__ __forceinline__ void raise(int c) {
    if (code == 0) code = c;
  }
};

// Python's max(a, b) / min(a, b) on floats: keep the first unless the second
// compares strictly greater / less (NaN-propagation and -0.0 as CPython).
__device__ __forceinline__ double pmax(double a, double b) { return (b > a) ? b : a; }
__device__ __forceinline__ double pmin(double a, double b) { return (b < a) ? b : a; }

__device__ __forceinline__ bool is_nan(double x) { return x != x; }
__device__ __forceinline__ bool is_inf(double x) { return fabs(x) == __longlong_as_double(0x7ff0000000000000LL); }
__device__ __forceinline__ bool is_finite(double x) { return fabs(x) < __longlong_as_double(0x7ff0000000000000LL); }

// glibc 2.39's pow, bit for bit (sd_glibc_pow.h; tests/test_glibc_pow.py
// checks the same source against the host libm), one out-of-line copy
__device__ __noinline__ double glibc_pow(double x, double y) { return sd_glibc::pow(x, y); }

// float ** k with CPython's OverflowError rule (float_pow: a finite base
// whose libm pow overflows raises; an underflow does not).  Exact: the
// reference's `x**k` is libm pow, whose last bit decides branches and
// signs (sd_glibc_pow.h).
__device__ __forceinline__ double pow_k(Err& e, double x, double k) {
  const double r = glibc_pow(x, k);
  if (is_inf(r) && is_finite(x)) e.raise(SD_ERR_OVERFLOW);
  return r;
}
__device__ __forceinline__ double pow2(Err& e, double x) { return pow_k(e, x, 2.0); }
__device__ __forceinline__ double pow3(Err& e, double x) { return pow_k(e, x, 3.0); }
__device__ __forceinline__ double pow6(Err& e, double x) { return pow_k(e, x, 6.0); }

// a / b, with a == +-0 over a non-zero, non-NaN b answered without the
// division (the same signed zero): libdevice's correctly rounded division
// takes its slow path whenever the quotient is zero
__device__ __forceinline__ double div_nz(double a, double b) {
  if (a == 0.0 && b != 0.0 && b == b) return (signbit(a) != signbit(b)) ? -0.0 : 0.0;
  return a / b;
}

// Correctly rounded x**3 and x**6 (double-double products, one final
// rounding; the fast path's first-level values, |x| below 2^160 so neither
// can overflow).  glibc's pow can differ from them by one ulp: the fast
// path bounds that difference in every decision (sd_fast3.cuh, classify3)
__device__ __forceinline__ double pow3_nc(double x) {
  const double h = __dmul_rn(x, x);
  const double l = fma(x, x, -h);
  const double hi = __dmul_rn(h, x);
  const double lo = fma(h, x, -hi) + __dmul_rn(l, x);
  return hi + lo;
}
__device__ __forceinline__ double pow6_nc(double x) {
  const double h = __dmul_rn(x, x);
  const double l = fma(x, x, -h);
  const double c = __dmul_rn(h, x);
  const double s = __dmul_rn(c, c);
  const double cl = fma(h, x, -c) + __dmul_rn(l, x);
  const double sl = fma(c, c, -s) + 2.0 * __dmul_rn(c, cl);
  return s + sl;
}

// math_1 rules: NaN from non-NaN -> ValueError (math domain error)
__device__ __forceinline__ double chk(Err& e, double r, double x) {
  if (is_nan(r) && !is_nan(x)) e.raise(SD_ERR_MATH_DOMAIN);
  return r;
}
__device__ __forceinline__ double py_sqrt(Err& e, double x) { return chk(e, sqrt(x), x); }
#if SD_LIT_CRLIBM
// correctly rounded (sd_crlibm.h): equal to glibc's wherever glibc rounds
// correctly (99.75-99.97% of arguments), one out-of-line copy each
__device__ __noinline__ double lit_acos(double x) { return sdcr_acos(x); }
__device__ __noinline__ double lit_asin(double x) { return sdcr_asin(x); }
__device__ __noinline__ void lit_sincos(double x, double* s, double* c) { sdcr_sincos(x, s, c); }
__device__ __noinline__ double lit_sin(double x) { return sdcr_sin(x); }
__device__ __noinline__ double lit_cos(double x) { return sdcr_cos(x); }
__device__ __noinline__ double lit_atan2(double y, double x) { return sdcr_atan2(y, x); }
__device__ __noinline__ double lit_hypot(double x, double y) { return sdcr_hypot(x, y); }
#else
__device__ __forceinline__ double lit_acos(double x) { return acos(x); }
__device__ __forceinline__ double lit_asin(double x) { return asin(x); }
__device__ __forceinline__ void lit_sincos(double x, double* s, double* c) { sincos(x, s, c); }
__device__ __forceinline__ double lit_sin(double x) { return sin(x); }
__device__ __forceinline__ double lit_cos(double x) { return cos(x); }
__device__ __forceinline__ double lit_atan2(double y, double x) { return atan2(y, x); }
__device__ __forceinline__ double lit_hypot(double x, double y) { return hypot(x, y); }
#endif
__device__ __forceinline__ double py_acos(Err& e, double x) { return chk(e, lit_acos(x), x); }
__device__ __forceinline__ double py_asin(Err& e, double x) { return chk(e, lit_asin(x), x); }
__device__ __forceinline__ double py_sin(Err& e, double x) { return chk(e, lit_sin(x), x); }
__device__ __forceinline__ double py_cos(Err& e, double x) { return chk(e, lit_cos(x), x); }
__device__ __forceinline__ void py_sincos(Err& e, double x, double* s, double* c) {
  lit_sincos(x, s, c);
  chk(e, *s, x);
}

// math.hypot for two arguments: CPython 3.12 vector_norm (lossless scaling
// by a power of two, error-free squares and compensated sums, one sqrt and
// a differential correction).  Bit-identical to CPython given IEEE sqrt/fma.
// `scale` = 2^-e.  With kMul the final h / scale is evaluated as h * inv,
// inv = 2^e, the same correctly rounded value (both are the exact h * 2^e
// rounded once) — valid whenever 2^e is a finite double.
template <bool kMul>
__device__ __forceinline__ double hypot_scaled(double a, double b, double scale, double inv) {
  double csum = 1.0, frac1 = 0.0, frac2 = 0.0;
  double v0 = __dmul_rn(a, scale), v1 = __dmul_rn(b, scale);
  {
    double hi = __dmul_rn(v0, v0), lo = fma(v0, v0, -hi);
    double s = csum + hi, r = (csum - s) + hi;
    csum = s;
    frac1 += lo;
    frac2 += r;
  }
  {
    double hi = __dmul_rn(v1, v1), lo = fma(v1, v1, -hi);
    double s = csum + hi, r = (csum - s) + hi;
    csum = s;
    frac1 += lo;
    frac2 += r;
  }
  double h = sqrt(csum - 1.0 + (frac1 + frac2));
  double hi = __dmul_rn(-h, h), lo = fma(-h, h, -hi);
  double s = csum + hi, r = (csum - s) + hi;
  csum = s;
  frac1 += lo;
  frac2 += r;
  double t = csum - 1.0 + (frac1 + frac2);
  // t == 0 (common when the operands carry few significant bits, e.g. the
  // rounding-noise off-diagonals of rotated scalar matrices): h + 0 / (2h)
  // is h bit for bit, and skipping the division avoids libdevice's slow
  // division path, which a zero quotient always takes
  if (t != 0.0) h += t / (2.0 * h);
  return kMul ? h * inv : h / scale;
}

// zero / inf / NaN / huge / subnormal magnitudes (CPython's special cases)
__device__ __noinline__ double py_hypot_abs_slow(double a, double b) {
  double mx = 0.0;
  bool found_nan = is_nan(a) || is_nan(b);
  if (a > mx) mx = a;
  if (b > mx) mx = b;
  if (is_inf(mx)) return mx;
  if (found_nan) return __longlong_as_double(0x7ff8000000000000LL);
  if (mx == 0.0) return mx;
  int ex;
  frexp(mx, &ex);
  if (ex < -1023) {
    const double dmin = 0x1p-1022;  // DBL_MIN: convert subnormals to normals
    a = a / dmin;
    b = b / dmin;
    frexp(pmax(a, b), &ex);
    return dmin * hypot_scaled<false>(a, b, ldexp(1.0, -ex), 0.0);
  }
  return hypot_scaled<false>(a, b, ldexp(1.0, -ex), 0.0);
}

__device__ __forceinline__ double py_hypot(double x, double y) {
  double a = fabs(x), b = fabs(y);
  double mx = pmax(a, b);
  // fast path: mx normal with 2^-1021 <= mx < 2^1022 so 2^-e is normal
  if (!(mx >= 0x1p-1021 && mx < 0x1p1022) || is_nan(a) || is_nan(b))
    return py_hypot_abs_slow(a, b);
  int ex = (int)((__double_as_longlong(mx) >> 52) & 0x7ff) - 1022;  // frexp exponent
  double scale = __longlong_as_double((long long)(1023 - ex) << 52);  // ldexp(1, -ex)
  const double inv = __longlong_as_double((long long)(1023 + ex) << 52);  // 2^ex
  return hypot_scaled<true>(a, b, scale, inv);
}

// math.remainder(x, pi) (exact) and the wrap helpers of core.py:29-51
// For |x| <= pi (every angle the solver wraps) the quotient x/pi lies in
// [-1, 1], so n = 0 for |x| <= pi/2 (x = +-pi/2 is an exact tie, rounded to
// even 0) and n = +-1 above; x - +-pi is then exact (Sterbenz), so this is
// bit-identical to remainder() without libdevice's general loop.
__device__ __forceinline__ double rem_pi(Err& e, double x) {
  const double ax = fabs(x);
  if (ax <= 0.5 * kPi) return x;
  if (ax <= kPi) {
    const double r = x - copysign(kPi, x);
    return (r == 0.0) ? copysign(0.0, x) : r;  // remainder's zero keeps x's sign
  }
  return chk(e, remainder(x, kPi), x);
}
// wrap_half_pi (core.py:37-46): representative in (-pi/2, pi/2], -0 -> +0
__device__ __forceinline__ double wrap_half_pi(Err& e, double phi) {
  double r = rem_pi(e, phi);
  if (r <= -0.5 * kPi) r = 0.5 * kPi;
  return (r != 0.0) ? r : 0.0;
}
// wrapped_diff_mod_pi (core.py:49-51)
__device__ __forceinline__ double wrapped_diff(Err& e, double a, double b) {
  return fabs(rem_pi(e, a - b));
}
// angle_of (core.py:238-246): atan2 with -pi mapped to pi
__device__ __forceinline__ double angle_of(Err& e, double x, double y) {
  if (x == 0.0 && y == 0.0) {
    e.raise(SD_ERR_ANGLE_OF_ZERO);
    return __longlong_as_double(0x7ff8000000000000LL);
  }
  double r = lit_atan2(y, x);
  if (r == -kPi) r = kPi;
  return r;
}

__device__ __forceinline__ double qnan() { return __longlong_as_double(0x7ff8000000000000LL); }

}  // namespace sd
