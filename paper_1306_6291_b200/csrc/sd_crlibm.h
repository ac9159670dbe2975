// sd_crlibm.h — correctly rounded sin, cos, acos, asin, atan2 and hypot in
// double precision, as C that compiles for the host (C11 / C++) and for
// sm_100a (the literal solver's libm, sd_math.cuh py_*).
//
// Why: the reference calls glibc's math.cos / sin / acos / asin / atan2 and
// numpy's hypot (glibc) on the decision path (eig3.py:143-174, 218-246,
// 288-379; core.py:238-246).  glibc 2.39's double functions are accurate to
// ~0.51 ulp, i.e. they return the correctly rounded value for all but
// 0.05-0.25% of arguments (tools/crlibm_vs_glibc.py measures it); CUDA's
// libdevice is accurate to 1-2 ulp and disagrees with glibc far more often.
// Last bits of the eigenvalues decide the reference's v / w clamps and the
// V_ZERO_EPS test on diagonal matrices with close eigenvalues (two c3 rows
// of 2^26, VERDICT r1 "weak" 1), so the literal solver computes these
// functions correctly rounded: it then agrees with glibc wherever glibc is
// itself correctly rounded.
//
// How: every function evaluates its result as a double-double (hi + lo,
// ~2^-100 relative) and rounds once:
//   sin / cos   Cody-Waite reduction by pi/2 split into four doubles (exact
//               products via FMA), Taylor polynomials of degree 29 / 28 on
//               |r| <= pi/4 (sd_crlibm_poly.h, generated constants).
//   acos/asin   one Newton step on cos / sin from the hardware estimate, in
//               double-double; for |x| > 0.5 through asin(sqrt((1-|x|)/2))
//               (1 - |x| exact), where the Newton step is well conditioned.
//   atan2       one Newton step on x sin z - y cos z = 0 (cubically
//               convergent) from the hardware estimate, after exact
//               power-of-two scaling.
//   hypot       sqrt of the exact double-double x^2 + y^2, after exact
//               power-of-two scaling, rounded once.
// Two phases (Ziv): each function first evaluates a QUICK double-double
// (sin/cos through a 27-entry table of sin/cos(j/32) and short polynomials
// on |t| <= 1/64, relative error < 2^-76; the inverse functions through the
// same Newton step on it) and returns its high word when the rounding is
// certain within 2^-70 relative; only the ~2^-16 of arguments that land
// closer than that to a rounding boundary take the accurate phase above
// (out of line on the device).  The literal pass's latency is these
// functions' dependent chains: the quick phase is ~4x shorter.
// Arguments outside the restated range (|x| > 2^20 for sin/cos, atan2
// operands more than 2^900 apart, non-finite values) return the hardware
// function's value, which is what glibc returns there to the extent the
// reference can reach them (it cannot: every angle is in [-2 pi, 2 pi]).
// A result whose exact value lies within 2^-98 relative of a rounding
// boundary is counted by sdcr_hard (never seen; probability ~2^-45).
#ifndef SD_CRLIBM_H
#define SD_CRLIBM_H

#include <math.h>
#include <stdint.h>
#include <string.h>

#if defined(__CUDACC__)
#define SDCR_FN static __host__ __device__ __forceinline__
#else
#define SDCR_FN static inline
#endif

#if defined(__CUDACC__)
#define SDCR_SLOW static __host__ __device__ __noinline__
#else
#define SDCR_SLOW static
#endif

typedef struct { double hi, lo; } sdcr_dd;

SDCR_FN sdcr_dd sdcr_mk(double hi, double lo) { sdcr_dd r; r.hi = hi; r.lo = lo; return r; }
SDCR_FN sdcr_dd sdcr_two_sum(double a, double b) {
  double s = a + b, bb = s - a;
  return sdcr_mk(s, (a - (s - bb)) + (b - bb));
}
SDCR_FN sdcr_dd sdcr_fast_two_sum(double a, double b) {  // |a| >= |b| or a == 0
  double s = a + b;
  return sdcr_mk(s, b - (s - a));
}
SDCR_FN sdcr_dd sdcr_two_prod(double a, double b) {
  double p = a * b;
  return sdcr_mk(p, fma(a, b, -p));
}
// accurate double-double sum: relative error <= 3 u^2 of the result
SDCR_FN sdcr_dd sdcr_add(sdcr_dd a, sdcr_dd b) {
  sdcr_dd s = sdcr_two_sum(a.hi, b.hi), t = sdcr_two_sum(a.lo, b.lo);
  s = sdcr_fast_two_sum(s.hi, s.lo + t.hi);
  return sdcr_fast_two_sum(s.hi, s.lo + t.lo);
}
SDCR_FN sdcr_dd sdcr_add_d(sdcr_dd a, double b) {
  sdcr_dd s = sdcr_two_sum(a.hi, b);
  return sdcr_fast_two_sum(s.hi, s.lo + a.lo);
}
SDCR_FN sdcr_dd sdcr_neg(sdcr_dd a) { return sdcr_mk(-a.hi, -a.lo); }
SDCR_FN sdcr_dd sdcr_mul(sdcr_dd a, sdcr_dd b) {
  sdcr_dd p = sdcr_two_prod(a.hi, b.hi);
  double t = fma(a.hi, b.lo, a.lo * b.hi);
  return sdcr_fast_two_sum(p.hi, p.lo + t);
}
SDCR_FN sdcr_dd sdcr_mul_d(sdcr_dd a, double b) {
  sdcr_dd p = sdcr_two_prod(a.hi, b);
  return sdcr_fast_two_sum(p.hi, fma(a.lo, b, p.lo));
}

#include "sd_crlibm_poly.h"

#if defined(__CUDA_ARCH__)
#define SDCR_HARD_COUNT() ((void)0)
#else
static unsigned long long sdcr_hard_count;
#define SDCR_HARD_COUNT() (sdcr_hard_count++)
#endif

#if defined(__CUDA_ARCH__)
SDCR_FN uint64_t sdcr_bits(double x) { return (uint64_t)__double_as_longlong(x); }
SDCR_FN double sdcr_from(uint64_t b) { return __longlong_as_double((long long)b); }
#else
SDCR_FN uint64_t sdcr_bits(double x) { uint64_t b; memcpy(&b, &x, 8); return b; }
SDCR_FN double sdcr_from(uint64_t b) { double x; memcpy(&x, &b, 8); return x; }
#endif

// Round a normalised double-double (hi = RN(hi + lo)) to double.  The exact
// value is within rel * |hi| of hi + lo; if that window reaches a rounding
// boundary (hi +- half an ulp) the result might not be the correctly
// rounded one: counted, never observed.
SDCR_FN double sdcr_round(sdcr_dd r) {
  const double hi = r.hi;
  if (r.lo != 0.0 && hi != 0.0) {
    const double up = sdcr_from(sdcr_bits(fabs(hi)) + 1) - fabs(hi);    // ulp above |hi|
    const double dn = fabs(hi) - sdcr_from(sdcr_bits(fabs(hi)) - 1);    // ulp below |hi|
    const double half = ((r.lo > 0.0) == (hi > 0.0) ? up : dn) * 0.5;
    if (fabs(fabs(r.lo) - half) <= 0x1p-98 * fabs(hi)) SDCR_HARD_COUNT();
  }
  return hi;
}

// x = k pi/2 + r, |r| <= ~pi/4 (double-double), for |x| <= 2^20
SDCR_FN int sdcr_reduce(double x, sdcr_dd* r) {
  const double k = rint(x * SDCR_2OPI);
  sdcr_dd p = sdcr_two_prod(k, SDCR_PIO2_0);
  sdcr_dd t = sdcr_two_sum(x, -p.hi);
  t = sdcr_add_d(t, -p.lo);
  p = sdcr_two_prod(k, SDCR_PIO2_1);
  t = sdcr_add(t, sdcr_neg(p));
  p = sdcr_two_prod(k, SDCR_PIO2_2);
  t = sdcr_add(t, sdcr_neg(p));
  t = sdcr_add_d(t, -k * SDCR_PIO2_3);
  *r = t;
  return (int)((int64_t)k & 3);
}

// sin(r), cos(r) of a reduced double-double argument
SDCR_FN sdcr_dd sdcr_sin_r(sdcr_dd r) {
  const sdcr_dd z = sdcr_mul(r, r);
  return sdcr_mul(sdcr_sin_poly(z), r);
}
SDCR_FN sdcr_dd sdcr_cos_r(sdcr_dd r) {
  return sdcr_cos_poly(sdcr_mul(r, r));
}

// sin and cos of a double as double-doubles (|x| <= 2^20)
SDCR_FN void sdcr_sincos_dd(double x, sdcr_dd* s, sdcr_dd* c) {
  sdcr_dd r;
  const int q = sdcr_reduce(x, &r);
  const sdcr_dd sr = sdcr_sin_r(r), cr = sdcr_cos_r(r);
  switch (q) {
    case 0: *s = sr; *c = cr; break;
    case 1: *s = cr; *c = sdcr_neg(sr); break;
    case 2: *s = sdcr_neg(sr); *c = sdcr_neg(cr); break;
    default: *s = sdcr_neg(cr); *c = sr; break;
  }
}

// ---- quick phase ---------------------------------------------------------
#if defined(__CUDACC__)
static __device__ const double sdcr_sc_tab_dev[27 * 4] = {SDCR_SC_TAB_INIT};
#endif
static const double sdcr_sc_tab_host[27 * 4] = {SDCR_SC_TAB_INIT};
#if defined(__CUDA_ARCH__)
#define SDCR_SC_TAB sdcr_sc_tab_dev
#else
#define SDCR_SC_TAB sdcr_sc_tab_host
#endif
#define SDCR_QUICK_EPS 0x1p-70

// Is hi the correctly rounded value of hi + lo + e for every |e| <= eps |hi|?
// (r normalised: hi = RN(hi + lo))
SDCR_FN int sdcr_certain(sdcr_dd r, double eps) {
  const double ah = fabs(r.hi);
  const uint64_t b = sdcr_bits(ah);
  if (b == 0) return r.lo == 0.0;
  const double up = sdcr_from(b + 1) - ah;  // ulp above |hi|
  const double dn = ah - sdcr_from(b - 1);  // ulp below |hi|
  const double half = ((r.lo > 0.0) == (r.hi > 0.0) ? up : dn) * 0.5;
  return fabs(r.lo) + eps * ah < half;
}

// sin and cos of a double as double-doubles, relative error < 2^-76
// (|x| <= 2^20): x = k pi/2 + r, |r| = j/32 + t with |t| <= 1/64 (the
// subtraction is exact), sin t and cos t from short series whose leading
// corrections are double-doubles, then the angle-addition formulas with
// sin(j/32), cos(j/32) from a double-double table.
SDCR_FN void sdcr_sincos_dd_q(double x, sdcr_dd* s, sdcr_dd* c) {
  sdcr_dd r;
  int q = 0;
  if (fabs(x) <= 0x1.921fb54442d18p-1) r = sdcr_mk(x, 0.0);
  else q = sdcr_reduce(x, &r);
  const int neg = r.hi < 0.0;
  const double ar = fabs(r.hi);
  const int j = (int)(ar * 32.0 + 0.5);  // 0..26
  const sdcr_dd t = sdcr_two_sum(ar - (double)j * 0.03125, neg ? -r.lo : r.lo);
  const double zh = t.hi * t.hi;
  const double zl = fma(t.hi, t.hi, -zh) + 2.0 * t.hi * t.lo;
  // sin t = t + t w, w = -z/6 (double-double) + z^2 (1/120 - z/5040 + z^2/362880)
  const double qs = zh * zh * (0x1.1111111111111p-7 + zh * (-0x1.a01a01a01a01ap-13 + zh * 0x1.71de3a556c734p-19));
  const double uh = zh * -0x1.5555555555555p-3;
  const double ul = fma(zh, -0x1.5555555555555p-3, -uh) + (zh * -0x1.5555555555555p-57 + zl * -0x1.5555555555555p-3);
  const double wl = ul + qs;
  const double ph = t.hi * uh;
  const double pl = fma(t.hi, uh, -ph) + (t.hi * wl + t.lo * uh);
  sdcr_dd st = sdcr_fast_two_sum(t.hi, ph);
  st = sdcr_fast_two_sum(st.hi, st.lo + (pl + t.lo));
  // cos t = 1 - z/2 + z^2 (1/24 - z/720 + z^2/40320 - z^3/3628800)
  const double qc = zh * zh * (0x1.5555555555555p-5 + zh * (-0x1.6c16c16c16c17p-10 + zh * (0x1.a01a01a01a01ap-16 + zh * -0x1.27e4fb7789f5cp-22)));
  sdcr_dd ct = sdcr_fast_two_sum(1.0, -0.5 * zh);
  ct = sdcr_fast_two_sum(ct.hi, ct.lo + (qc - 0.5 * zl));
  // angle addition with a = j/32
  const double* T = SDCR_SC_TAB + 4 * j;
  const sdcr_dd S = sdcr_mk(T[0], T[1]), C = sdcr_mk(T[2], T[3]);
  const sdcr_dd a1 = sdcr_mul(S, ct), b1 = sdcr_mul(C, st);  // |a1| >= |b1| or a1 == 0
  sdcr_dd sr = sdcr_fast_two_sum(a1.hi, b1.hi);
  sr = sdcr_fast_two_sum(sr.hi, sr.lo + (a1.lo + b1.lo));
  const sdcr_dd a2 = sdcr_mul(C, ct), b2 = sdcr_mul(S, st);  // |a2| >= 0.68 > |b2|
  sdcr_dd cr = sdcr_fast_two_sum(a2.hi, -b2.hi);
  cr = sdcr_fast_two_sum(cr.hi, cr.lo + (a2.lo - b2.lo));
  if (neg) sr = sdcr_neg(sr);
  switch (q) {
    case 0: *s = sr; *c = cr; break;
    case 1: *s = cr; *c = sdcr_neg(sr); break;
    case 2: *s = sdcr_neg(sr); *c = sdcr_neg(cr); break;
    default: *s = sdcr_neg(cr); *c = sr; break;
  }
}

// quick != 0: the quick phase; else the accurate one
SDCR_FN void sdcr_sincos_dd_any(double x, sdcr_dd* s, sdcr_dd* c, int quick) {
  if (quick) sdcr_sincos_dd_q(x, s, c);
  else sdcr_sincos_dd(x, s, c);
}

SDCR_FN int sdcr_trig_ok(double x) { return fabs(x) <= 0x1p20; }

SDCR_SLOW void sdcr_sincos_slow(double x, double* s, double* c) {
  sdcr_dd sd, cd;
  sdcr_sincos_dd(x, &sd, &cd);
  *s = sdcr_round(sd);
  *c = sdcr_round(cd);
}
SDCR_FN double sdcr_sin(double x) {
  if (!sdcr_trig_ok(x)) return sin(x);
  if (fabs(x) < 0x1p-26) return x;  // sin x = x (1 - x^2/6): rounds to x, sign of zero kept
  sdcr_dd s, c;
  sdcr_sincos_dd_q(x, &s, &c);
  if (sdcr_certain(s, SDCR_QUICK_EPS)) return s.hi;
  double sv, cv;
  sdcr_sincos_slow(x, &sv, &cv);
  return sv;
}
SDCR_FN double sdcr_cos(double x) {
  if (!sdcr_trig_ok(x)) return cos(x);
  if (fabs(x) < 0x1p-27) return 1.0;
  sdcr_dd s, c;
  sdcr_sincos_dd_q(x, &s, &c);
  if (sdcr_certain(c, SDCR_QUICK_EPS)) return c.hi;
  double sv, cv;
  sdcr_sincos_slow(x, &sv, &cv);
  return cv;
}
SDCR_FN void sdcr_sincos(double x, double* s, double* c) {
  if (!sdcr_trig_ok(x)) { *s = sin(x); *c = cos(x); return; }
  if (fabs(x) < 0x1p-27) { *s = x; *c = 1.0; return; }
  sdcr_dd sd, cd;
  sdcr_sincos_dd_q(x, &sd, &cd);
  double sv = sd.hi, cv = cd.hi;
  if (!(sdcr_certain(sd, SDCR_QUICK_EPS) && sdcr_certain(cd, SDCR_QUICK_EPS)))
    sdcr_sincos_slow(x, &sv, &cv);
  *s = fabs(x) < 0x1p-26 ? x : sv;
  *c = cv;
}

// asin of a double-double s in [0, 0.5] as a double-double: one Newton step
// on sin from the hardware estimate (error ~ e0^2 tan(z) / 2 ~ 2^-103 z)
SDCR_FN sdcr_dd sdcr_asin_dd_small(sdcr_dd s, int quick) {
  double z0 = asin(s.hi), corr;
  if (z0 == 0.0) return s;
  for (int it = 0;; it++) {
    sdcr_dd sn, cs;
    sdcr_sincos_dd_any(z0, &sn, &cs, quick);
    corr = -(sdcr_add(sn, sdcr_neg(s)).hi / cs.hi);  // -(sin z0 - s) / cos z0
    if (it == 1 || !(fabs(corr) > 0x1p-50 * z0)) break;
    z0 = z0 + corr;
  }
  return sdcr_two_sum(z0, corr);
}

// sqrt((1 - |x|) / 2) as a double-double, 0.5 <= |x| <= 1 (1 - |x| exact)
SDCR_FN sdcr_dd sdcr_half_versine_sqrt(double ax) {
  const double t = (1.0 - ax) * 0.5;
  const double h = sqrt(t);
  if (h == 0.0) return sdcr_mk(0.0, 0.0);
  return sdcr_fast_two_sum(h, fma(-h, h, t) / (2.0 * h));
}

// acos(x) as a double-double, |x| <= 1
SDCR_FN sdcr_dd sdcr_acos_dd(double x, int quick) {
  if (fabs(x) <= 0.5) {
    // acos(x) in [pi/3, 2pi/3]: Newton on cos y - x (error ~ e0^2 cot / 2)
    double y0 = acos(x), corr;
    for (int it = 0;; it++) {
      sdcr_dd sn, cs;
      sdcr_sincos_dd_any(y0, &sn, &cs, quick);
      corr = sdcr_add_d(cs, -x).hi / sn.hi;       // (cos y0 - x) / sin y0
      if (it == 1 || !(fabs(corr) > 0x1p-50 * y0)) break;
      y0 = y0 + corr;  // estimate off by more than ~2 ulp: one more step
    }
    return sdcr_two_sum(y0, corr);
  }
  const sdcr_dd z = sdcr_asin_dd_small(sdcr_half_versine_sqrt(fabs(x)), quick);
  const sdcr_dd z2 = sdcr_mk(2.0 * z.hi, 2.0 * z.lo);
  if (x > 0.0) return z2;
  return sdcr_add(sdcr_mk(SDCR_PI_HI, SDCR_PI_LO), sdcr_neg(z2));
}
SDCR_SLOW double sdcr_acos_slow(double x) { return sdcr_round(sdcr_acos_dd(x, 0)); }
SDCR_FN double sdcr_acos(double x) {
  if (!(fabs(x) <= 1.0)) return acos(x);  // NaN (CPython: ValueError)
  const sdcr_dd r = sdcr_acos_dd(x, 1);
  if (sdcr_certain(r, SDCR_QUICK_EPS)) return r.hi;
  return sdcr_acos_slow(x);
}

// asin(|x|) as a double-double, 2^-26 <= |x| <= 1
SDCR_FN sdcr_dd sdcr_asin_dd(double ax, int quick) {
  if (ax <= 0.5) return sdcr_asin_dd_small(sdcr_mk(ax, 0.0), quick);
  const sdcr_dd z = sdcr_asin_dd_small(sdcr_half_versine_sqrt(ax), quick);
  return sdcr_add(sdcr_mk(SDCR_PIO2_HI, SDCR_PIO2_LO), sdcr_mk(-2.0 * z.hi, -2.0 * z.lo));
}
SDCR_SLOW double sdcr_asin_slow(double ax) { return sdcr_round(sdcr_asin_dd(ax, 0)); }
SDCR_FN double sdcr_asin(double x) {
  if (!(fabs(x) <= 1.0)) return asin(x);
  if (x == 0.0 || fabs(x) < 0x1p-26) return x;  // asin x = x (1 + x^2/6 ...): rounds to x
  const sdcr_dd r = sdcr_asin_dd(fabs(x), 1);
  return copysign(sdcr_certain(r, SDCR_QUICK_EPS) ? r.hi : sdcr_asin_slow(fabs(x)), x);
}

// atan2 of exactly scaled finite non-zero operands, max(|xs|, |ys|) in [0.5, 1)
SDCR_FN sdcr_dd sdcr_atan2_dd(double ys, double xs, int quick) {
  const double z0 = atan2(ys, xs);
  sdcr_dd sn, cs;
  sdcr_sincos_dd_any(z0, &sn, &cs, quick);
  // f(z) = x sin z - y cos z, f'(z) = x cos z + y sin z; f'' = -f
  const sdcr_dd f = sdcr_add(sdcr_mul_d(sn, xs), sdcr_neg(sdcr_mul_d(cs, ys)));
  const double fp = xs * cs.hi + ys * sn.hi;
  return sdcr_two_sum(z0, -(f.hi / fp));
}
SDCR_SLOW double sdcr_atan2_slow(double ys, double xs) { return sdcr_round(sdcr_atan2_dd(ys, xs, 0)); }
SDCR_FN double sdcr_atan2(double y, double x) {
  if (!(fabs(x) < INFINITY && fabs(y) < INFINITY) || x == 0.0 || y == 0.0)
    return atan2(y, x);  // NaN, infinities, zeros: exact special values
  int ex, ey;
  frexp(x, &ex);
  frexp(y, &ey);
  if (ex - ey > 900 || ey - ex > 900) return atan2(y, x);
  const int e = ex > ey ? ex : ey;
  const double xs = ldexp(x, -e), ys = ldexp(y, -e);  // exact, max(|xs|,|ys|) in [0.5, 1)
  const sdcr_dd r = sdcr_atan2_dd(ys, xs, 1);
  if (sdcr_certain(r, SDCR_QUICK_EPS)) return r.hi;
  return sdcr_atan2_slow(ys, xs);
}

SDCR_FN double sdcr_hypot(double x, double y) {
  double ax = fabs(x), ay = fabs(y);
  if (!(ax < INFINITY && ay < INFINITY)) return hypot(x, y);
  if (ax < ay) { const double t = ax; ax = ay; ay = t; }
  if (ay == 0.0) return ax;
  int e;
  frexp(ax, &e);
  if (e - 0 > 1000 || e < -1000) return hypot(x, y);  // far from the reference's range
  const double xs = ldexp(ax, -e), ys = ldexp(ay, -e);
  // s = xs^2 + ys^2 exactly enough as a double-double
  const sdcr_dd s = sdcr_add(sdcr_two_prod(xs, xs), sdcr_two_prod(ys, ys));
  const double h = sqrt(s.hi);
  // sqrt(s) = h + (s - h^2) / (2h): one correction in double-double
  const double rem = (fma(-h, h, s.hi) + s.lo) / (2.0 * h);
  return ldexp(sdcr_round(sdcr_fast_two_sum(h, rem)), e);
}

#endif  // SD_CRLIBM_H
