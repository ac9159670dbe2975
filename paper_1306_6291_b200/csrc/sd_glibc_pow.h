// sd_glibc_pow.h — glibc 2.39's double-precision pow, bit for bit, as
// portable C++ that compiles both for the host (tests/test_glibc_pow.py
// checks it against the installed libm) and for sm_100a (the device's
// exact x**2, x**3, x**6).
//
// Why: every `x**k` of the reference (eig3.py:89, 99, 105-108, 140, 147,
// 151; core.py:107-108) is CPython float_pow -> libm pow(), which on an
// x86-64 host with FMA/AVX2 is glibc's __pow_fma: the ARM optimized-routines
// algorithm (sysdeps/ieee754/dbl-64/e_pow.c) compiled with -mfma -mavx2,
// so gcc fused several a*b+c into FMAs.  pow is not correctly rounded
// (<= 0.52 ulp), so x*x differs from pow(x, 2) in ~0.08% of calls; those
// last bits decide the reference's branch (p, disc thresholds), the sign of
// q on rotated scalar matrices (eig3.py:150) and, through the acos argument,
// eigenvalues of nearly double roots (VERDICT r1 "missing" 2).
//
// Algorithm (restated; the contraction pattern is the one of the FMA build,
// read off its machine code):
//   x = 2^k z, z in [0x1.69555p-1, 0x1.69555p0), table entry i of the
//   subinterval: log x = k ln2 + log c + log1p(r), r = fma(z, 1/c, -1) exact,
//   with a degree-7 polynomial; the double-double (hi, lo) of log x is
//   multiplied by y with an FMA-exact product; exp of the result: x = k
//   ln2/N + r, 2^(k/N) from a 128-entry table as scale (1 + tail), a
//   degree-5 polynomial, result = fma(scale, tmp, scale).
// Tables: sd_glibc_tables.h, computed by tools/gen_glibc_tables.py from
// their published construction.  Constants below: the published
// coefficients of e_pow_log_data.c / e_exp_data.c (POW_LOG_POLY_ORDER 8,
// EXP_POLY_ORDER 5, N = 128).
//
// Scope: any x; y an integer-valued double with 2^-65 <= |y| < 2^63 (the
// reference only raises to 2, 3 and 6; glibc's special-y branch is not
// restated).  Overflow returns +-inf (CPython: OverflowError), underflow
// the correctly signed result glibc returns (0 or subnormal), negative x
// with odd y a negative result.
#pragma once

#include <cstdint>
#include <cstring>
#include <cmath>

#if defined(__CUDACC__)
#define SD_GP_HD __host__ __device__ __forceinline__
#else
#define SD_GP_HD inline
#endif

#if defined(__CUDACC__)
#define SD_GLIBC_TABLE __device__ const
#else
#define SD_GLIBC_TABLE static const
#endif
namespace sd_glibc {
#include "sd_glibc_tables.h"
}
#if defined(__CUDACC__)
// host-side copies for the host compilation pass of the same translation
// unit (the __device__ arrays are not readable from host code)
namespace sd_glibc_host {
#undef SD_GLIBC_TABLE
#define SD_GLIBC_TABLE static const
#include "sd_glibc_tables.h"
}
#endif

namespace sd_glibc {

SD_GP_HD double asdouble(uint64_t b) {
#if defined(__CUDA_ARCH__)
  return __longlong_as_double((long long)b);
#else
  double d;
  std::memcpy(&d, &b, 8);
  return d;
#endif
}
SD_GP_HD uint64_t asuint64(double d) {
#if defined(__CUDA_ARCH__)
  return (uint64_t)__double_as_longlong(d);
#else
  uint64_t b;
  std::memcpy(&b, &d, 8);
  return b;
#endif
}
SD_GP_HD double fma_(double a, double b, double c) {
#if defined(__CUDA_ARCH__)
  return __fma_rn(a, b, c);
#else
  return std::fma(a, b, c);
#endif
}
// plain IEEE operations (never contracted: the device library is built with
// -fmad=false, the host checker with -ffp-contract=off)
SD_GP_HD double mul_(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dmul_rn(a, b);
#else
  return a * b;
#endif
}
SD_GP_HD double add_(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dadd_rn(a, b);
#else
  return a + b;
#endif
}
SD_GP_HD double sub_(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dsub_rn(a, b);
#else
  return a - b;
#endif
}

SD_GP_HD uint64_t log_tab(int i, int f) {
#if defined(__CUDA_ARCH__)
  return (uint64_t)__ldg(reinterpret_cast<const unsigned long long*>(&kPowLogTab[3 * i + f]));
#elif defined(__CUDACC__)
  return sd_glibc_host::kPowLogTab[3 * i + f];
#else
  return kPowLogTab[3 * i + f];
#endif
}
SD_GP_HD uint64_t exp_tab(int j) {
#if defined(__CUDA_ARCH__)
  return (uint64_t)__ldg(reinterpret_cast<const unsigned long long*>(&kExpTab[j]));
#elif defined(__CUDACC__)
  return sd_glibc_host::kExpTab[j];
#else
  return kExpTab[j];
#endif
}

// e_pow_log_data.c: ln2 split and the log1p polynomial (A[0] = -1/2)
constexpr double kLn2hi = 0x1.62e42fefa3800p-1;
constexpr double kLn2lo = 0x1.ef35793c76730p-45;
constexpr double kA0 = -0x1p-1;
constexpr double kA1 = 0x1.555555555556p-2 * -2;
constexpr double kA2 = -0x1.0000000000006p-2 * -2;
constexpr double kA3 = 0x1.999999959554ep-3 * 4;
constexpr double kA4 = -0x1.555555529a47ap-3 * 4;
constexpr double kA5 = 0x1.2495b9b4845e9p-3 * -8;
constexpr double kA6 = -0x1.0002b8b263fc3p-3 * -8;
// e_exp_data.c (N = 128)
constexpr double kInvLn2N = 0x1.71547652b82fep0 * 128;
constexpr double kShift = 0x1.8p52;
constexpr double kNegLn2hiN = -0x1.62e42fefa0000p-8;
constexpr double kNegLn2loN = -0x1.cf79abc9e3b3ap-47;
constexpr double kC2 = 0x1.ffffffffffdbdp-2;
constexpr double kC3 = 0x1.555555555543cp-3;
constexpr double kC4 = 0x1.55555cf172b91p-5;
constexpr double kC5 = 0x1.1111167a4d017p-7;
constexpr uint64_t kOff = 0x3fe6955500000000ULL;
constexpr uint64_t kSignBias = 0x800ULL << 7;

// log_inline: log(x) as hi + tail for the positive normal bit pattern ix
SD_GP_HD double log_inline(uint64_t ix, double* tail) {
  const uint64_t tmp = ix - kOff;
  const int i = (int)((tmp >> 45) % 128);
  const int k = (int)((int64_t)tmp >> 52);
  const uint64_t iz = ix - (tmp & (0xfffULL << 52));
  const double z = asdouble(iz);
  const double kd = (double)k;
  const double invc = asdouble(log_tab(i, 0));
  const double logc = asdouble(log_tab(i, 1));
  const double logctail = asdouble(log_tab(i, 2));
  const double r = fma_(z, invc, -1.0);
  const double t1 = fma_(kd, kLn2hi, logc);            // kd*Ln2hi + logc, fused
  const double t2 = add_(t1, r);
  const double lo1 = fma_(kd, kLn2lo, logctail);        // kd*Ln2lo + logctail, fused
  const double lo2 = add_(sub_(t1, t2), r);
  const double ar = mul_(kA0, r);
  const double ar2 = mul_(r, ar);
  const double ar3 = mul_(r, ar2);
  const double hi = add_(t2, ar2);
  const double lo3 = fma_(ar, r, -ar2);
  const double lo4 = add_(sub_(t2, hi), ar2);
  // p = ar3 * (A1 + r A2 + ar2 (A3 + r A4 + ar2 (A5 + r A6))), each
  // "a + r*b" and "a + ar2*b" fused, and p folded into the lo sum by an FMA
  const double q56 = fma_(r, kA6, kA5);
  const double q34 = fma_(r, kA4, kA3);
  const double q12 = fma_(r, kA2, kA1);
  const double q3456 = fma_(q56, ar2, q34);
  const double poly = fma_(ar2, q3456, q12);
  const double losum = add_(add_(add_(lo1, lo2), lo3), lo4);
  const double lo = fma_(ar3, poly, losum);
  const double y = add_(hi, lo);
  *tail = add_(sub_(hi, y), lo);
  return y;
}

// specialcase of exp_inline: scale's exponent over/underflowed (abstop == 0)
SD_GP_HD double exp_specialcase(double tmp, uint64_t sbits, uint64_t ki) {
  if ((ki & 0x80000000ULL) == 0) {
    // k > 0: the exponent of scale might have overflowed by <= 460
    sbits -= 1009ULL << 52;
    const double scale = asdouble(sbits);
    return mul_(0x1p1009, fma_(scale, tmp, scale));
  }
  // k < 0: careful rounding in the subnormal range
  sbits += 1022ULL << 52;
  const double scale = asdouble(sbits);
  const double st = mul_(scale, tmp);  // one product, used twice (not fused)
  double y = add_(scale, st);
  if (std::fabs(y) < 1.0) {
    const double one = (y < 0.0) ? -1.0 : 1.0;
    double lo = add_(sub_(scale, y), st);
    const double hi = add_(one, y);
    lo = add_(add_(sub_(one, hi), y), lo);
    y = sub_(add_(lo, hi), one);
    if (y == 0.0) y = asdouble(sbits & 0x8000000000000000ULL);
  }
  return mul_(0x1p-1022, y);
}

SD_GP_HD uint32_t top12(double x) { return (uint32_t)(asuint64(x) >> 52); }

// exp_inline(x, xtail, sign_bias)
SD_GP_HD double exp_inline(double x, double xtail, uint32_t sign_bias) {
  uint32_t abstop = top12(x) & 0x7ff;
  if (abstop - 0x3c9u >= 0x408u - 0x3c9u) {   // |x| < 2^-54 or >= 512 (or NaN)
    if ((int32_t)(abstop - 0x3c9u) < 0) {
      const double one = add_(1.0, x);         // tiny x: exp(x) rounds to 1 (+x)
      return sign_bias ? -one : one;
    }
    if (abstop >= 0x409u) {                    // |x| >= 1024: over/underflow
      if (asuint64(x) >> 63) {
        // __math_uflow: (+-0x1p-767) * 0x1p-767
        const double t = sign_bias ? -0x1p-767 : 0x1p-767;
        return mul_(t, 0x1p-767);
      }
      const double t = sign_bias ? -0x1p769 : 0x1p769;
      return mul_(t, 0x1p769);                 // __math_oflow: +-inf
    }
    abstop = 0;                                // large x: specialcase below
  }
  const double kd0 = fma_(x, kInvLn2N, kShift); // z + Shift with z = InvLn2N x, fused
  const uint64_t ki = asuint64(kd0);
  const double kd = sub_(kd0, kShift);
  double r = fma_(kd, kNegLn2loN, fma_(kd, kNegLn2hiN, x));
  r = add_(xtail, r);
  const uint64_t idx = 2 * (ki % 128);
  const uint64_t top = (ki + sign_bias) << (52 - 7);
  const double tail = asdouble(exp_tab((int)idx));
  const uint64_t sbits = exp_tab((int)idx + 1) + top;
  const double r2 = mul_(r, r);
  const double p23 = fma_(r, kC3, kC2);
  const double p45 = fma_(r, kC5, kC4);
  const double tr = add_(tail, r);
  const double t = fma_(p23, r2, tr);
  const double r4 = mul_(r2, r2);
  const double tmp = fma_(p45, r4, t);
  if (abstop == 0) return exp_specialcase(tmp, sbits, ki);
  const double scale = asdouble(sbits);
  return fma_(scale, tmp, scale);
}

// checkint for an integer-valued y: 1 odd, 2 even
SD_GP_HD int y_parity(uint64_t iy) {
  const int e = (int)((iy >> 52) & 0x7ff);
  if (e < 0x3ff) return 0;
  if (e > 0x3ff + 52) return 2;
  if (iy & ((1ULL << (0x3ff + 52 - e)) - 1)) return 0;
  if (iy & (1ULL << (0x3ff + 52 - e))) return 1;
  return 2;
}

// pow(x, y) for finite x and finite integer-valued y with 2^-65 <= |y| < 2^63
SD_GP_HD double pow(double x, double y) {
  uint64_t ix = asuint64(x);
  const uint64_t iy = asuint64(y);
  uint32_t topx = top12(x);
  uint32_t sign_bias = 0;
  if (topx - 0x001u >= 0x7ffu - 0x001u) {
    // x <= 0, subnormal, or non-finite
    if (2 * ix - 1 >= 2 * 0x7ff0000000000000ULL - 1) {  // x = +-0, +-inf or NaN
      double x2 = mul_(x, x);
      if ((ix >> 63) && y_parity(iy) == 1) x2 = -x2;
      return (iy >> 63) ? 1.0 / x2 : x2;
    }
    if (ix >> 63) {                            // x < 0
      const int yint = y_parity(iy);
      if (yint == 0) return asdouble(0x7ff8000000000000ULL);  // __math_invalid
      if (yint == 1) sign_bias = (uint32_t)kSignBias;
      ix &= 0x7fffffffffffffffULL;
      topx &= 0x7ff;
    }
    if (topx == 0) {                           // subnormal: normalize
      ix = asuint64(mul_(asdouble(ix), 0x1p52));
      ix &= 0x7fffffffffffffffULL;
      ix -= 52ULL << 52;
    }
  }
  double lo;
  const double hi = log_inline(ix, &lo);
  const double ehi = mul_(y, hi);
  const double elo = fma_(y, lo, fma_(y, hi, -ehi));  // y*lo + fma(y, hi, -ehi), fused
  return exp_inline(ehi, elo, sign_bias);
}

}  // namespace sd_glibc
