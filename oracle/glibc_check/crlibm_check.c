/* Host checker (test infrastructure): the device's correctly rounded libm
 * (paper_1306_6291_b200/csrc/sd_crlibm.h, compiled here as plain C) and the
 * installed glibc libm side by side, for tests/test_crlibm.py.
 *   fn: 0 sin, 1 cos, 2 acos, 3 asin, 4 atan2(x, y), 5 hypot(x, y)
 *   which: 0 = sd_crlibm (quick phase + accurate fallback), 1 = glibc,
 *          2 = sd_crlibm's accurate phase alone                            */
#include "../../paper_1306_6291_b200/csrc/sd_crlibm.h"

void cr_eval(int fn, int which, const double* x, const double* y, double* out, long n) {
  for (long i = 0; i < n; i++) {
    double r;
    switch (fn) {
      case 0: r = which ? sin(x[i]) : sdcr_sin(x[i]); break;
      case 1: r = which ? cos(x[i]) : sdcr_cos(x[i]); break;
      case 2: r = which ? acos(x[i]) : sdcr_acos(x[i]); break;
      case 3: r = which ? asin(x[i]) : sdcr_asin(x[i]); break;
      case 4: r = which ? atan2(x[i], y[i]) : sdcr_atan2(x[i], y[i]); break;
      default: r = which ? hypot(x[i], y[i]) : sdcr_hypot(x[i], y[i]); break;
    }
    out[i] = r;
  }
}

static double slow_eval(int fn, double x, double y) {
  double s, c;
  switch (fn) {
    case 0: if (!sdcr_trig_ok(x) || fabs(x) < 0x1p-26) return sdcr_sin(x); sdcr_sincos_slow(x, &s, &c); return s;
    case 1: if (!sdcr_trig_ok(x) || fabs(x) < 0x1p-27) return sdcr_cos(x); sdcr_sincos_slow(x, &s, &c); return c;
    case 2: return fabs(x) <= 1.0 ? sdcr_acos_slow(x) : sdcr_acos(x);
    case 3: return (fabs(x) <= 1.0 && fabs(x) >= 0x1p-26) ? copysign(sdcr_asin_slow(fabs(x)), x) : sdcr_asin(x);
    case 4: {
      if (!(fabs(x) < INFINITY && fabs(y) < INFINITY) || x == 0.0 || y == 0.0) return sdcr_atan2(x, y);
      int ex, ey;
      frexp(y, &ex);
      frexp(x, &ey);
      if (ex - ey > 900 || ey - ex > 900) return sdcr_atan2(x, y);
      const int e = ex > ey ? ex : ey;
      return sdcr_atan2_slow(ldexp(x, -e), ldexp(y, -e));
    }
    default: return sdcr_hypot(x, y);
  }
}

void cr_eval_slow(int fn, const double* x, const double* y, double* out, long n) {
  for (long i = 0; i < n; i++) out[i] = slow_eval(fn, x[i], y[i]);
}

/* max relative distance between the quick and the accurate double-double
 * sin / cos over the arguments, and how many calls the quick phase could not
 * certify (returned through *uncertain) */
double cr_quick_sincos_err(const double* x, long n, long* uncertain) {
  double worst = 0.0;
  long unc = 0;
  for (long i = 0; i < n; i++) {
    sdcr_dd qs, qc, ss, sc;
    sdcr_sincos_dd_q(x[i], &qs, &qc);
    sdcr_sincos_dd(x[i], &ss, &sc);
    const double es = fabs((qs.hi - ss.hi) + (qs.lo - ss.lo)) / fabs(ss.hi);
    const double ec = fabs((qc.hi - sc.hi) + (qc.lo - sc.lo)) / fabs(sc.hi);
    if (ss.hi != 0.0 && es > worst) worst = es;
    if (sc.hi != 0.0 && ec > worst) worst = ec;
    unc += !sdcr_certain(qs, SDCR_QUICK_EPS) + !sdcr_certain(qc, SDCR_QUICK_EPS);
  }
  *uncertain = unc;
  return worst;
}

unsigned long long cr_hard_count(void) { return sdcr_hard_count; }
