/* Host checker (test infrastructure): the device's correctly rounded libm
 * (paper_1306_6291_b200/csrc/sd_crlibm.h, compiled here as plain C) and the
 * installed glibc libm side by side, for tests/test_crlibm.py.
 *   fn: 0 sin, 1 cos, 2 acos, 3 asin, 4 atan2(x, y), 5 hypot(x, y)
 *   which: 0 = sd_crlibm, 1 = glibc                                       */
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

unsigned long long cr_hard_count(void) { return sdcr_hard_count; }
