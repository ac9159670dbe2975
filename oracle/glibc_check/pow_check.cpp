// Host checker (test infrastructure): the device's glibc-pow restatement
// (paper_1306_6291_b200/csrc/sd_glibc_pow.h, compiled here as plain C++)
// against the installed libm's pow, bit for bit.
//   pow_check <n_random> <seed>   -> prints "checked N mismatches M" and
//   the first mismatches; exit 0 iff M == 0.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>

#include "../../paper_1306_6291_b200/csrc/sd_glibc_pow.h"

static uint64_t bits(double x) { uint64_t b; std::memcpy(&b, &x, 8); return b; }
static double from(uint64_t b) { double x; std::memcpy(&x, &b, 8); return x; }

static long long checked = 0, bad = 0;
static void check(double x, double y) {
  volatile double yy = y;  // keep gcc from expanding pow(x, 2.0) into x*x
  const double ref = std::pow(x, yy);
  const double got = sd_glibc::pow(x, y);
  checked++;
  if (bits(ref) != bits(got) && !(std::isnan(ref) && std::isnan(got))) {
    if (bad < 20)
      std::printf("MISMATCH x=%a y=%g libm=%a ours=%a\n", x, y, ref, got);
    bad++;
  }
}

int main(int argc, char** argv) {
  const long long n = argc > 1 ? std::atoll(argv[1]) : 1000000;
  const unsigned seed = argc > 2 ? (unsigned)std::atoi(argv[2]) : 1;
  std::mt19937_64 rng(seed);
  const double ys[] = {2.0, 3.0, 6.0, 4.0, 5.0, 1.0};
  // edge values: zeros, subnormals, normal boundaries, huge, over/underflow
  // thresholds of each power, exact integers, powers of two, the table
  // boundaries of z (OFF + i 2^45) and their neighbours
  for (double y : ys) {
    const double e[] = {0.0, -0.0, 1.0, -1.0, 0.5, 2.0, 3.0, 1e-300, 1e300, 4.9e-324,
                        2.2250738585072014e-308, 2.2250738585072009e-308, 1.3407807929942596e154,
                        1.3407807929942597e154, 5.6e102, 5.7e102, 1e-155, 1e-160, 1e-170,
                        1.4916681462400413e-154, 1e51, 3.4e51, -7.0, -1e-200, INFINITY,
                        -INFINITY, NAN};
    for (double x : e) { check(x, y); check(-x, y); }
    for (uint64_t i = 0; i < 256; i++) {
      const uint64_t b = 0x3fe6955500000000ULL + i * (1ULL << 45);
      for (int d = -2; d <= 2; d++) check(from(b + d), y);
    }
  }
  for (long long t = 0; t < n; t++) {
    const double y = ys[t % 3];
    const uint64_t r = rng();
    double x;
    switch ((r >> 60) & 7) {
      case 0: x = from(r & 0x7fffffffffffffffULL); break;               // any bit pattern
      case 1: x = std::ldexp((double)(r >> 11), -53); break;            // [0, 1)
      case 2: x = std::ldexp((double)(r >> 11), -53) * 20.0 - 10.0; break;
      case 3: x = std::ldexp((double)((r >> 11) | 1), -53 - (int)(r & 1023)); break;
      case 4: x = (double)((int64_t)(r >> 40) - (1LL << 23)); break;    // integers
      case 5: x = std::ldexp(1.0 + std::ldexp((double)(r >> 12), -52), (int)(r & 511) - 256); break;
      default: {
        std::normal_distribution<double> nd(0.0, 1.0);
        x = nd(rng) * std::ldexp(1.0, (int)(r & 63) - 32);
      }
    }
    if (std::isnan(x) || std::isinf(x)) continue;
    check(x, y);
  }
  std::printf("checked %lld mismatches %lld\n", checked, bad);
  return bad == 0 ? 0 : 1;
}
