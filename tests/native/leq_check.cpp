// Host check: eb::leq (integer max(1, |a|, |b|) scale, csrc/eb_exact.cuh)
// against feasibility.py:28-30 restated with Python's max chain, plus the
// margin form the level/prefix bounds use.  Usage: leq_check N SEED -> prints
// mismatches.  Covers NaN, +-inf, +-0, subnormals and values straddling 1.0.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include "eb_exact.cuh"

static uint64_t s;
static uint64_t next() { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return s; }
static double pymax3(double a, double b, double c) { double m = a; if (b > m) m = b; if (c > m) m = c; return m; }
static bool leq_py(double a, double b) { return (a - b) <= 1e-9 * pymax3(1.0, std::fabs(a), std::fabs(b)); }
static bool fails_py(double a, double b) { return (a - b) > 1.00001e-9 * pymax3(1.0, std::fabs(a), std::fabs(b)); }
static bool fails_dev(double a, double b) { return eb::sub(a, b) > eb::mul(1.00001e-9, eb::leq_scale(a, b)); }

int main(int argc, char** argv) {
  long n = argc > 1 ? atol(argv[1]) : 1000000;
  s = argc > 2 ? strtoull(argv[2], 0, 10) * 2654435761ULL + 88172645463325252ULL : 88172645463325252ULL;
  const double sp[] = {0.0, -0.0, 1.0, -1.0, 1.0000000000000002, 0.9999999999999999, INFINITY, -INFINITY, NAN, -NAN,
                       5e-324, -5e-324, 2.2250738585072014e-308, 1e300, -1e300, 1e-9, 1 + 1e-9, 1 - 1e-9, 0.5, 2.0, 1e9};
  const int ns = sizeof(sp) / sizeof(sp[0]);
  long bad = 0;
  auto check = [&](double a, double b) {
    if (eb::leq(a, b) != leq_py(a, b) || fails_dev(a, b) != fails_py(a, b)) {
      if (bad < 10) fprintf(stderr, "mismatch a=%a b=%a\n", a, b);
      ++bad;
    }
  };
  for (int i = 0; i < ns; ++i)
    for (int j = 0; j < ns; ++j) check(sp[i], sp[j]);
  for (long k = 0; k < n; ++k) {
    const uint64_t r1 = next(), r2 = next();
    double a, b;
    switch (k % 4) {
      case 0: a = eb::as_f64(r1); b = eb::as_f64(r2); break;                       // any bit pattern
      case 1: a = (double)(r1 % 100000) / 1000.0; b = a * (1 + ((double)(int)(r2 % 2001) - 1000) * 1e-12); break;
      case 2: a = std::ldexp((double)(r1 % 1000003), (int)(r2 % 80) - 40);          // around the 1e-9 slack
              b = std::nextafter(a, (r2 & 1) ? INFINITY : -INFINITY) * (1 + ((double)(int)(r1 % 7) - 3) * 1e-9); break;
      default: a = (double)(r1 % 3) - 1.0 + (double)(r2 % 1000) * 1e-12; b = (double)(r2 % 3) - 1.0; break;
    }
    check(a, b);
  }
  printf("%ld\n", bad);
  return 0;
}
