// Host check: the device log2 port (eb::log2_glibc) against the libm log2
// that CPython's math.log2 calls.  Usage: log2_check N SEED -> prints mismatches.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cmath>
#include "eb_exact.cuh"

static uint64_t s;
static uint64_t next() { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return s; }

int main(int argc, char** argv) {
  long n = argc > 1 ? atol(argv[1]) : 1000000;
  s = argc > 2 ? strtoull(argv[2], 0, 10) * 2654435761ULL + 88172645463325252ULL : 88172645463325252ULL;
  long bad = 0;
  for (long i = 0; i < n; ++i) {
    double x;
    switch (i % 4) {
      case 0: x = eb::as_f64((next() >> 1) % 0x7ff0000000000000ULL); break;        // any positive finite/subnormal
      case 1: x = 1.0 + eb::as_f64(0x3c00000000000000ULL + next() % 0x0c00000000000000ULL); break; // 1 + [2^-63, 2^-15)
      case 2: x = 1.0 + (double)(next() >> 11) * 0x1p-53 * 0.1; break;               // near 1 (both paths)
      default: x = 1.0 + std::ldexp((double)(next() >> 11) * 0x1p-53, (int)(next() % 120) - 40); break; // 1 + ratio (radio domain)
    }
    double a = eb::log2_glibc(x), b = log2(x);
    if (eb::as_u64(a) != eb::as_u64(b) && !(std::isnan(a) && std::isnan(b))) {
      if (bad < 10) fprintf(stderr, "mismatch x=%a port=%a libm=%a\n", x, a, b);
      ++bad;
    }
  }
  printf("%ld\n", bad);
  return 0;
}
