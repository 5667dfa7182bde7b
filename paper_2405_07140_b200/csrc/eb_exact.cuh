// eb_exact.cuh -- Python-faithful scalar arithmetic for the edgebatch hot path.
//
// Contract: every value is IEEE binary64 evaluated in
// CPython's order (left-associative, no FMA contraction, no reassociation);
// Python ints are exact, carried here as int64 and converted with
// round-to-nearest-even exactly like int.__float__.  On the device every op
// goes through an explicit _rn intrinsic so that ptxas cannot contract or
// reorder; the library is additionally compiled with -fmad=false.  The same
// header compiles for the host (tests/log2 check) with -ffp-contract=off.
#pragma once
#include <stdint.h>
#include "log2_glibc_table.h"

#if defined(__CUDACC__)
#define EB_HD __host__ __device__ __forceinline__
// out of line on the device: a bulky routine called a few times per instance
#define EB_HD_OUTLINE static __host__ __device__ __noinline__
#else
#define EB_HD static inline
#define EB_HD_OUTLINE static inline
#endif

#if defined(__CUDA_ARCH__)
#define EB_DEV 1
#define EB_LOG2_POLY EB_LOG2_POLY_D
#define EB_LOG2_POLY1 EB_LOG2_POLY1_D
#define EB_LOG2_TAB EB_LOG2_TAB_D
#else
#define EB_LOG2_POLY EB_LOG2_POLY_H
#define EB_LOG2_POLY1 EB_LOG2_POLY1_H
#define EB_LOG2_TAB EB_LOG2_TAB_H
#define EB_DEV 0
#include <math.h>
#include <string.h>
#endif

namespace eb {

EB_HD double add(double a, double b) {
#if EB_DEV
  return __dadd_rn(a, b);
#else
  volatile double r = a + b; return r;
#endif
}
EB_HD double sub(double a, double b) {
#if EB_DEV
  return __dsub_rn(a, b);
#else
  volatile double r = a - b; return r;
#endif
}
EB_HD double mul(double a, double b) {
#if EB_DEV
  return __dmul_rn(a, b);
#else
  volatile double r = a * b; return r;
#endif
}
EB_HD double div(double a, double b) {
#if EB_DEV
  return __ddiv_rn(a, b);
#else
  volatile double r = a / b; return r;
#endif
}
EB_HD double fma_(double a, double b, double c) {
#if EB_DEV
  return __fma_rn(a, b, c);
#else
  return fma(a, b, c);
#endif
}
// float(int): CPython int.__float__ rounds to nearest, ties to even.
EB_HD double i2d(int64_t v) {
#if EB_DEV
  return __ll2double_rn(v);
#else
  return (double)v;  // x86-64 cvtsi2sd honours the default RN mode
#endif
}
EB_HD uint64_t as_u64(double x) {
#if EB_DEV
  return (uint64_t)__double_as_longlong(x);
#else
  uint64_t u; memcpy(&u, &x, 8); return u;
#endif
}
EB_HD double as_f64(uint64_t u) {
#if EB_DEV
  return __longlong_as_double((long long)u);
#else
  double x; memcpy(&x, &u, 8); return x;
#endif
}
EB_HD double fabs_(double x) { return as_f64(as_u64(x) & 0x7fffffffffffffffULL); }

// Python min(a, b) / max(a, b): the first argument wins ties.
EB_HD double pymin(double a, double b) { return (b < a) ? b : a; }
EB_HD double pymax(double a, double b) { return (b > a) ? b : a; }

// max(1.0, abs(a), abs(b)) for leq and its margin variants, on the bit
// patterns: sign-cleared non-NaN doubles order like their (hi, lo) words, so
// two 32-bit compares per operand replace three FP64 max sequences (each a
// DSETP.MAX plus NaN fix-ups on sm_100a).  With a NaN operand the result may
// differ from Python's max, but then a - b is NaN and every comparison
// against the scale is false either way, so leq's value is unchanged.
EB_HD double leq_scale(double a, double b) {
  const uint64_t ua = as_u64(a), ub = as_u64(b);
  const uint32_t ha = (uint32_t)(ua >> 32) & 0x7fffffffu, hb = (uint32_t)(ub >> 32) & 0x7fffffffu;
  const uint32_t la = (uint32_t)ua, lb = (uint32_t)ub;
  uint32_t hm = 0x3ff00000u, lm = 0u;                 // 1.0
  if (ha >= 0x3ff00000u) { hm = ha; lm = la; }        // |a| >= 1.0
  if (hb > hm || (hb == hm && lb > lm)) { hm = hb; lm = lb; }
  return as_f64(((uint64_t)hm << 32) | lm);
}

// feasibility.py:28-30  leq(a, b) = a - b <= 1e-9 * max(1.0, abs(a), abs(b))
EB_HD bool leq(double a, double b) {
  return sub(a, b) <= mul(1e-9, leq_scale(a, b));
}

// ---------------------------------------------------------------------------
// glibc 2.39 log2 (FMA/AVX2 IFUNC variant), the function CPython math.log2
// calls (reference radio.py:68).  Restated from the published ARM
// optimized-routines algorithm (glibc sysdeps/ieee754/dbl-64/e_log2.c) with
// the FMA contractions exactly as gcc emitted them in libm.so.6 (read from
// objdump: see tools/gen_log2_table.py).  Bit-identical to the host libm on
// every input, which tests/test_log2.py checks on >10^7 inputs.
// ---------------------------------------------------------------------------
EB_HD_OUTLINE double log2_glibc(double x) {
  const double InvLn2hi = EB_LOG2_INVLN2HI;
  const double InvLn2lo = EB_LOG2_INVLN2LO;
  uint64_t ix = as_u64(x);
  uint32_t top = (uint32_t)(ix >> 48);
  // |x - 1| < ~0.044: separate polynomial (LO = 1 - 0x1.5b51p-5).
  if (ix - 0x3feea4af00000000ULL < 0x210aa00000000ULL) {
    if (ix == 0x3ff0000000000000ULL) return 0.0;
    const double* B = EB_LOG2_POLY1;
    double r = sub(x, 1.0);
    double hi = mul(InvLn2hi, r);
    double r2 = mul(r, r);
    double t = fma_(InvLn2hi, r, -hi);
    double r4 = mul(r2, r2);
    double p01 = fma_(r, B[1], B[0]);
    double lo = fma_(r, InvLn2lo, t);
    double y = fma_(p01, r2, hi);
    double hy = sub(hi, y);
    double t3 = fma_(p01, r2, hy);
    double p23 = fma_(r, B[3], B[2]);
    lo = add(t3, lo);
    double p45 = fma_(r, B[5], B[4]);
    double q1 = fma_(p45, r2, p23);
    double p67 = fma_(r, B[7], B[6]);
    double p89 = fma_(r, B[9], B[8]);
    double q2 = fma_(p89, r2, p67);
    double q = fma_(q2, r4, q1);
    double res = fma_(q, r4, lo);
    return add(y, res);
  }
  if (top - 0x0010u >= 0x7ff0u - 0x0010u) {
    if ((ix << 1) == 0) return as_f64(0xfff0000000000000ULL);  // log2(+-0) = -inf
    if (ix == 0x7ff0000000000000ULL) return x;             // log2(inf) = inf
    if ((top & 0x8000u) || (top & 0x7ff0u) == 0x7ff0u)    // negative or NaN
      return as_f64(0x7ff8000000000000ULL);
    ix = as_u64(mul(x, 0x1p52));                           // subnormal
    ix -= 52ULL << 52;
  }
  const double* A = EB_LOG2_POLY;
  uint64_t tmp = ix - 0x3fe6000000000000ULL;
  int i = (int)((tmp >> 46) & 63);
  int64_t k = ((int64_t)tmp) >> 52;
  uint64_t iz = ix - (tmp & 0xfff0000000000000ULL);
  double invc = EB_LOG2_TAB[2 * i];
  double logc = EB_LOG2_TAB[2 * i + 1];
  double z = as_f64(iz);
  double kd = i2d(k);
  double t3 = add(kd, logc);
  double r = fma_(z, invc, -1.0);
  double pA01 = fma_(r, A[1], A[0]);
  double t1 = mul(InvLn2hi, r);
  double e = fma_(InvLn2hi, r, -t1);
  double hi = add(t1, t3);
  double d1 = sub(t3, hi);
  double t2 = fma_(r, InvLn2lo, e);
  double r2 = mul(r, r);
  double lo = add(d1, t1);
  lo = add(lo, t2);
  double pA23 = fma_(r, A[3], A[2]);
  double r4 = mul(r2, r2);
  double pA45 = fma_(r, A[5], A[4]);
  double q = fma_(pA23, r2, pA01);
  double p = fma_(pA45, r4, q);
  double y = fma_(r2, p, lo);
  return add(y, hi);
}

// ---------------------------------------------------------------------------
// Exact integer cost model, costs.py:62-112 (Python ints -> int64; callers
// guarantee no overflow, see eb_capi.cu's bound check).
// ---------------------------------------------------------------------------
struct Model {
  int64_t L, d, heads, head_dim, ffn, bpp;
};

// costs.py:62-67
EB_HD int64_t weight_bytes(const Model& m) {
  int64_t per_layer = 4 * m.bpp * m.d * m.head_dim * m.heads + 2 * m.bpp * m.d * m.ffn;
  return m.L * per_layer;
}
// costs.py:70-72
EB_HD int64_t kv_per_token(const Model& m) { return 2 * m.bpp * m.L * m.d; }
// costs.py:87-97
EB_HD int64_t flops_initial(const Model& m, int64_t s) {
  int64_t d = m.d, f = m.ffn;
  int64_t per_layer = 6 * s * d * d + (4 * s * s * d + 2 * s * d * d) + 4 * s * d * f;
  return m.L * per_layer;
}
// costs.py:100-112 (closed form; equals the stepwise sum exactly)
EB_HD int64_t flops_autoregressive(const Model& m, int64_t s, int64_t n) {
  int64_t d = m.d;
  int64_t base = 8 * d * d + 4 * s * d + 4 * d * m.ffn;
  return m.L * (n - 1) * (base + 2 * d * n);
}
// feasibility.py:155 gen_base
EB_HD int64_t gen_base(const Model& m, int64_t s) {
  return 8 * m.d * m.d + 4 * s * m.d + 4 * m.d * m.ffn;
}

// ---------------------------------------------------------------------------
// Link math, radio.py:64-84.
//   eta  = log2(1.0 + p * g / N0)          (N0 = density * band, radio.py:35-43)
//   frac = float(bits) / (slot * band * eta)
// Returns eta; frac via out-param (only meaningful when eta > 0).
// ---------------------------------------------------------------------------
EB_HD double spectral_efficiency(double p, double g, double noise_w) {
  return log2_glibc(add(1.0, div(mul(p, g), noise_w)));
}
EB_HD double fraction_per_token(double bits, double slot, double band, double eta) {
  return div(bits, mul(mul(slot, band), eta));
}

}  // namespace eb
