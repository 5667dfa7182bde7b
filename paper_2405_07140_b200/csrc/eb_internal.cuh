// eb_internal.cuh -- shared device-side helpers and launch plumbing.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/edgebatch_b200.h"
#include "eb_exact.cuh"

#define EB_FULL 0xffffffffu

namespace eb {

// Per-context scalars every kernel needs, derived once per instance from
// eb_context exactly as the reference derives them.
struct Ctx {
  Model m;
  double alpha, beta, delta;
  double B_up, B_dn, P_dn, N0_up, N0_dn, T_up, T_dn, fbits;
  double C, M;
  int64_t gpus;
  bool has_cap;
  double cap_s;
  double slots;      // uplink_slot_s + downlink_slot_s  (feasibility.py:112, :214)
};

__device__ __forceinline__ Ctx load_ctx(const eb_context* __restrict__ p) {
  Ctx c;
  c.m.L = p->layers; c.m.d = p->hidden_dim; c.m.heads = p->head_count;
  c.m.head_dim = p->head_dim; c.m.ffn = p->ffn_dim; c.m.bpp = p->bytes_per_param;
  c.alpha = p->alpha; c.beta = p->beta; c.delta = p->delta_ppl;
  c.B_up = p->uplink_band_hz; c.B_dn = p->downlink_band_hz; c.P_dn = p->downlink_power_w;
  c.N0_up = mul(p->noise_density_w_hz, p->uplink_band_hz);     // radio.py:35-37
  c.N0_dn = mul(p->noise_density_w_hz, p->downlink_band_hz);   // radio.py:40-43
  c.T_up = p->uplink_slot_s; c.T_dn = p->downlink_slot_s;
  c.fbits = i2d(p->bits_per_token);
  c.C = p->flops_per_s; c.M = p->memory_bytes; c.gpus = p->gpu_count;
  c.has_cap = p->has_slot_cap != 0; c.cap_s = p->slot_cap_s;
  c.slots = add(c.T_up, c.T_dn);
  return c;
}

// uplink_fraction_per_token radio.py:71-76; returns status (0 ok).
// spectral_efficiency radio.py:63-64 raises ValueError("power, gain and noise
// must be strictly positive") first; `<= 0` is false for NaN, as in Python.
__device__ __forceinline__ int k_up_of(const Ctx& c, double gain, double pup, double* out) {
  if (pup <= 0.0 || gain <= 0.0 || c.N0_up <= 0.0) { *out = 0.0; return EB_ERR_NONPOSITIVE_LINK; }
  double eff = spectral_efficiency(pup, gain, c.N0_up);
  if (eff <= 0.0) { *out = 0.0; return EB_ERR_UPLINK_EFF_ZERO; }    // radio.py:74
  *out = fraction_per_token(c.fbits, c.T_up, c.B_up, eff);
  return 0;
}
// downlink_fraction_per_token radio.py:79-84
__device__ __forceinline__ int k_dn_of(const Ctx& c, double gain, double* out) {
  if (c.P_dn <= 0.0 || gain <= 0.0 || c.N0_dn <= 0.0) { *out = 0.0; return EB_ERR_NONPOSITIVE_LINK; }
  double eff = spectral_efficiency(c.P_dn, gain, c.N0_dn);
  if (eff <= 0.0) { *out = 0.0; return EB_ERR_DOWNLINK_EFF_ZERO; }  // radio.py:82
  *out = fraction_per_token(c.fbits, c.T_dn, c.B_dn, eff);
  return 0;
}

// tau_base feasibility.py:110-114: ((deadline - waiting - slots) * C) / beta
__device__ __forceinline__ double tau_base_of(const Ctx& c, double deadline, double waiting) {
  return div(mul(sub(sub(deadline, waiting), c.slots), c.C), c.beta);
}

// compute seconds of a batch (feasibility.py:216, costs.py:148): beta*flops/C
__device__ __forceinline__ double compute_seconds(const Ctx& c, int64_t flops) {
  return div(mul(c.beta, i2d(flops)), c.C);
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

}  // namespace eb

// Launch accounting shared by all translation units (per handle).
struct eb_handle {
  int device;
  cudaStream_t stream;       // caller-visible stream
  bool own_stream;
  cudaStream_t pipe[3];      // staging pipeline streams (host-memory calls)
  cudaEvent_t ev[3];
  cudaStream_t up;           // host->device uploads of the DFTSP pipeline, back to back
  cudaEvent_t cev[64];       // per-chunk "inputs landed" events (reused modulo 64)
  int num_sms;
  int64_t launches;
  // device scratch (grow-only)
  void* dscratch;
  size_t dscratch_bytes;
  void* pinned;
  size_t pinned_bytes;
  // DFTSP node-count tables (K <= 32, <= 3 classes), one per flag variant
  // (0: pruning off, 1: pruning, 2: pruning + inclusive bound); built on
  // first use (eb_dftsp.cu count_table_kernel)
  void* ctab[3];
  void* ctab_m[3];     // four/five-class tables (eb_dftsp.cu count_table_m_kernel)
  // per pipeline stream device arena of the host-memory DFTSP path (grow-only;
  // chunk c and chunk c+3 share a stream, so reuse is stream-ordered)
  void* arena[3];
  size_t arena_bytes[3];
  // inputs of every chunk of a call (uploads never wait for a buffer to free)
  void* in_arena;
  size_t in_arena_bytes;
  // brute-force evidence counters [combinations checked, prefixes pruned]
  // (eb_exhaustive_counters), device memory, zeroed at handle creation
  unsigned long long* exh_stats;
};

namespace eb {
inline unsigned long long* exh_stats(eb_handle* h) { return h->exh_stats; }
void set_error(const char* fmt, ...);
int cuda_fail(cudaError_t e, const char* what);
int ensure_dscratch(eb_handle* h, size_t bytes);
int ensure_pinned(eb_handle* h, size_t bytes);
}  // namespace eb

#define EB_CUDA(call)                                   \
  do {                                                  \
    cudaError_t _e = (call);                            \
    if (_e != cudaSuccess) return eb::cuda_fail(_e, #call); \
  } while (0)
