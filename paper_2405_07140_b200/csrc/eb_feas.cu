// eb_feas.cu -- K1 (link math, coefficients, admission) and K2 (batched
// check_direct / check_knapsack / batch_cost) plus the benchmark-batching
// baselines (baselines.py).  One thread per independent unit (request row,
// subset, plan or queue); every formula follows the reference statement
// order via the eb_exact.cuh primitives.
#include <climits>

#include "eb_internal.cuh"

namespace eb {
namespace {

__device__ __forceinline__ int ctx_at(const int32_t* idx, int64_t i, int n_ctx) {
  int c = idx ? idx[i] : 0;
  return (c < 0 || c >= n_ctx) ? -1 : c;
}

// ---- link math radio.py:64-101 ------------------------------------------
// Block-strided tiles of 128 requests: the SoA columns are read coalesced (one
// element per thread), the six results of each request are staged in shared
// memory column-major ([field][request], conflict-free writes), and the tile's
// 6 x 128 doubles -- contiguous in the ABI's row-major out[j*6 + k] -- leave as
// coalesced 16-byte stores (the ragged last tile element-wise).
constexpr int kLinkTile = 128;

__global__ void __launch_bounds__(kLinkTile) link_kernel(const eb_context* ctxs, int n_ctx, eb_requests req,
                                                         int64_t n, const int32_t* req_ctx, int32_t* status,
                                                         double* out) {
  __shared__ double tile[6][kLinkTile + 1];
  for (int64_t t0 = (int64_t)blockIdx.x * kLinkTile; t0 < n; t0 += (int64_t)gridDim.x * kLinkTile) {
    const int64_t j = t0 + threadIdx.x;
    const int rows = (int)min((int64_t)kLinkTile, n - t0);
    double o[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    bool write = false;
    if (j < n) {
      const int ci = ctx_at(req_ctx, j, n_ctx);
      if (ci < 0) {
        status[j] = EB_ERR_INVALID_ARG;     // row left untouched, as before
      } else {
        const Ctx c = load_ctx(&ctxs[ci]);
        const double g = req.channel_gain[j], pu = req.uplink_power_w[j];
        int st = 0;
        double eu = 0.0, ed = 0.0, ku = 0.0, kd = 0.0;
        // radio.py:63-64: nonpositive power/gain/noise raise before log2
        if (pu <= 0.0 || g <= 0.0 || c.N0_up <= 0.0) st = EB_ERR_NONPOSITIVE_LINK;
        else {
          eu = spectral_efficiency(pu, g, c.N0_up);
          if (eu <= 0.0) st = EB_ERR_UPLINK_EFF_ZERO; else ku = fraction_per_token(c.fbits, c.T_up, c.B_up, eu);
        }
        if (c.P_dn <= 0.0 || g <= 0.0 || c.N0_dn <= 0.0) { if (!st) st = EB_ERR_NONPOSITIVE_LINK; }
        else {
          ed = spectral_efficiency(c.P_dn, g, c.N0_dn);
          if (ed <= 0.0) { if (!st) st = EB_ERR_DOWNLINK_EFF_ZERO; } else kd = fraction_per_token(c.fbits, c.T_dn, c.B_dn, ed);
        }
        o[0] = eu; o[1] = ed; o[2] = ku; o[3] = kd;
        o[4] = mul(i2d(req.prompt_tokens[j]), ku);   // min_uplink_fraction radio.py:87-94
        o[5] = mul(i2d(req.output_tokens[j]), kd);   // min_downlink_fraction radio.py:97-101
        status[j] = st;
        write = true;
      }
    }
    const bool all = __syncthreads_and(write || j >= n) && rows == kLinkTile;
#pragma unroll
    for (int k = 0; k < 6; ++k) tile[k][threadIdx.x] = o[k];
    __syncthreads();
    double* base = out + 6 * t0;
    if (all && ((uintptr_t)base & 15) == 0) {
      // 3 x 128 double2 stores cover the tile; pair q holds flat values 2q, 2q+1
      double2* b2 = reinterpret_cast<double2*>(base);
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        const int q = r * kLinkTile + threadIdx.x;
        const int f0 = 2 * q, f1 = 2 * q + 1;
        b2[q] = make_double2(tile[f0 % 6][f0 / 6], tile[f1 % 6][f1 / 6]);
      }
    } else {
      for (int f = threadIdx.x; f < 6 * rows; f += kLinkTile) {
        const int r = f / 6;
        if (req_ctx && ctx_at(req_ctx, t0 + r, n_ctx) < 0) continue;   // invalid rows stay untouched
        base[f] = tile[f % 6][r];
      }
    }
    __syncthreads();
  }
}

// ---- derive_coefficients feasibility.py:133-167 (thread per instance) ----
__global__ void coeff_kernel(const eb_context* ctxs, int n_ctx, int64_t n_inst, const int64_t* off,
                             const int32_t* ctx_index, int64_t req_base, eb_requests req,
                             const int64_t* padded_len, int32_t* status, int32_t* err_index,
                             double* out_scalar, double* out_req) {
  // one warp per instance, lanes over its rows (coalesced SoA loads); the
  // reference's sequential scans become ballots for the first offending row
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < n_inst; i += warps) {
    const int ci = ctx_at(ctx_index, i, n_ctx);
    if (ci < 0) { if (lane == 0) status[i] = EB_ERR_INVALID_ARG; continue; }
    const Ctx c = load_ctx(&ctxs[ci]);
    const int64_t lo = off[i] - req_base, hi = off[i + 1] - req_base;
    int64_t padded = padded_len ? padded_len[i] : 0;
    int st = 0, err = -1;
    if (padded <= 0) {
      int m = 0;
      for (int64_t r = lo + lane; r < hi; r += 32) m = max(m, req.prompt_tokens[r]);
      padded = (int64_t)__reduce_max_sync(EB_FULL, m);
    } else {
      for (int64_t r0 = lo; r0 < hi && !st; r0 += 32) {                 // feasibility.py:142-143
        const int64_t r = r0 + lane;
        const unsigned bad = __ballot_sync(EB_FULL, r < hi && req.prompt_tokens[r] > padded);
        if (bad) { st = EB_ERR_PADDED_TOO_SMALL; err = (int)(r0 - lo) + __ffs(bad) - 1; }
      }
    }
    const int64_t m1 = weight_bytes(c.m);
    const double headroom = sub(div(c.M, c.alpha), i2d(m1));
    if (!st && headroom < 0) st = EB_ERR_WEIGHTS_DO_NOT_FIT;
    if (!st) {
      if (lane == 0) {
        double* sc = out_scalar + 6 * i;
        const int64_t kv = kv_per_token(c.m);
        const int64_t gb = gen_base(c.m, padded);
        sc[0] = div(headroom, i2d(kv));
        sc[1] = i2d(flops_initial(c.m, padded) - c.m.L * gb);
        sc[2] = i2d(c.m.L * (gb - 2 * c.m.d));
        sc[3] = i2d(2 * c.m.L * c.m.d);
        sc[4] = c.has_cap ? div(mul(c.cap_s, c.C), c.beta) : __longlong_as_double(0x7ff8000000000000LL);
        sc[5] = (double)padded;
      }
      // feasibility.py:164-166 in pool order: rows before the first link error are written
      for (int64_t r0 = lo; r0 < hi; r0 += 32) {
        const int64_t r = r0 + lane;
        double ku = 0.0, kd = 0.0;
        int s2 = 0;
        if (r < hi) {
          s2 = k_up_of(c, req.channel_gain[r], req.uplink_power_w[r], &ku);
          if (!s2) s2 = k_dn_of(c, req.channel_gain[r], &kd);
        }
        const unsigned bad = __ballot_sync(EB_FULL, s2 != 0);
        const int first = bad ? __ffs(bad) - 1 : 32;
        if (r < hi && lane < first) {
          double* o = out_req + 4 * r;
          o[0] = ku; o[1] = kd;
          o[2] = tau_base_of(c, req.deadline_s[r], req.waiting_s[r]);
          o[3] = mul(i2d(req.prompt_tokens[r]), ku);
        }
        if (bad) { st = __shfl_sync(EB_FULL, s2, first); err = (int)(r0 - lo) + first; break; }
      }
    }
    if (lane == 0) {
      status[i] = st;
      if (err_index) err_index[i] = err;
    }
  }
}

// check_direct on rows (given in subset order), feasibility.py:192-223.
// Returns 1/0, or -status on a link-math error; fills met (up, dn, mem, cs).
template <typename RowFn>
__device__ int check_direct_rows(const Ctx& c, const eb_requests& req, int z, RowFn row,
                                 int64_t padded, double* met) {
  double up = 0.0, dn = 0.0;
  int64_t sn = 0;
  for (int j = 0; j < z; ++j) {
    int64_t r = row(j);
    double ku, kd;
    int st = k_up_of(c, req.channel_gain[r], req.uplink_power_w[r], &ku);
    if (!st) st = k_dn_of(c, req.channel_gain[r], &kd);
    if (st) return -st;
    up = add(up, mul(i2d(req.prompt_tokens[r]), ku));
    dn = add(dn, mul(i2d(req.output_tokens[r]), kd));
    sn += req.output_tokens[r];
  }
  int64_t kv = kv_per_token(c.m);
  int64_t mem = weight_bytes(c.m) + kv * padded * z;
  mem += kv * sn;
  int64_t flops = z ? (int64_t)z * flops_initial(c.m, padded) : 0;
  for (int j = 0; j < z; ++j) flops += flops_autoregressive(c.m, padded, req.output_tokens[row(j)]);
  double cs = compute_seconds(c, flops);
  if (met) { met[0] = up; met[1] = dn; met[2] = mul(c.alpha, i2d(mem)); met[3] = cs; }
  if (!(leq(up, 1.0) && leq(dn, 1.0))) return 0;
  if (!leq(mul(c.alpha, i2d(mem)), c.M)) return 0;
  if (c.has_cap && !leq(cs, c.cap_s)) return 0;
  for (int j = 0; j < z; ++j) {
    int64_t r = row(j);
    if (!leq(add(add(req.waiting_s[r], c.slots), cs), req.deadline_s[r])) return 0;
  }
  return 1;
}

__global__ void check_direct_kernel(const eb_context* ctxs, int n_ctx, eb_requests req,
                                    int64_t n_sub, const int64_t* sub_off, const int32_t* members,
                                    const int32_t* sub_ctx, const int64_t* padded_len,
                                    int32_t* status, uint8_t* ok, double* met) {
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n_sub;
       s += (int64_t)gridDim.x * blockDim.x) {
    int ci = ctx_at(sub_ctx, s, n_ctx);
    if (ci < 0) { status[s] = EB_ERR_INVALID_ARG; ok[s] = 0; continue; }
    const Ctx c = load_ctx(&ctxs[ci]);
    int64_t lo = sub_off[s];
    int z = (int)(sub_off[s + 1] - lo);
    int res = check_direct_rows(c, req, z, [&](int j) { return (int64_t)members[lo + j]; },
                                padded_len[s], met ? met + 4 * s : nullptr);
    status[s] = res < 0 ? -res : 0;
    ok[s] = res > 0;
  }
}

// check_knapsack feasibility.py:170-189 given coefficients.
__global__ void check_knapsack_kernel(int64_t n_sub, const int64_t* sub_off, const int32_t* prompt,
                                      const int32_t* output, const double* k_up, const double* k_dn,
                                      const double* coeff, const int32_t* zv, const double* tau_min,
                                      uint8_t* ok) {
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n_sub;
       s += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = sub_off[s];
    int m = (int)(sub_off[s + 1] - lo);
    int z = zv[s];
    if (m != z) { ok[s] = 0; continue; }
    const double* co = coeff + 6 * s;
    double k2 = co[0], k3 = co[1], k4 = co[2], k5 = co[3], sb = co[4];
    int64_t padded = (int64_t)co[5];
    double up = 0.0, dn = 0.0, lat = 0.0;
    int64_t mem = 0;
    for (int j = 0; j < m; ++j) {
      int64_t r = lo + j;
      double fn = i2d(output[r]);
      up = add(up, mul(k_up[r], i2d(prompt[r])));
      dn = add(dn, mul(k_dn[r], fn));
      mem += output[r];
      lat = add(lat, add(mul(k4, fn), mul(mul(k5, fn), fn)));
    }
    double fz = i2d(z);
    double slot = (sb != sb) ? __longlong_as_double(0x7ff0000000000000LL) : sub(sb, mul(k3, fz));
    double cap = pymin(tau_min[s], slot);
    double mem_budget = sub(k2, i2d(padded * z));
    ok[s] = leq(up, 1.0) && leq(dn, 1.0) && leq(i2d(mem), mem_budget) && leq(lat, cap);
  }
}

// sim._dftsp_candidates sim.py:264-274 (accuracy filter + alone prefilter).
__global__ void __launch_bounds__(128) admission_kernel(const eb_context* ctxs, int n_ctx, int64_t n_inst,
                                                        const int64_t* off, const int32_t* ctx_index,
                                                        int64_t req_base, eb_requests req, int acc_check,
                                                        int prefilter, int32_t* status, uint8_t* keep) {
  // Each block owns one contiguous range of rows, walked in tiles of 128.
  // The instance of a row is found by binary search in a shared-memory
  // window of the offsets starting at the instance of the tile's first row;
  // that instance is carried from tile to tile (one global search per block,
  // not per tile), so no tile waits on a chain of dependent global loads.
  constexpr int W = 128;
  __shared__ int64_t win[W + 1];
  __shared__ int64_t s_i0;
  const int64_t n_rows = off[n_inst] - off[0];
  const int64_t per_blk = ((n_rows + gridDim.x - 1) / gridDim.x + W - 1) / W * W;
  const int64_t q_lo = (int64_t)blockIdx.x * per_blk;
  const int64_t q_hi = q_lo + per_blk < n_rows ? q_lo + per_blk : n_rows;
  if (q_lo >= n_rows) return;
  auto global_search = [&](int64_t row, int64_t lo) -> int64_t {   // off[lo] <= row < off[lo + 1]
    int64_t hi = n_inst;
    while (hi - lo > 1) { const int64_t mid = (lo + hi) >> 1; if (off[mid] <= row) lo = mid; else hi = mid; }
    return lo;
  };
  if (threadIdx.x == 0) s_i0 = global_search(off[0] + q_lo, 0);
  for (int64_t t0 = q_lo; t0 < q_hi; t0 += W) {
    __syncthreads();                 // s_i0 is set; the previous tile is done with win
    const int64_t i0 = s_i0;
    for (int k = threadIdx.x; k <= W; k += blockDim.x) win[k] = (i0 + k <= n_inst) ? off[i0 + k] : INT64_MAX;
    __syncthreads();
    auto inst_of = [&](int64_t row) -> int64_t {
      if (row < win[W]) {
        int a = 0, b = W;            // win[a] <= row < win[a + 1]
        while (b - a > 1) { const int mid = (a + b) >> 1; if (win[mid] <= row) a = mid; else b = mid; }
        return i0 + a;
      }
      return global_search(row, i0 + W);   // more than W (empty) instances in the tile
    };
    if (threadIdx.x == 0 && t0 + W < q_hi) s_i0 = inst_of(off[0] + t0 + W);   // next tile's first row
    const int64_t q = t0 + threadIdx.x;
    if (q < q_hi) {
      const int64_t row = off[0] + q;
      const int64_t inst = inst_of(row);
      const int ci = ctx_at(ctx_index, inst, n_ctx);
      const int64_t r = row - req_base;
      if (ci < 0) {
        status[r] = EB_ERR_INVALID_ARG;
        keep[r] = 0;
      } else {
        const Ctx c = load_ctx(&ctxs[ci]);
        int st = 0;
        bool k = true;
        if (acc_check) {
          const double tol = req.tolerance[r];
          if (c.delta < 0 || tol < 0) { st = EB_ERR_INVALID_ARG; k = false; }   // catalog.py:153-154
          else k = c.delta <= tol;                                              // catalog.py:155
        }
        if (k && prefilter) {
          const int res = check_direct_rows(c, req, 1, [&](int) { return r; }, (int64_t)req.prompt_tokens[r], nullptr);
          if (res < 0) { st = -res; k = false; } else k = res > 0;
        }
        status[r] = st;
        keep[r] = k;
      }
    }
    __syncthreads();
  }
}

// batch_cost costs.py:131-148
__global__ void batch_cost_kernel(const eb_context* ctxs, int n_ctx, int64_t n, const int64_t* off,
                                  const int32_t* prompt, const int32_t* output, const int64_t* padded,
                                  const int64_t* copies, const int32_t* plan_ctx, double* out) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    int ci = ctx_at(plan_ctx, p, n_ctx);
    if (ci < 0) { out[2 * p] = out[2 * p + 1] = __longlong_as_double(0x7ff8000000000000LL); continue; }
    const Ctx c = load_ctx(&ctxs[ci]);
    int64_t lo = off[p], hi = off[p + 1];
    int64_t b = hi - lo, pl = padded[p];
    int64_t sn = 0;
    for (int64_t r = lo; r < hi; ++r) sn += output[r];
    int64_t kv = kv_per_token(c.m);
    int64_t mem = (copies ? copies[p] : 1) * weight_bytes(c.m) + kv * pl * b + kv * sn;
    int64_t flops = b ? b * flops_initial(c.m, pl) : 0;
    for (int64_t r = lo; r < hi; ++r) flops += flops_autoregressive(c.m, pl, output[r]);
    out[2 * p] = mul(c.alpha, i2d(mem));
    out[2 * p + 1] = compute_seconds(c, flops);
  }
}

// CPython float // float (Objects/floatobject.c _float_div_mod)
__device__ double py_floordiv(double vx, double wx) {
  double mod = fmod(vx, wx);
  double dv = div(sub(vx, mod), wx);
  if (mod != 0.0) {
    if ((wx < 0) != (mod < 0)) { mod = add(mod, wx); dv = sub(dv, 1.0); }
  }
  double fd;
  if (dv != 0.0) {
    fd = floor(dv);
    if (sub(dv, fd) > 0.5) fd = add(fd, 1.0);
  } else {
    fd = copysign(0.0, div(vx, wx));
  }
  return fd;
}

// static_batch_size baselines.py:51-65
__global__ void static_b_kernel(const eb_context* ctxs, int n, const double* slot_s,
                                const int64_t* s_max, const int64_t* n_max, int64_t* out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const Ctx c = load_ctx(&ctxs[i]);
    int64_t m1 = weight_bytes(c.m);
    if (mul(c.alpha, i2d(m1)) > c.M) { out[i] = 0; continue; }
    int64_t kvr = kv_per_token(c.m) * (s_max[i] + n_max[i]);
    double mb = py_floordiv(sub(div(c.M, c.alpha), i2d(m1)), i2d(kvr));
    int64_t fpr = flops_initial(c.m, s_max[i]) + flops_autoregressive(c.m, s_max[i], n_max[i]);
    double lb = div(mul(slot_s[i], c.C), mul(c.beta, i2d(fpr)));
    int64_t mem_bound = (int64_t)mb, lat_bound = (int64_t)lb;   // int() truncation
    int64_t b = min(mem_bound, lat_bound);
    out[i] = b > 0 ? b : 0;
  }
}

// stb_schedule baselines.py:68-87 (thread per queue)
__global__ void stb_kernel(const eb_context* ctxs, int n_ctx, int64_t n_inst, const int64_t* off,
                           const int32_t* ctx_index, int64_t req_base, eb_requests req, const int64_t* bv,
                           int acc_check, int32_t* status, uint8_t* sel) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_inst;
       i += (int64_t)gridDim.x * blockDim.x) {
    int ci = ctx_at(ctx_index, i, n_ctx);
    int64_t lo = off[i] - req_base, hi = off[i + 1] - req_base;
    for (int64_t r = lo; r < hi; ++r) sel[r] = 0;
    if (ci < 0) { status[i] = EB_ERR_INVALID_ARG; continue; }
    const Ctx c = load_ctx(&ctxs[ci]);
    int64_t chosen = 0, b = bv[i];
    int st = 0;
    for (int64_t r = lo; r < hi; ++r) {
      if (chosen >= b) break;
      if (acc_check && c.delta > req.tolerance[r]) continue;
      double ku, kd;
      st = k_up_of(c, req.channel_gain[r], req.uplink_power_w[r], &ku);
      if (st) break;
      if (mul(i2d(req.prompt_tokens[r]), ku) > 1.0) continue;
      st = k_dn_of(c, req.channel_gain[r], &kd);
      if (st) break;
      if (mul(i2d(req.output_tokens[r]), kd) > 1.0) continue;
      sel[r] = 1;
      ++chosen;
    }
    status[i] = st;
  }
}

// nob_assign baselines.py:90-121 (thread per queue)
__global__ void nob_kernel(const eb_context* ctxs, int n_ctx, int64_t n_inst, const int64_t* off,
                           const int32_t* ctx_index, int64_t req_base, eb_requests req, const double* now,
                           int acc_check, const int32_t* n_dev, int max_dev, double* busy, int32_t* status, int8_t* action,
                           double* completion, int32_t* order) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_inst;
       i += (int64_t)gridDim.x * blockDim.x) {
    int ci = ctx_at(ctx_index, i, n_ctx);
    int64_t lo = off[i] - req_base, hi = off[i + 1] - req_base;
    for (int64_t r = lo; r < hi; ++r) { action[r] = 0; completion[r] = 0.0; order[r] = -1; }
    if (ci < 0) { status[i] = EB_ERR_INVALID_ARG; continue; }
    const Ctx c = load_ctx(&ctxs[ci]);
    int G = n_dev ? n_dev[i] : (int)c.gpus;
    if (G > max_dev) { status[i] = EB_ERR_INVALID_ARG; continue; }
    double* bu = busy + (int64_t)i * max_dev;
    double fpd = div(c.C, i2d(c.gpus)), mpd = div(c.M, i2d(c.gpus));   // per_gpu_* costs.py:30-36
    double ready = add(now[i], c.T_up);
    // idle list in device order (baselines.py:102), consumed FIFO
    int head = 0, pos = 0;
    for (int64_t r = lo; r < hi; ++r) {
      // next idle device at or after `head`
      while (head < G && !(bu[head] <= ready)) ++head;
      if (head >= G) break;
      if (acc_check && c.delta > req.tolerance[r]) continue;
      int64_t s = req.prompt_tokens[r], no = req.output_tokens[r];
      int64_t kv = kv_per_token(c.m);
      int64_t mem = weight_bytes(c.m) + kv * s + kv * no;
      int64_t fl = flops_initial(c.m, s) + flops_autoregressive(c.m, s, no);
      double cm = mul(c.alpha, i2d(mem));
      double lat = div(mul(c.beta, i2d(fl)), fpd);
      if (!leq(cm, mpd)) { action[r] = 2; continue; }
      int g = head++;
      double start = pymax(bu[g], ready);
      bu[g] = add(start, lat);
      completion[r] = add(bu[g], c.T_dn);
      action[r] = 1;
      order[r] = pos++;
    }
    status[i] = 0;
  }
}

inline unsigned grid_for(eb_handle* h, int64_t n, int threads) {
  int64_t g = (n + threads - 1) / threads;
  int64_t cap = (int64_t)h->num_sms * 16;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (unsigned)g;
}

}  // namespace

#define EB_LAUNCHED() do { EB_CUDA(cudaGetLastError()); h->launches += 1; } while (0)

int launch_link(eb_handle* h, cudaStream_t st, const eb_context* ctxs, int n_ctx, const eb_requests& req,
                int64_t n, const int32_t* req_ctx, int32_t* status, double* out) {
  if (n <= 0) return EB_OK;
  link_kernel<<<grid_for(h, n, kLinkTile), kLinkTile, 0, st>>>(ctxs, n_ctx, req, n, req_ctx, status, out);
  EB_LAUNCHED();
  return EB_OK;
}
int launch_coeff(eb_handle* h, cudaStream_t st, const eb_context* ctxs, int n_ctx, int64_t n_inst,
                 const int64_t* off, const int32_t* ci, int64_t req_base, const eb_requests& req,
                 const int64_t* padded, int32_t* status, int32_t* err, double* sc, double* rq) {
  if (n_inst <= 0) return EB_OK;
  coeff_kernel<<<grid_for(h, n_inst * 32, 128), 128, 0, st>>>(ctxs, n_ctx, n_inst, off, ci, req_base, req, padded,
                                                        status, err, sc, rq);
  EB_LAUNCHED();
  return EB_OK;
}
int launch_check_direct(eb_handle* h, cudaStream_t st, const eb_context* ctxs, int n_ctx,
                        const eb_requests& req, int64_t n_sub, const int64_t* sub_off,
                        const int32_t* members, const int32_t* sub_ctx, const int64_t* padded,
                        int32_t* status, uint8_t* ok, double* met) {
  if (n_sub <= 0) return EB_OK;
  check_direct_kernel<<<grid_for(h, n_sub, 128), 128, 0, st>>>(ctxs, n_ctx, req, n_sub, sub_off, members,
                                                              sub_ctx, padded, status, ok, met);
  EB_LAUNCHED();
  return EB_OK;
}
int launch_check_knapsack(eb_handle* h, cudaStream_t st, int64_t n_sub, const int64_t* sub_off,
                          const int32_t* prompt, const int32_t* output, const double* ku,
                          const double* kd, const double* coeff, const int32_t* z,
                          const double* tau_min, uint8_t* ok) {
  if (n_sub <= 0) return EB_OK;
  check_knapsack_kernel<<<grid_for(h, n_sub, 128), 128, 0, st>>>(n_sub, sub_off, prompt, output, ku, kd,
                                                                coeff, z, tau_min, ok);
  EB_LAUNCHED();
  return EB_OK;
}
int launch_admission(eb_handle* h, cudaStream_t st, const eb_context* ctxs, int n_ctx, int64_t n_inst,
                     int64_t n_rows, const int64_t* off, const int32_t* ci, int64_t req_base,
                     const eb_requests& req, int acc, int pre, int32_t* status, uint8_t* keep) {
  if (n_inst <= 0 || n_rows <= 0) return EB_OK;
  admission_kernel<<<grid_for(h, n_rows, 128), 128, 0, st>>>(ctxs, n_ctx, n_inst, off, ci, req_base, req,
                                                            acc, pre, status, keep);
  EB_LAUNCHED();
  return EB_OK;
}
int launch_batch_cost(eb_handle* h, cudaStream_t st, const eb_context* ctxs, int n_ctx, int64_t n,
                      const int64_t* off, const int32_t* prompt, const int32_t* output,
                      const int64_t* padded, const int64_t* copies, const int32_t* pc, double* out) {
  if (n <= 0) return EB_OK;
  batch_cost_kernel<<<grid_for(h, n, 128), 128, 0, st>>>(ctxs, n_ctx, n, off, prompt, output, padded, copies,
                                                        pc, out);
  EB_LAUNCHED();
  return EB_OK;
}
int launch_static_b(eb_handle* h, cudaStream_t st, const eb_context* ctxs, int n, const double* slot,
                    const int64_t* smax, const int64_t* nmax, int64_t* out) {
  if (n <= 0) return EB_OK;
  static_b_kernel<<<grid_for(h, n, 128), 128, 0, st>>>(ctxs, n, slot, smax, nmax, out);
  EB_LAUNCHED();
  return EB_OK;
}
int launch_stb(eb_handle* h, cudaStream_t st, const eb_context* ctxs, int n_ctx, int64_t n_inst,
               const int64_t* off, const int32_t* ci, int64_t req_base, const eb_requests& req,
               const int64_t* b, int acc, int32_t* status, uint8_t* sel) {
  if (n_inst <= 0) return EB_OK;
  stb_kernel<<<grid_for(h, n_inst, 128), 128, 0, st>>>(ctxs, n_ctx, n_inst, off, ci, req_base, req, b, acc,
                                                      status, sel);
  EB_LAUNCHED();
  return EB_OK;
}
int launch_nob(eb_handle* h, cudaStream_t st, const eb_context* ctxs, int n_ctx, int64_t n_inst,
               const int64_t* off, const int32_t* ci, int64_t req_base, const eb_requests& req,
               const double* now, int acc, const int32_t* n_dev, int max_dev, double* busy, int32_t* status,
               int8_t* action, double* completion, int32_t* order) {
  if (n_inst <= 0) return EB_OK;
  nob_kernel<<<grid_for(h, n_inst, 128), 128, 0, st>>>(ctxs, n_ctx, n_inst, off, ci, req_base, req, now, acc,
                                                      n_dev, max_dev, busy, status, action, completion, order);
  EB_LAUNCHED();
  return EB_OK;
}

}  // namespace eb
