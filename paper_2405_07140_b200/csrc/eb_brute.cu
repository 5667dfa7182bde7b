// eb_brute.cu -- K4: brute-force subset search (reference
// exhaustive_optimal(mode="subsets"), dftsp.py:288-313).
//
// The reference tries itertools.combinations(pool, z) for z = K..1 and
// returns the first subset that passes check_direct.  Equivalently: the
// largest z with any feasible subset, and within it the smallest
// lexicographic rank; nodes_visited is then
// sum_{z'>z} C(K,z') + rank + 1.  On the device threads take chunks of
// consecutive ranks of one level from a work counter (shared memory in the
// batch kernel, global in the range kernel), unrank a chunk's first
// combination once, then walk lexicographic successors with branch and bound
// over prefixes; the folds of the first z-1 members stay in registers across
// the common last-position step, so a subset costs O(1) there while every
// sum is still the left-to-right fold check_direct computes.  A block-level
// (batch kernel) or grid-level (range kernel) atomicMin keeps the first
// feasible rank.  Threads count checked combinations and pruned prefixes into
// the handle's counters (eb_exhaustive_counters).
#include <climits>
#include <cstdlib>

#include "eb_internal.cuh"

namespace eb {

__device__ uint64_t g_binom[EB_MAX_K + 1][EB_MAX_K + 1];

namespace {

__global__ void binom_init_kernel() {
  int n = threadIdx.x;
  if (n > EB_MAX_K) return;
  // row n: C(n, k) -- computed sequentially by one thread per row (exact).
  uint64_t c = 1;
  for (int k = 0; k <= EB_MAX_K; ++k) {
    if (k > n) { g_binom[n][k] = 0; continue; }
    g_binom[n][k] = c;
    // C(n, k+1) = C(n, k) * (n - k) / (k + 1), exact in 128-bit
    unsigned __int128 t = (unsigned __int128)c * (unsigned)(n - k);
    c = (uint64_t)(t / (unsigned)(k + 1));
  }
}

__device__ __forceinline__ uint64_t binom(int n, int k) {
  if (k < 0 || n < 0 || k > n) return 0;
  return g_binom[n][k];
}

// Binomials C(m, k) for m, k <= nmax, copied into shared memory per block
// (the scan reads one per step and nmax + z per unranking; global g_binom
// reads were ~12% of the range kernel's stall samples, r02 ncu capture).
struct Binom {
  const uint64_t* t;
  int s;               // row stride (nmax + 1)
  __device__ __forceinline__ uint64_t operator()(int n, int k) const {
    if (k < 0 || n < 0 || k > n) return 0;
    return t[n * s + k];
  }
};
__device__ Binom binom_smem(uint64_t* dst, int nmax) {
  const int s = nmax + 1;
  for (int e = threadIdx.x; e < s * s; e += blockDim.x) dst[e] = g_binom[e / s][e % s];
  return Binom{dst, s};
}
// Per-thread combination idx[0..z) in shared memory, one byte per position,
// positions strided by the block width (no local-memory stack).
struct Idx {
  uint8_t* p;
  int s;
  __device__ __forceinline__ uint8_t& operator[](int j) const { return p[j * s]; }
};
// dynamic shared memory of the scanning kernels: binomial table, then idx
__host__ __device__ inline size_t scan_smem_bytes(int nmax, int threads) {
  return (size_t)(nmax + 1) * (nmax + 1) * 8 + (size_t)nmax * threads;
}

// Per-instance member terms, in pool order (check_direct's summation order).
struct Members {
  double a[EB_MAX_K];      // float(s) * k_up       feasibility.py:204
  double b[EB_MAX_K];      // float(n) * k_down     feasibility.py:205
  double ws[EB_MAX_K];     // waiting + slots       feasibility.py:222
  double dl[EB_MAX_K];     // deadline
  double sl[EB_MAX_K];     // slack dl - ws (the scan's least-slack member)
  int64_t far[EB_MAX_K];   // flops_autoregressive(padded, n)
  int32_t nout[EB_MAX_K];
  int n;
  int status;              // link-math error (raised inside check_direct)
  int64_t m1, kvp, kv, fi; // weight bytes, kv*padded, kv, flops_initial(padded)
  double alpha, M, beta, C, cap_s;
  double invC;             // 1/C: the scan's division-free compute-time estimate (cs_est)
  int has_cap;
  // level bounds: sums of the z smallest per-member terms (index z)
  int64_t lo_far[EB_MAX_K + 1];
  int64_t lo_n[EB_MAX_K + 1];
  double lo_a[EB_MAX_K + 1], lo_b[EB_MAX_K + 1];
  // deadline bound: bit z-1 set when some size-z subset may meet every
  // member's deadline under its least compute time (build_level_bounds)
  unsigned long long lat_ok;
  // scratch of the bound build: far-ascending order, slack-descending rank
  uint8_t far_order[EB_MAX_K], slack_rank[EB_MAX_K];
  int64_t srt_far[EB_MAX_K];
  int32_t srt_n[EB_MAX_K];
  double srt_a[EB_MAX_K], srt_b[EB_MAX_K];
};

// true only if leq(a, b) is false for every a >= a_lo (leq is monotone in a);
// the margin (1e-5 of the 1e-9 slack) dwarfs any rounding of the bounds.
__device__ __forceinline__ bool fails_margin(double a_lo, double b) {
  const double m = leq_scale(a_lo, b);
  return sub(a_lo, b) > mul(1.00001e-9, m);
}

// Sound level skip: no size-z subset can pass check_direct when the minimum
// over subsets of memory, compute time, uplink or downlink sum fails by a
// margin (every sum is minimised by the z smallest terms; memory and FLOPs
// are exact integers, the float sums lose < 64 ulp, covered by 1e-12).
__device__ __forceinline__ bool level_infeasible(const Members& S, int z) {
  int64_t mem = S.m1 + S.kvp * z + S.kv * S.lo_n[z];
  if (fails_margin(mul(S.alpha, i2d(mem)), S.M)) return true;
  double cs = div(mul(S.beta, i2d((int64_t)z * S.fi + S.lo_far[z])), S.C);
  if (S.has_cap && fails_margin(cs, S.cap_s)) return true;
  if (fails_margin(mul(S.lo_a[z], 0.999999999999), 1.0)) return true;
  if (fails_margin(mul(S.lo_b[z], 0.999999999999), 1.0)) return true;
  return !((S.lat_ok >> (z - 1)) & 1ULL);
}

// Level bounds, block-cooperative (every thread calls it; n <= 64).
//  * Sorted prefixes: the z smallest far / n / uplink / downlink terms
//    (rank sort, one thread per member, then one thread folds the prefixes).
//  * Deadline bound: a feasible subset S has a member j with the least slack
//    (dl - ws; the largest slack rank in S), and every other member ranks
//    above it.  Its compute time is at least that of z * fi + far_j + the
//    z - 1 smallest far terms among the members ranked above j, and j must
//    meet its deadline (and the slot cap) under it.  Thread j walks the
//    far-ascending order once, adding the members ranked above it, and marks
//    every z whose bound passes; a level no member marks is infeasible.  The
//    FLOP sums are exact integers and the checks are the monotone leq of
//    check_direct with the fails_margin slack, so the bound is sound.
// Bound keys of a member.  A NaN term or slack (NaN deadline, waiting time
// or gain, or an infinite deadline minus an infinite wait) makes every
// check_direct containing the member fail (each leq on NaN is false), so the
// bounds may treat it as +inf (uplink/downlink term) or -inf (slack): the
// keys stay totally ordered and the ranks a permutation, and no feasible
// subset is refuted.  The checks themselves read the raw values.
__device__ __forceinline__ double bound_term(double x) { return isnan(x) ? __longlong_as_double(0x7ff0000000000000LL) : x; }
__device__ __forceinline__ double bound_slack(const Members& S, int i) {
  const double s = sub(S.dl[i], S.ws[i]);
  return isnan(s) ? __longlong_as_double((long long)0xfff0000000000000ULL) : s;
}

__device__ void build_level_bounds(Members& S) {
  const int n = S.n;
  if (threadIdx.x == 0) S.lat_ok = 0ULL;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    int rf = 0, rn = 0, ra = 0, rb = 0, rs = 0;
    const double si = bound_slack(S, i), ai = bound_term(S.a[i]), bi = bound_term(S.b[i]);
    for (int j = 0; j < n; ++j) {
      const int jl = j < i;
      const double aj = bound_term(S.a[j]), bj = bound_term(S.b[j]);
      rf += (S.far[j] < S.far[i]) | ((S.far[j] == S.far[i]) & jl);
      rn += (S.nout[j] < S.nout[i]) | ((S.nout[j] == S.nout[i]) & jl);
      ra += (aj < ai) | ((aj == ai) & jl);
      rb += (bj < bi) | ((bj == bi) & jl);
      const double sj = bound_slack(S, j);
      rs += (sj > si) | ((sj == si) & jl);
    }
    S.srt_far[rf] = S.far[i];
    S.far_order[rf] = (uint8_t)i;
    S.srt_n[rn] = S.nout[i];
    S.srt_a[ra] = ai;
    S.srt_b[rb] = bi;
    S.slack_rank[i] = (uint8_t)rs;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    S.lo_far[0] = 0; S.lo_n[0] = 0; S.lo_a[0] = 0.0; S.lo_b[0] = 0.0;
    for (int z = 1; z <= n; ++z) {
      S.lo_far[z] = S.lo_far[z - 1] + S.srt_far[z - 1];
      S.lo_n[z] = S.lo_n[z - 1] + S.srt_n[z - 1];
      S.lo_a[z] = add(S.lo_a[z - 1], S.srt_a[z - 1]);
      S.lo_b[z] = add(S.lo_b[z - 1], S.srt_b[z - 1]);
    }
  }
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    const int p = S.slack_rank[j];
    unsigned long long ok = 0ULL;
    int64_t acc = 0;
    int c = 0;
    for (int q = 0;; ++q) {
      const int z = c + 1;
      const double cs = div(mul(S.beta, i2d((int64_t)z * S.fi + S.far[j] + acc)), S.C);
      const bool pass = !fails_margin(add(S.ws[j], cs), S.dl[j]) && !(S.has_cap && fails_margin(cs, S.cap_s));
      if (pass) ok |= 1ULL << (z - 1);
      else break;                        // the bound only grows with z
      for (; q < n; ++q) {
        const int i = S.far_order[q];
        if (S.slack_rank[i] < p) break;
      }
      if (q >= n) break;
      acc += S.far[S.far_order[q]];
      ++c;
    }
    if (ok) atomicOr(&S.lat_ok, ok);
  }
  __syncthreads();
}

// Cooperative (block) load of one instance's members; returns after sync.
__device__ void load_members(Members& S, const Ctx& c, const eb_requests& req, int64_t r0, int n) {
  __shared__ int s_pad;
  __shared__ int s_err;
  if (threadIdx.x == 0) { s_pad = 0; s_err = INT_MAX; }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) atomicMax(&s_pad, req.prompt_tokens[r0 + i]);
  __syncthreads();
  const int padded = s_pad;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    int64_t r = r0 + i;
    double ku = 0.0, kd = 0.0;
    int st = k_up_of(c, req.channel_gain[r], req.uplink_power_w[r], &ku);
    if (!st) st = k_dn_of(c, req.channel_gain[r], &kd);
    if (st) atomicMin(&s_err, i * 64 + st);
    int s = req.prompt_tokens[r], no = req.output_tokens[r];
    S.a[i] = mul(i2d(s), ku);
    S.b[i] = mul(i2d(no), kd);
    S.ws[i] = add(req.waiting_s[r], c.slots);
    S.dl[i] = req.deadline_s[r];
    S.sl[i] = sub(S.dl[i], S.ws[i]);
    S.far[i] = flops_autoregressive(c.m, padded, no);
    S.nout[i] = no;
  }
  if (threadIdx.x == 0) {
    S.n = n;
    S.m1 = weight_bytes(c.m);
    S.kv = kv_per_token(c.m);
    S.kvp = S.kv * (int64_t)padded;
    S.fi = flops_initial(c.m, padded);
    S.alpha = c.alpha; S.M = c.M; S.beta = c.beta; S.C = c.C; S.cap_s = c.cap_s;
    S.invC = div(1.0, c.C);
    S.has_cap = c.has_cap;
  }
  __syncthreads();
  if (threadIdx.x == 0) S.status = (s_err == INT_MAX) ? 0 : (s_err & 63);
  build_level_bounds(S);
}

// compute_s = (beta * float(flops)) / C without the division: within ~4 ulp
// of the exact quotient, so only fails_margin tests (1e-14 relative slack)
// may read it, and only where the tested value is at least the estimate (the
// slot cap; a deadline with a non-negative ws) so the error stays below the
// slack -- a refutation by it is then a refutation of the exact value.
__device__ __forceinline__ double cs_est(const Members& S, int64_t flops) {
  return mul(mul(S.beta, i2d(flops)), S.invC);
}
__device__ __forceinline__ bool late_est(const Members& S, int t, double ce) {
  return S.ws[t] >= 0.0 && fails_margin(add(S.ws[t], ce), S.dl[t]);
}

// check_direct on the current combination given its prefix folds.
__device__ __forceinline__ bool feasible(const Members& S, int z, const Idx& idx, int tight, int last,
                                         double up, double dn, int64_t sn, int64_t sf) {
  if (!(leq(up, 1.0) && leq(dn, 1.0))) return false;
  int64_t mem = S.m1 + S.kvp * z;
  mem += S.kv * sn;
  if (!leq(mul(S.alpha, i2d(mem)), S.M)) return false;
  int64_t flops = (int64_t)z * S.fi + sf;
  {
    // division-free refutation first (most leaves that reach here fail a
    // deadline or the slot cap by far more than the estimate's error)
    const double ce = cs_est(S, flops);
    if (S.has_cap && fails_margin(ce, S.cap_s)) return false;
    if (late_est(S, tight, ce) || late_est(S, last, ce)) return false;
  }
  double cs = div(mul(S.beta, i2d(flops)), S.C);
  if (S.has_cap && !leq(cs, S.cap_s)) return false;
  // every member must meet its deadline (an AND, so the order is free): the
  // prefix member with the least slack and the last member first, then all
  if (!leq(add(S.ws[tight], cs), S.dl[tight]) || !leq(add(S.ws[last], cs), S.dl[last])) return false;
  for (int j = 0; j < z; ++j)
    if (!leq(add(S.ws[idx[j]], cs), S.dl[idx[j]])) return false;
  return true;
}

// A prefix idx[0..p) of a size-z combination cannot be completed into a
// subset that passes check_direct.  Every check_direct quantity is monotone
// in the member set: the uplink/downlink folds only grow when terms are
// appended (IEEE addition of a non-negative term is monotone and never
// decreases the sum), memory and FLOPs are exact integer sums, and the
// compute time only grows with FLOPs.  So the completion's sums are at least
// the prefix sums plus the c = z - p smallest terms of the pool (lo_*[c]).
// The integer bounds are exact; the float bounds on lookahead terms carry the
// fails_margin slack.  `tight` is the prefix member with the least
// deadline slack seen so far: it must meet its deadline under the lower
// bound of the compute time.
__device__ __forceinline__ bool prefix_infeasible(const Members& S, int z, int p, double pu, double pd,
                                                  int64_t ps, int64_t pf, int tight) {
  const int c = z - p;
  // uplink / downlink: the prefix sum plus the c smallest remaining terms
  // (lo_*[0] = 0), refuted with the fails_margin slack (a separate exact
  // leq of the bare prefix sum only adds refutations inside that slack)
  if (fails_margin(mul(add(pu, S.lo_a[c]), 0.999999999999), 1.0) ||
      fails_margin(mul(add(pd, S.lo_b[c]), 0.999999999999), 1.0))
    return true;
  const int64_t mem = S.m1 + S.kvp * z + S.kv * (ps + S.lo_n[c]);
  if (!leq(mul(S.alpha, i2d(mem)), S.M)) return true;
  const double cs = cs_est(S, (int64_t)z * S.fi + pf + S.lo_far[c]);
  if (S.has_cap && fails_margin(cs, S.cap_s)) return true;
  return late_est(S, tight, cs);
}

// Scan ranks [r_lo, r_hi) of level z (lex order) and return the first
// feasible rank, or -1.  `stop` is polled so a thread quits once an earlier
// rank is known feasible.  Branch and bound over the lexicographic order:
// when a prefix idx[0..q] cannot be completed (prefix_infeasible), the whole
// rank range of its completions -- C(n - idx[q] - 1, z - q - 1) ranks, all
// infeasible -- is skipped, so the first feasible rank is unchanged.
//
// Per-thread state is the combination idx[] (one byte per position, L1
// resident) plus the folds of its first z-1 members in registers.  A
// successor that changes only the last position (the common step) reuses
// them; one that changes position j < z-1 refolds positions 0..z-2 from
// scratch -- the same left-to-right sums check_direct computes, so every
// value is bit-identical to a fold kept per position, without per-position
// stacks (which spilled 2.2 KB per thread to DRAM).
struct ScanCounters {
  unsigned long long leaves;    // combinations checked with the full check_direct
  unsigned long long pruned;    // prefixes cut by prefix_infeasible (whole subtrees skipped)
};

__device__ int64_t scan_chunk(const Members& S, const Binom& binom, const Idx& idx, int z, int64_t r_lo,
                              int64_t r_hi, const unsigned long long* stop, ScanCounters& cnt) {
  const int n = S.n;
  {
    // unrank r_lo: position j takes the first v whose block of C(n-v-1,
    // z-j-1) completions contains r.  r_lo < C(n, z), so every probed row
    // n-v-1 stays >= z-j-1 >= 0 and the table is read without bounds checks,
    // walking up one row per step.
    uint64_t r = (uint64_t)r_lo;
    int v = 0;
    for (int j = 0; j < z; ++j) {
      const uint64_t* p = binom.t + (n - v - 1) * binom.s + (z - j - 1);
      for (;;) {
        const uint64_t c = *p;
        if (r < c) break;
        r -= c; ++v; p -= binom.s;
      }
      idx[j] = (uint8_t)v;
      ++v;
    }
  }
  double cu = 0.0, cd = 0.0;      // folds of positions 0..z-2 (valid when `cached`)
  int64_t cs = 0, cf = 0;
  int ct = 0;
  bool cached = false;
  int from = 0;
  bool first = true;     // r_lo may sit inside a subtree: no skipping on it
  int64_t rank = r_lo;
  int steps = 0;
  while (rank < r_hi) {
    int q = z - 1;       // subtree to leave: the full combination (1 rank)
    bool dead = false;
    if (!cached || from < z - 1) {
      double pu = 0.0, pd = 0.0;
      int64_t ps = 0, pf = 0;
      int t = idx[0];
      double tsl = S.sl[t];
      for (int j = 0; j < z - 1; ++j) {
        const int i = idx[j];
        pu = add(pu, S.a[i]);
        pd = add(pd, S.b[i]);
        ps += S.nout[i];
        pf += S.far[i];
        const double sli = S.sl[i];
        if (j > 0 && !(tsl <= sli)) { t = i; tsl = sli; }
        if (j >= from && !first && prefix_infeasible(S, z, j + 1, pu, pd, ps, pf, t)) {
          q = j;
          dead = true;
          break;
        }
      }
      cached = !dead;
      cu = pu; cd = pd; cs = ps; cf = pf; ct = t;
    }
    if (dead) {
      ++cnt.pruned;
    } else {
      const int i = idx[z - 1];
      ++cnt.leaves;
      // ct is a prefix member (positions 0..z-2); at z = 1 there is no prefix
      if (feasible(S, z, idx, z > 1 ? ct : i, i, add(cu, S.a[i]), add(cd, S.b[i]), cs + S.nout[i], cf + S.far[i])) return rank;
    }
    first = false;
    rank += (int64_t)binom(n - idx[q] - 1, z - q - 1);
    if ((++steps & 127) == 0 && *(volatile const unsigned long long*)stop < (unsigned long long)rank) return -1;
    // successor of the last combination of subtree(idx[0..q])
    int j = q;
    while (j >= 0 && idx[j] == n - z + j) --j;
    if (j < 0) break;
    // positions j.. become consecutive from the incremented value: computed
    // stores, no load-after-store chain through shared memory
    const int nb = idx[j] + 1 - j;
    for (int q2 = j; q2 < z; ++q2) idx[q2] = (uint8_t)(nb + q2);
    from = j;
  }
  return -1;
}

__device__ __forceinline__ void flush_counters(const ScanCounters& c, unsigned long long* stats) {
  if (!stats) return;
  if (c.leaves) atomicAdd(&stats[0], c.leaves);
  if (c.pruned) atomicAdd(&stats[1], c.pruned);
}

struct BatchArgs {
  const eb_context* ctxs;
  int n_ctx;
  int64_t n_inst;
  const int64_t* offsets;
  const int32_t* ctx_index;
  int64_t req_base;
  eb_requests req;
  int cap;
  int32_t* status;
  int32_t* z_found;
  int64_t* lexrank;
  int64_t* nodes;
  uint64_t* mask;
  unsigned long long* stats;   // [leaves checked, prefixes pruned] (handle counters)
};

__device__ uint64_t unrank_mask(int n, int z, uint64_t r) {
  uint64_t m = 0;
  int v = 0;
  for (int j = 0; j < z; ++j)
    for (;;) {
      uint64_t cnt = binom(n - v - 1, z - j - 1);
      if (r < cnt) { m |= 1ULL << v; ++v; break; }
      r -= cnt; ++v;
    }
  return m;
}

// One block per instance (many small instances).  Each live level's rank
// range is cut into chunks that the threads take in rank order from a shared
// counter (no static split: a thread that finishes early takes the next
// chunk), and every thread stops once a rank below its chunk is known
// feasible; one barrier per level decides it.
__global__ void __launch_bounds__(256) exh_batch_kernel(const __grid_constant__ BatchArgs A) {
  __shared__ Members S;
  __shared__ unsigned long long best;
  __shared__ unsigned long long next;
  extern __shared__ __align__(8) unsigned char dyn[];
  const int nmax = A.cap < 1 ? 1 : A.cap < EB_MAX_K ? A.cap : EB_MAX_K;
  const Binom bt = binom_smem((uint64_t*)dyn, nmax);
  const Idx idx{dyn + (size_t)(nmax + 1) * (nmax + 1) * 8 + threadIdx.x, (int)blockDim.x};
  ScanCounters cnt{0ULL, 0ULL};
  for (int64_t inst = blockIdx.x; inst < A.n_inst; inst += gridDim.x) {
    int64_t row0 = A.offsets[inst];
    int n = (int)(A.offsets[inst + 1] - row0);
    int ci = A.ctx_index ? A.ctx_index[inst] : 0;
    bool tid0 = threadIdx.x == 0;
    if (n == 0 || n > A.cap || n > EB_MAX_K || ci < 0 || ci >= A.n_ctx) {
      if (tid0) {
        A.status[inst] = (ci < 0 || ci >= A.n_ctx) ? EB_ERR_INVALID_ARG
                         : (n == 0) ? EB_OK
                         : (n > A.cap) ? EB_ERR_CAP_EXCEEDED : EB_ERR_K_TOO_LARGE;
        A.z_found[inst] = 0; A.lexrank[inst] = -1; A.nodes[inst] = 0;
        if (A.mask) A.mask[inst] = 0;
      }
      __syncthreads();
      continue;
    }
    const Ctx c = load_ctx(&A.ctxs[ci]);
    load_members(S, c, A.req, row0 - A.req_base, n);
    if (S.status) {
      if (tid0) {
        A.status[inst] = S.status; A.z_found[inst] = 0; A.lexrank[inst] = -1; A.nodes[inst] = 0;
        if (A.mask) A.mask[inst] = 0;
      }
      __syncthreads();
      continue;
    }
    int zf = 0;
    int64_t rk = -1, skipped = 0;
    for (int z = n; z >= 1; --z) {
      uint64_t total = binom(n, z);
      if (level_infeasible(S, z)) { skipped += (int64_t)total; continue; }   // block-uniform
      if (tid0) { best = ULLONG_MAX; next = 0ULL; }
      __syncthreads();
      // ~8 chunks per thread, at least 32 ranks each
      uint64_t per = total / (8ULL * blockDim.x) + 1;
      if (per < 32) per = 32;
      for (;;) {
        const uint64_t lo = atomicAdd(&next, per);
        if (lo >= total || lo > *(volatile unsigned long long*)&best) break;
        const uint64_t hi = lo + per < total ? lo + per : total;
        int64_t r = scan_chunk(S, bt, idx, z, (int64_t)lo, (int64_t)hi, &best, cnt);
        if (r >= 0) { atomicMin(&best, (unsigned long long)r); break; }
      }
      __syncthreads();
      unsigned long long b = best;
      __syncthreads();
      if (b != ULLONG_MAX) { zf = z; rk = (int64_t)b; break; }
      skipped += (int64_t)total;
    }
    if (tid0) {
      A.status[inst] = EB_OK;
      A.z_found[inst] = zf;
      A.lexrank[inst] = rk;
      A.nodes[inst] = zf ? skipped + rk + 1 : skipped;   // 2^n - 1 when none
      if (A.mask) A.mask[inst] = zf ? unrank_mask(n, zf, (uint64_t)rk) : 0ULL;
    }
    __syncthreads();
  }
  flush_counters(cnt, A.stats);
}

struct RangeArgs {
  Ctx c;
  eb_requests req;
  int n, z;
  int64_t lo, hi, per;
  unsigned long long* best;    // [0] first feasible rank, [1] next chunk (grid work counter)
  int* status;
  unsigned long long* stats;
};

// Grid-wide: one level, rank range [lo, hi) in chunks of `per` that the
// threads take in rank order from a global counter.
// blocks per SM the range kernel's register budget targets (64 registers and
// 4 blocks by default; EB_BRUTE_MINB: tuning)
#ifndef EB_BRUTE_MINB
#define EB_BRUTE_MINB 1
#endif
__global__ void __launch_bounds__(256, EB_BRUTE_MINB) exh_range_kernel(const __grid_constant__ RangeArgs A) {
  __shared__ Members S;
  extern __shared__ __align__(8) unsigned char dyn[];
  const Binom bt = binom_smem((uint64_t*)dyn, A.n);     // visible after load_members' barriers
  const Idx idx{dyn + (size_t)(A.n + 1) * (A.n + 1) * 8 + threadIdx.x, (int)blockDim.x};
  load_members(S, A.c, A.req, 0, A.n);
  if (S.status) {
    if (blockIdx.x == 0 && threadIdx.x == 0) *A.status = S.status;
    return;
  }
  if (level_infeasible(S, A.z)) return;     // no size-z subset can be feasible
  const unsigned long long span = (unsigned long long)(A.hi - A.lo);
  ScanCounters cnt{0ULL, 0ULL};
  for (;;) {
    const unsigned long long off = atomicAdd(&A.best[1], (unsigned long long)A.per);
    if (off >= span) break;
    const int64_t lo = A.lo + (int64_t)off;
    if ((unsigned long long)lo > *(volatile unsigned long long*)A.best) break;
    const int64_t hi = lo + A.per < A.hi ? lo + A.per : A.hi;
    int64_t r = scan_chunk(S, bt, idx, A.z, lo, hi, A.best, cnt);
    if (r >= 0) { atomicMin(A.best, (unsigned long long)r); break; }
  }
  flush_counters(cnt, A.stats);
}

// One block: the level bounds of one instance as a bit mask (bit z-1 = level
// z not refuted).
__global__ void __launch_bounds__(256) exh_levels_kernel(const __grid_constant__ RangeArgs A,
                                                         unsigned long long* out) {
  __shared__ Members S;
  load_members(S, A.c, A.req, 0, A.n);
  if (threadIdx.x != 0) return;
  if (S.status) { *A.status = S.status; *out = 0ULL; return; }
  unsigned long long m = 0ULL;
  for (int z = 1; z <= A.n; ++z)
    if (!level_infeasible(S, z)) m |= 1ULL << (z - 1);
  *out = m;
}

}  // namespace

int binom_init(cudaStream_t st) {
  binom_init_kernel<<<1, EB_MAX_K + 1, 0, st>>>();
  EB_CUDA(cudaGetLastError());
  return EB_OK;
}

int launch_exh_batch(eb_handle* h, cudaStream_t st, const eb_context* d_ctxs, int n_ctx,
                     int64_t n_inst, const int64_t* d_off, const int32_t* d_ci, int64_t req_base,
                     const eb_requests& d_req, int cap, int32_t* d_status, int32_t* d_z,
                     int64_t* d_rank, int64_t* d_nodes, uint64_t* d_mask) {
  if (n_inst <= 0) return EB_OK;
  BatchArgs A{d_ctxs, n_ctx, n_inst, d_off, d_ci, req_base, d_req, cap, d_status, d_z, d_rank, d_nodes, d_mask,
              exh_stats(h)};
  int64_t grid = n_inst < (int64_t)h->num_sms * 8 ? n_inst : (int64_t)h->num_sms * 8;
  const int nmax = cap < 1 ? 1 : cap < EB_MAX_K ? cap : EB_MAX_K;
  const size_t dsm = scan_smem_bytes(nmax, 256);
  if (dsm > 48 * 1024) EB_CUDA(cudaFuncSetAttribute(exh_batch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm));
  exh_batch_kernel<<<(unsigned)grid, 256, dsm, st>>>(A);
  EB_CUDA(cudaGetLastError());
  h->launches += 1;
  return EB_OK;
}

// One level of one instance over a rank range; synchronous; device pointers.
static void fill_ctx(Ctx& c, const eb_context& ctx_host);

// Live levels of one instance (synchronous; device pointers).
int exh_levels(eb_handle* h, cudaStream_t st, const eb_context& ctx_host, const eb_requests& d_req, int n,
               unsigned long long* d_mask, int* d_status, uint64_t* mask, int* status) {
  RangeArgs A;
  fill_ctx(A.c, ctx_host);
  A.req = d_req; A.n = n; A.z = 0; A.lo = A.hi = 0; A.per = 1; A.best = d_mask; A.status = d_status;
  A.stats = nullptr;
  int zero = 0;
  EB_CUDA(cudaMemcpyAsync(d_status, &zero, sizeof(zero), cudaMemcpyHostToDevice, st));
  exh_levels_kernel<<<1, 256, 0, st>>>(A, d_mask);
  EB_CUDA(cudaGetLastError());
  h->launches += 1;
  unsigned long long m = 0;
  EB_CUDA(cudaMemcpyAsync(&m, d_mask, sizeof(m), cudaMemcpyDeviceToHost, st));
  EB_CUDA(cudaMemcpyAsync(status, d_status, sizeof(int), cudaMemcpyDeviceToHost, st));
  EB_CUDA(cudaStreamSynchronize(st));
  *mask = m;
  return EB_OK;
}

int exh_range(eb_handle* h, cudaStream_t st, const eb_context& ctx_host, const eb_requests& d_req,
              int n, int z, int64_t lo, int64_t hi, unsigned long long* d_best, int* d_status,
              int64_t* first_rank, int* status) {
  RangeArgs A;
  fill_ctx(A.c, ctx_host);
  A.req = d_req; A.n = n; A.z = z; A.lo = lo; A.hi = hi;
  const int64_t span = hi - lo;
  const int threads = 256;
  const int64_t max_threads = (int64_t)h->num_sms * 8 * threads;
  // ~2 chunks per resident thread (dynamic: early finishers take more), >= 64
  // ranks each.  Measured on the K=32 adversarial family (bench.py --config
  // 4): 8 chunks per thread 86 inst/s, 4: 121, 2: 149, 1: 140 -- smaller
  // chunks pay an unranking and a global atomic each and scan further past
  // the answer before the stop flag is seen.  (EB_BRUTE_CHUNKS /
  // EB_BRUTE_MINCHUNK: tuning)
  int64_t cpt = 2, minc = 64;
  if (const char* e = getenv("EB_BRUTE_CHUNKS")) { const long v = atol(e); if (v >= 1 && v <= 1024) cpt = v; }
  if (const char* e = getenv("EB_BRUTE_MINCHUNK")) { const long v = atol(e); if (v >= 1) minc = v; }
  int64_t per = span / (max_threads * cpt) + 1;
  if (per < minc) per = minc;
  A.per = per;
  A.best = d_best; A.status = d_status; A.stats = exh_stats(h);
  const int64_t nchunks = (span + per - 1) / per;
  int64_t grid = (nchunks + threads - 1) / threads;
  if (grid > (int64_t)h->num_sms * 8) grid = (int64_t)h->num_sms * 8;
  if (grid < 1) grid = 1;
  const unsigned long long init[2] = {ULLONG_MAX, 0ULL};
  int zero = 0;
  EB_CUDA(cudaMemcpyAsync(d_best, init, sizeof(init), cudaMemcpyHostToDevice, st));
  EB_CUDA(cudaMemcpyAsync(d_status, &zero, sizeof(zero), cudaMemcpyHostToDevice, st));
  const size_t dsm = scan_smem_bytes(n, threads);
  if (dsm > 48 * 1024) EB_CUDA(cudaFuncSetAttribute(exh_range_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm));
  exh_range_kernel<<<(unsigned)grid, threads, dsm, st>>>(A);
  EB_CUDA(cudaGetLastError());
  h->launches += 1;
  unsigned long long b;
  EB_CUDA(cudaMemcpyAsync(&b, d_best, sizeof(b), cudaMemcpyDeviceToHost, st));
  EB_CUDA(cudaMemcpyAsync(status, d_status, sizeof(int), cudaMemcpyDeviceToHost, st));
  EB_CUDA(cudaStreamSynchronize(st));
  *first_rank = (b == ULLONG_MAX) ? -1 : (int64_t)b;
  return EB_OK;
}

// Ctx is built host-side with the same arithmetic (only products/sums of
// config scalars, no libm), mirroring load_ctx.
static void fill_ctx(Ctx& c, const eb_context& ctx_host) {
  RangeArgs A;
  A.c.m.L = ctx_host.layers; A.c.m.d = ctx_host.hidden_dim; A.c.m.heads = ctx_host.head_count;
  A.c.m.head_dim = ctx_host.head_dim; A.c.m.ffn = ctx_host.ffn_dim; A.c.m.bpp = ctx_host.bytes_per_param;
  A.c.alpha = ctx_host.alpha; A.c.beta = ctx_host.beta; A.c.delta = ctx_host.delta_ppl;
  A.c.B_up = ctx_host.uplink_band_hz; A.c.B_dn = ctx_host.downlink_band_hz; A.c.P_dn = ctx_host.downlink_power_w;
  A.c.N0_up = ctx_host.noise_density_w_hz * ctx_host.uplink_band_hz;
  A.c.N0_dn = ctx_host.noise_density_w_hz * ctx_host.downlink_band_hz;
  A.c.T_up = ctx_host.uplink_slot_s; A.c.T_dn = ctx_host.downlink_slot_s;
  A.c.fbits = (double)ctx_host.bits_per_token;
  A.c.C = ctx_host.flops_per_s; A.c.M = ctx_host.memory_bytes; A.c.gpus = ctx_host.gpu_count;
  A.c.has_cap = ctx_host.has_slot_cap != 0; A.c.cap_s = ctx_host.slot_cap_s;
  A.c.slots = ctx_host.uplink_slot_s + ctx_host.downlink_slot_s;
  c = A.c;
}

}  // namespace eb
