// eb_dftsp.cu -- K3: instance-parallel DFTSP (reference dftsp.py:237-285).
//
// One warp per scheduling instance.  Inside the warp:
//   setup   lanes = requests: coefficients (feasibility.py:133-167, device
//           glibc-log2 port), normalized-deadline order (dftsp.py:257),
//           output-length classes and within-class uplink order
//           (dftsp.py:54-82), class sizes per pool width (ballots).
//   search  two algorithms with identical results.
//           v2 (leaf-parallel, default; search_v2): windows of 32 dfs calls
//           (lane = call) of the reference's (z, d) sequence after a
//           per-target skip; sound greedy-leaf skip per call; the surviving
//           calls' leaves unranked and checked 32 at a time (class prefixes
//           folded on the fly exactly as SearchTables.build sums them);
//           node counts from the combinatorial recurrence F(k, r) -- a
//           per-handle table for <= 64 requests and <= 3 classes, streamed
//           or row-based otherwise -- plus the winner's partial count.
//           v1 (literal; dfs_step): lanes = consecutive dfs calls, each a
//           restatement of the dfs node loop (dftsp.py:153-234); the v2
//           fallback (u32 count overflow) and the path for >= 4 classes
//           above 64 requests.
//   finish  recover_subset + check_direct re-verification (dftsp.py:276),
//           solution sorted by id (and as a selection mask), derived metrics.
// Kernels: dftsp_lock_kernel (v2, lockstep blocks: every warp of a block
// crosses the same phase barriers, so an SM runs one phase's code at a time),
// dftsp_lock_wide_kernel (v2, 65..255 requests, <= 3 classes), dftsp_kernel
// (v1 main/fallback pass), dftsp_wide_kernel (v1, 65..255 requests),
// count_table_kernel (node-count tables), dfs_single_kernel (one dfs call).
#include <climits>
#include <cstdlib>
#include <type_traits>

#include "eb_internal.cuh"

namespace eb {
namespace {

#ifdef EB_STATS
// Debug-only search statistics (a -DEB_STATS build; see tools/search_stats.py).
__device__ unsigned long long g_stats[16];
#define EB_STAT(i, v) do { if ((threadIdx.x & 31) == 0) atomicAdd(&g_stats[i], (unsigned long long)(v)); } while (0)
#else
#define EB_STAT(i, v) do { } while (0)
#endif

constexpr int RING = 64;  // in-flight window of dfs calls per warp
constexpr int EB_STATUS_FALLBACK = 99;  // internal: v2 tables overflowed, v1 pass pending

struct __align__(8) LevelInfo {
  uint16_t off;       // table offset (entries) of x = 0 for this class
  uint8_t size;       // class size
  uint8_t tail_next;  // sum of sizes of deeper classes (tail[k+1])
  uint8_t g;          // global class index (length / weight lookup)
  uint8_t pad[3];
};

__host__ __device__ constexpr inline size_t al8(size_t x) { return (x + 7) & ~size_t(7); }

// Per-warp shared memory layout (bytes).  K = max instance size, G = max
// classes.  Tables hold sum_{d=1..K} (d + G) entries per array.
struct Lay {
  size_t a_tau, a_key, a_id, a_len;                         // input order
  size_t o_tau, o_key, o_dnt, o_ws, o_dl, o_id, o_s, o_len; // tau order
  size_t o_local, o_g, o_kr;
  size_t c_len, c_w, c_start, c_cnt, c_list;                // classes
  size_t sizes, ncls, lvl;                                  // per pool width d
  size_t t_up, t_dn, t_tau;                                 // prefix tables
  size_t ring_v, ring_p, ring_done, sol;
  size_t pq, pre, pf;                                       // v2: unranking / call prefix / F tables
  size_t pm;                                                // v2, K <= 64: class-list positions per width
  size_t c_kd;                                              // v2, K <= 64: (k_up s, k_dn n) per class-list position
  size_t total;
  int T;
};

__host__ __device__ constexpr inline Lay make_lay(int K, int G, bool exact, bool v2) {
  Lay L{};
  size_t o = 0;
  auto take = [&](size_t bytes) { size_t r = o; o = al8(o + bytes); return r; };
  L.a_tau = take(8 * K); L.a_key = take(8 * K); L.a_id = take(8 * K); L.a_len = take(4 * K);
  L.o_tau = take(8 * K); L.o_key = take(8 * K); L.o_dnt = take(8 * K); L.o_ws = take(8 * K);
  L.o_dl = take(8 * K); L.o_id = take(8 * K); L.o_s = take(4 * K); L.o_len = take(4 * K);
  L.o_local = take(K); L.o_g = take(K); L.o_kr = take(K);
  L.c_len = take(4 * G); L.c_w = take(8 * G); L.c_start = take(4 * (G + 1)); L.c_cnt = take(4 * G);
  L.c_list = take(K);
  L.sizes = take((size_t)K * G); L.ncls = take(K); L.lvl = take(8 * (size_t)K * G);
  L.T = K * (K + 1) / 2 + K * G;
  if (!v2) {
    L.t_up = take(8 * (size_t)L.T); L.t_dn = take(8 * (size_t)L.T);
    L.t_tau = exact ? take(8 * (size_t)L.T) : 0;
  } else {
    // the leaf-parallel search folds each class prefix on the fly (a leaf
    // batch per instance, typically); no per-width prefix tables
    L.t_up = L.t_dn = L.t_tau = 0;
  }
  if (!v2) { L.ring_v = take(8 * RING); L.ring_p = take(8 * RING); L.ring_done = take(RING); }
  else { L.ring_v = L.ring_p = L.ring_done = 0; }
  L.sol = take(K);
  if (v2) {
    const int lvls = G > 1 ? G - 1 : 1;
    // the unranking tables (search) and the winner's count rows (counts
    // phase, after the search) share one region
    // the unranking tables (search), then the count rows of the lanes =
    // widths pass and the winner's count rows (counts phase) share a region
    // (partitions of at most three levels unrank in closed form: no tables)
    const size_t pq_bytes = G >= 4 ? 4 * (size_t)K * lvls * (K + 2) : 0, pf_bytes = 16 * (size_t)G * (K + 1);
    // (count rows only for partitions of four or more levels; three stream)
    const size_t rows_bytes = G >= 4 ? 32 * 2 * 4 * (size_t)(K + 1) : 0;
    size_t sc = pq_bytes > pf_bytes ? pq_bytes : pf_bytes;
    if (rows_bytes > sc) sc = rows_bytes;
    L.pq = take(sc);
    L.pf = L.pq;
    L.pre = take(4 * 64 + 8 * 32);
    L.pm = K <= 64 ? take(8 * (size_t)K) : 0;
    if (K <= 64) { o = (o + 15) & ~size_t(15); L.c_kd = take(16 * (size_t)K); } else { L.c_kd = 0; }
  } else {
    L.pq = L.pre = L.pf = L.pm = L.c_kd = 0;
  }
  L.total = (o + 15) & ~size_t(15);   // 16-byte warp stride: a_tau (offset 0) is read as double2
  return L;
}

struct DftspArgs {
  const eb_context* ctxs;
  int n_ctx;
  eb_search_params prm;
  int64_t n_inst;
  const int64_t* offsets;     // launch-local instance i -> absolute request rows
  const int32_t* ctx_index;
  int64_t req_base;           // absolute row of req arrays' element 0
  eb_requests req;
  int K, G;
  size_t warp_bytes;
  eb_dftsp_result out;        // per-instance arrays launch-local; solution at row - req_base
  int64_t traj_base;          // absolute row of out.traj element 0
  int* counter;               // [0] instance queue, [1] fallback count
  const uint2* ctab;          // node-count table for this flag variant (K <= 64), or null
  const int32_t* inst_list;   // wide pass: the instances to solve (indices), or null = all
  const int* list_count;      // wide pass: length of inst_list (device)
  Lay lay;                    // per-warp shared-memory layout (make_lay(K, G, exact, algorithm 2))
  int fallback_pass;
};

// sum of the 8-bit counts of levels [0, k) (every count <= 64 and their
// total <= 64, so the byte-sum multiply never carries between bytes)
__device__ __forceinline__ int sumV_below(uint64_t v0, uint64_t v1, int k) {
  const uint64_t m0 = k >= 8 ? ~0ULL : ((1ULL << (8 * k)) - 1ULL);
  int s = (int)(((v0 & m0) * 0x0101010101010101ULL) >> 56);
  if (k > 8) {
    const uint64_t m1 = k >= 16 ? ~0ULL : ((1ULL << (8 * (k - 8))) - 1ULL);
    s += (int)(((v1 & m1) * 0x0101010101010101ULL) >> 56);
  }
  return s;
}
// V8: at most 8 levels known at compile time (the compiled-in layouts), so
// every count sits in v0
template <bool V8 = false>
__device__ __forceinline__ int getV(uint64_t v0, uint64_t v1, int k) {
  if (V8) return (int)((v0 >> (8 * k)) & 0xff);
  return (int)(((k < 8) ? (v0 >> (8 * k)) : (v1 >> (8 * (k - 8)))) & 0xff);
}
template <bool V8 = false>
__device__ __forceinline__ void setV(uint64_t& v0, uint64_t& v1, int k, int x) {
  if (V8 || k < 8) v0 = (v0 & ~(0xffULL << (8 * k))) | ((uint64_t)x << (8 * k));
  else v1 = (v1 & ~(0xffULL << (8 * (k - 8)))) | ((uint64_t)x << (8 * (k - 8)));
}

// Inverse of the call numbering: calls for z = n, n-1, ..., each d = z..n.
__device__ __forceinline__ void call_zd(int n, int c, int& z, int& d) {
  int m = (int)((sqrtf(8.0f * (float)c + 1.0f) - 1.0f) * 0.5f);
  while ((m + 1) * (m + 2) / 2 <= c) ++m;
  while (m * (m + 1) / 2 > c) --m;
  z = n - m;
  d = z + (c - m * (m + 1) / 2);
}

// One dfs call's state (dftsp.py:157-182) with the per-level accumulator
// arrays collapsed to the current level; the count stack val[] is packed
// 8 bits per level into V0/V1.
struct Lane {
  int z, k, x, sel, ncl;
  uint64_t V0, V1;
  double acc_up, acc_dn, acc_lat, acc_tau;
  int64_t acc_mem;
  double k3z, slot_cap, lat_cap, mem_cap;
  uint64_t vis, prn;
};
struct Tables {
  const LevelInfo* row;   // levels of this partition
  const double* up;       // prefix tables (entries at row[k].off + x)
  const double* dn;
  const double* tau;
  const int32_t* len;     // by LevelInfo::g
  const double* w;        // latency_weight by LevelInfo::g
};

// dfs entry (dftsp.py:161-182).  Returns 1 when the call ends at the root.
template <bool PRUNE, bool INCL, bool EXACT>
__device__ __forceinline__ int dfs_begin(Lane& s, const Tables& T, int z, int tail0, int ncl, double k3,
                                         double slot_base, bool has_cap, double tau_min, double k2,
                                         int64_t padded) {
  const double INF = __longlong_as_double(0x7ff0000000000000LL);
  s.z = z;
  s.ncl = ncl;
  s.k3z = mul(k3, i2d(z));                                   // k3z = coeff.k3 * z
  s.slot_cap = has_cap ? sub(slot_base, s.k3z) : INF;        // slot_budget(z) feasibility.py:120-125
  s.lat_cap = EXACT ? s.slot_cap : pymin(tau_min, s.slot_cap);  // dftsp.py:163
  s.mem_cap = sub(k2, i2d(padded * (int64_t)z));             // mem_budget(z) feasibility.py:102-104
  s.vis = 0; s.prn = 0;
  if (PRUNE && tail0 < z) { s.prn = 1; return 1; }           // dftsp.py:166-167
  s.vis = 1;
  if (ncl == 0) return 1;                                    // dftsp.py:170-171
  s.k = 0; s.sel = 0; s.V0 = s.V1 = 0;
  s.acc_up = s.acc_dn = s.acc_lat = 0.0; s.acc_mem = 0; s.acc_tau = INF;
  s.x = min(z, (int)T.row[0].size);                          // dftsp.py:182
  return 0;
}

// One iteration of the dfs loop (dftsp.py:183-234): returns 0 (continue),
// 1 (search exhausted, no solution) or 2 (leaf passed; counts in V0/V1
// with val[k] = x).
template <bool PRUNE, bool INCL, bool EXACT>
__device__ __forceinline__ int dfs_step(Lane& s, const Tables& T) {
  const LevelInfo li = T.row[s.k];
  bool back = false;
  bool skip = false;
  if (PRUNE) {
    int cap_below = li.tail_next + (INCL ? li.size : 0);     // dftsp.py:186
    if (s.sel + s.x + cap_below < s.z) { s.prn += s.x + 1; skip = true; back = true; }
  }
  if (!skip) {
    s.vis += 1;
    int total = s.sel + s.x;
    if (total == s.z) {                                      // leaf dftsp.py:193-210
      double u = add(s.acc_up, T.up[li.off + s.x]);
      double dl = add(s.acc_dn, T.dn[li.off + s.x]);
      int64_t mem = s.acc_mem + (int64_t)s.x * T.len[li.g];
      double lat = add(s.acc_lat, mul(i2d(s.x), T.w[li.g]));
      double cap;
      if (EXACT) {
        double tau = (s.x == 0) ? s.acc_tau : pymin(s.acc_tau, T.tau[li.off + s.x]);
        cap = pymin(sub(tau, s.k3z), s.slot_cap);
      } else {
        cap = s.lat_cap;
      }
      if (leq(u, 1.0) && leq(dl, 1.0) && leq(i2d(mem), s.mem_cap) && leq(lat, cap)) {
        setV(s.V0, s.V1, s.k, s.x);
        return 2;
      }
      if (s.x > 0) { s.x -= 1; return 0; }
      back = true;
    } else if (s.k == s.ncl - 1) {                           // dead end dftsp.py:211-214
      s.vis += s.x;
      back = true;
    } else {                                                 // descend dftsp.py:215-226
      setV(s.V0, s.V1, s.k, s.x);
      s.acc_up = add(s.acc_up, T.up[li.off + s.x]);
      s.acc_dn = add(s.acc_dn, T.dn[li.off + s.x]);
      s.acc_mem += (int64_t)s.x * T.len[li.g];
      s.acc_lat = add(s.acc_lat, mul(i2d(s.x), T.w[li.g]));
      if (EXACT && s.x != 0) s.acc_tau = pymin(s.acc_tau, T.tau[li.off + s.x]);
      s.sel = total;
      s.k += 1;
      s.x = min(s.z - total, (int)T.row[s.k].size);
      return 0;
    }
  }
  (void)back;
  // backtrack dftsp.py:227-234
  for (;;) {
    if (s.k == 0) return 1;
    s.k -= 1;
    s.x = getV(s.V0, s.V1, s.k) - 1;
    if (s.x >= 0) break;
  }
  // accumulators of level k = the same left fold over levels < k
  s.sel = 0; s.acc_up = 0.0; s.acc_dn = 0.0; s.acc_lat = 0.0; s.acc_mem = 0;
  s.acc_tau = __longlong_as_double(0x7ff0000000000000LL);
  for (int j = 0; j < s.k; ++j) {
    const LevelInfo lj = T.row[j];
    int v = getV(s.V0, s.V1, j);
    s.sel += v;
    s.acc_up = add(s.acc_up, T.up[lj.off + v]);
    s.acc_dn = add(s.acc_dn, T.dn[lj.off + v]);
    s.acc_mem += (int64_t)v * T.len[lj.g];
    s.acc_lat = add(s.acc_lat, mul(i2d(v), T.w[lj.g]));
    if (EXACT && v != 0) s.acc_tau = pymin(s.acc_tau, T.tau[lj.off + v]);
  }
  return 0;
}


// ===========================================================================
// v2 search: leaf-parallel enumeration with combinatorial node counting.
//
// Facts used (all from the dfs loop, dftsp.py:183-234):
//  * the leaves of dfs(z) on a partition are exactly the count vectors c
//    (0 <= c_k <= s_k, sum c = z), met in lexicographically descending order;
//    the leaf check (dftsp.py:193-203) is a pure function of c (the
//    accumulator chain is a left fold over the classes; trailing zero counts
//    add +0.0, which is exact);
//  * every other step is data independent, so the node counts of a fully
//    searched (failed) subtree depend only on the class sizes, the remaining
//    target and the flags: F(k, r) below, a per-level recurrence over prefix
//    sums that restates the prune / visit / dead-end / descend rules;
//  * therefore the reference's first successful (z, d, leaf) in sequence
//    order can be found by evaluating leaves in parallel (32 per warp step,
//    in order, ballot + first set lane), and nodes_visited / nodes_pruned
//    are sum F over the failed calls plus the partial count of the winning
//    call up to its leaf.
//  * the first leaf of a call is the greedy low-output fill, which minimises
//    the memory sum (exact integers) and the latency sum (weights ascend with
//    the output length); a call whose greedy leaf fails memory or latency by
//    a margin far beyond floating-point error cannot contain a passing leaf
//    and is skipped without enumeration (its node counts are still added).
// ===========================================================================
// Exact warp sum of int64 values (butterfly; every lane gets the total).
__device__ __forceinline__ int64_t warp_sum_i64(int64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(EB_FULL, v, o);
  return v;
}

__device__ __forceinline__ bool fails_with_margin(double a_lo, double b) {
  // true only if leq(a, b) is false for every a >= a_lo (leq is monotone in a)
  const double m = leq_scale(a_lo, b);
  return sub(a_lo, b) > mul(1.00001e-9, m);
}

// Blocked warp-wide inclusive prefix over r = 0..n of two u64 sequences.
template <int QMAX, typename ValFn, typename StoreFn>
__device__ __forceinline__ void warp_prefix2(int n, ValFn val, StoreFn store) {
  const int lane = threadIdx.x & 31;
  const int q = (n + 32) >> 5;                 // ceil((n + 1) / 32) <= QMAX
  uint64_t va[QMAX], vb[QMAX], la = 0, lb = 0;
#pragma unroll
  for (int j = 0; j < QMAX; ++j) {
    int r = lane * q + j;
    va[j] = vb[j] = 0;
    if (j < q && r <= n) val(r, va[j], vb[j]);
    la += va[j];
    lb += vb[j];
  }
  uint64_t ia = la, ib = lb;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint64_t ta = __shfl_up_sync(EB_FULL, ia, o), tb = __shfl_up_sync(EB_FULL, ib, o);
    if (lane >= o) { ia += ta; ib += tb; }
  }
  uint64_t ra = ia - la, rb = ib - lb;
#pragma unroll
  for (int j = 0; j < QMAX; ++j) {
    int r = lane * q + j;
    if (j < q && r <= n) { ra += va[j]; rb += vb[j]; store(r, ra, rb); }
  }
}

// Single-sequence version of warp_prefix2.
template <int QMAX, typename ValFn, typename StoreFn>
__device__ __forceinline__ void warp_prefix1(int n, ValFn val, StoreFn store) {
  const int lane = threadIdx.x & 31;
  const int q = (n + 32) >> 5;
  uint64_t va[QMAX], la = 0;
#pragma unroll
  for (int j = 0; j < QMAX; ++j) {
    int r = lane * q + j;
    va[j] = (j < q && r <= n) ? val(r) : 0;
    la += va[j];
  }
  uint64_t ia = la;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint64_t ta = __shfl_up_sync(EB_FULL, ia, o);
    if (lane >= o) ia += ta;
  }
  uint64_t ra = ia - la;
#pragma unroll
  for (int j = 0; j < QMAX; ++j) {
    int r = lane * q + j;
    if (j < q && r <= n) { ra += va[j]; store(r, ra); }
  }
}

// Full-traversal node counts of one dfs level (dftsp.py:183-234) entered at
// level k with remaining target r >= 1: (visited, pruned).  pf(q, v, p)
// returns the prefix sums over r' = 1..q of F(k+1, r') (q >= 0, 0 at q = 0):
// a table lookup, or the closed form of the deepest level.
template <bool PRUNE, bool INCL, typename PFN>
__device__ __forceinline__ void level_counts_f(const LevelInfo& li, bool last, int r, PFN pf, uint64_t& fv,
                                               uint64_t& fp) {
  const int s = li.size, cap = li.tail_next + (INCL ? li.size : 0);
  const int x0 = min(r, s);
  const int xs = PRUNE ? max(0, r - cap) : 0;          // lowest unpruned count
  if (PRUNE && x0 < xs) { fv = 0; fp = (uint64_t)x0 + 1; return; }
  if (last) {
    if (x0 == r) {                                      // leaf, then x = r - 1
      if (PRUNE && r - 1 < xs) { fv = 1; fp = (uint64_t)r; }
      else { fv = 1 + (uint64_t)r; fp = 0; }            // dead end: 1 + bulk (r - 1)
    } else {
      fv = 1 + (uint64_t)x0; fp = 0;                    // dead end at x0
    }
    return;
  }
  fv = (uint64_t)(x0 - xs + 1);                         // nodes x = x0 .. xs visited
  fp = (PRUNE && xs > 0) ? (uint64_t)xs : 0;            // prune event at x = xs - 1
  const int xb = (x0 == r) ? x0 - 1 : x0;               // descending nodes x = xb .. xs
  if (xb >= xs) {
    uint64_t hv, hp, lv, lp;
    pf(r - xs, hv, hp);
    pf(r - xb - 1, lv, lp);
    fv += hv - lv;
    fp += hp - lp;
  }
}

template <bool PRUNE, bool INCL, typename PT>
__device__ __forceinline__ void level_counts(const LevelInfo& li, bool last, int r, const PT* PFV, const PT* PFP,
                                             uint64_t& fv, uint64_t& fp) {
  level_counts_f<PRUNE, INCL>(li, last, r, [&](int q, uint64_t& v, uint64_t& p) {
    v = (uint64_t)PFV[q];
    p = (uint64_t)PFP[q];
  }, fv, fp);
}

// Phase barrier of the lockstep (ALGO 2) kernel: every warp of the block
// passes the same three barriers per instance round, so the SM executes one
// phase's code at a time (instruction-cache locality).
#ifndef EB_LOCK_BARRIERS
#define EB_LOCK_BARRIERS 3   // which phase barriers synchronize (bit i = barrier i; measured: 3 > 5 > 7 > 1)
#endif
template <int ALGO>
__device__ __forceinline__ void phase_barrier(int& passed) {
  if constexpr (ALGO == 2) {
    if ((EB_LOCK_BARRIERS >> passed) & 1) __syncthreads();
  }
  ++passed;
}

// exhaustive_optimal(mode="counts") (dftsp.py:316-332) rides on the v2 leaf
// stream: same count vectors in the same order (_count_vectors dftsp.py:335),
// but the check is check_knapsack's per-member sequential fold over the
// recovered subset (feasibility.py:170-189) and nodes = vectors tried.
struct CountsMode {
  bool on;
  const int32_t* c_start;   // class member lists (kr order), tau-rank values
  const uint8_t* c_list;
  const double* o_key;      // k_up * s  per tau rank
  const double* o_dnt;      // k_down * n per tau rank
  const double2* c_kd;      // (k_up * s, k_down * n) per class-list position (K <= 64)
};

// SearchTables.build (dftsp.py:110-132) for class g of pool width d: the
// up / dn (/ tau-min) prefix tables over the class members among the d first
// in tau order, in within-class key order, at offset base(d) + sum over
// classes g2 < g of (size + 1).  One lane; the folds are sequential (each
// prefix is the previous one plus one term, as in the reference).
template <bool EXACT>
__device__ __forceinline__ void build_width_tables(int d, int g, int Gi, const uint8_t* sizes, const int32_t* c_start,
                                                   const uint8_t* c_list, const double* o_key, const double* o_dnt,
                                                   const double* o_tau, double* t_up, double* t_dn, double* t_tau) {
  const int base = (d - 1) * d / 2 + (d - 1) * Gi;
  int start = 0;
  for (int g2 = 0; g2 < g; ++g2) start += sizes[(d - 1) * Gi + g2] + 1;
  const int off = base + start;
  double cu = 0.0, cd = 0.0, tm = __longlong_as_double(0x7ff0000000000000LL);
  t_up[off] = cu; t_dn[off] = cd;
  if (EXACT) t_tau[off] = tm;
  int x = 0;
  const int b = c_start[g], e = c_start[g + 1];
  for (int q = b; q < e; ++q) {
    const int t = c_list[q];
    if (t < d) {
      ++x;
      cu = add(cu, o_key[t]);                    // cu[-1] + k_up*s   (dftsp.py:126)
      cd = add(cd, o_dnt[t]);                    // cd[-1] + k_down*n (dftsp.py:127)
      t_up[off + x] = cu;
      t_dn[off + x] = cd;
      if (EXACT) { tm = pymin(tm, o_tau[t]); t_tau[off + x] = tm; }  // dftsp.py:128
    }
  }
}

// Prefix sums over r of the deepest level's counts (F(m-1, r) is a leaf,
// dead end or prune; see level_counts), in closed form.
template <bool PRUNE, bool INCL>
__device__ __forceinline__ void last_level_prefix(uint32_t s, uint32_t rr, uint64_t& v, uint64_t& p) {
  // s, rr <= EB_MAX_K_DFTSP + 1, so every product below fits 32 bits
  const uint32_t t = rr < s ? rr : s;
  if (PRUNE && !INCL) {            // r <= s: (1, r); r > s: (0, s + 1)
    v = t;
    p = t * (t + 1) / 2 + (rr - t) * (s + 1);
  } else if (!PRUNE) {             // r <= s: (1 + r, 0); r > s: (1 + s, 0)
    v = t + t * (t + 1) / 2 + (rr - t) * (1 + s);
    p = 0;
  } else {                         // inclusive: r <= s: 1 + r; s < r <= 2s: 1 + s; r > 2s: prune s + 1
    const uint32_t u = rr < 2 * s ? rr : 2 * s;
    v = t + t * (t + 1) / 2 + (u - t) * (1 + s);
    p = (rr - u) * (s + 1);
  }
}

// Node-count tables for instances of at most 64 requests and at most three
// output classes.  Per partition shape (m classes of sizes s0, s1, s2 >= 1,
// in level order, s0 + s1 + s2 <= 64) a row holds PF0(q) = sum over
// r = 1..q of F(0, r) (visited, pruned), q = 0..64: the full-traversal counts
// of dfs calls with target r, computed by the same recurrence as search_v2
// (level_counts_f / last_level_prefix).  Summing F(0, z) over a z range is
// then two lookups.  Layout: a u32 header of row offsets -- O3[s0 * CT + s1]
// = row of (s0, s1, 1), O2[s0] = row of (s0, 1), R1 = row of (1) -- then the
// rows of CT uint2 entries (43,744 rows, 22.7 MB per flag variant).
constexpr int CT = 65;
constexpr int CT_HDR = CT * CT + CT + 1;                  // u32 entries
constexpr size_t CT_HDR_BYTES = ((size_t)CT_HDR * 4 + 255) & ~(size_t)255;
constexpr int CT_ROWS = 41664 + 2016 + 64;                // C(64,3) + C(64,2) + 64
// the header's spare tail holds the four/five-class table's address (or 0)
constexpr size_t CT_MPTR_OFF = ((size_t)CT_HDR * 4 + 7) & ~(size_t)7;
static_assert(CT_MPTR_OFF + 8 <= CT_HDR_BYTES, "count-table header has no room for the pointer");

__host__ __device__ __forceinline__ int ct_row(const uint32_t* hdr, int m, int s0, int s1, int s2) {
  if (m == 3) return (int)hdr[s0 * CT + s1] + s2 - 1;
  if (m == 2) return (int)hdr[CT * CT + s0] + s1 - 1;
  return (int)hdr[CT * CT + CT] + s0 - 1;
}

// The same row index in closed form (no dependent header load on the
// device): shapes are numbered s0-major with 64 - s0 - s1 rows per (s0, s1),
// so the rows before s0 are Tet(62) - Tet(63 - s0), Tet(k) = k(k+1)(k+2)/6.
__host__ __device__ __forceinline__ int ct_row_closed(int m, int s0, int s1, int s2) {
  auto tet = [](int k) { return k * (k + 1) * (k + 2) / 6; };
  if (m == 3) return tet(62) - tet(63 - s0) + (s1 - 1) * (64 - s0) - (s1 - 1) * s1 / 2 + s2 - 1;
  if (m == 2) return 41664 + (s0 - 1) * 64 - (s0 - 1) * s0 / 2 + s1 - 1;
  return 41664 + 2016 + s0 - 1;
}

// Host: the header (row offsets in shape order).
static void ct_header(uint32_t* hdr) {
  for (int i = 0; i < CT_HDR; ++i) hdr[i] = 0;
  uint32_t row = 0;
  for (int s0 = 1; s0 <= 62; ++s0)
    for (int s1 = 1; s0 + s1 <= 63; ++s1) { hdr[s0 * CT + s1] = row; row += 64 - s0 - s1; }
  for (int s0 = 1; s0 <= 63; ++s0) { hdr[CT * CT + s0] = row; row += 64 - s0; }
  hdr[CT * CT + CT] = row;
}

template <bool PRUNE, bool INCL>
__global__ void count_table_kernel(const uint32_t* __restrict__ hdr, uint2* __restrict__ rows) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int n3 = 64 * 64 * 64, n2 = 64 * 64;
  int m, sz[3] = {0, 0, 0};
  if (t < n3) { m = 3; sz[0] = 1 + t / 4096; sz[1] = 1 + (t / 64) % 64; sz[2] = 1 + t % 64; }
  else if (t < n3 + n2) { m = 2; sz[0] = 1 + (t - n3) / 64; sz[1] = 1 + (t - n3) % 64; }
  else if (t < n3 + n2 + 64) { m = 1; sz[0] = 1 + (t - n3 - n2); }
  else return;
  const int d = sz[0] + sz[1] + sz[2];
  if (d > 64) return;
  LevelInfo row[3];
  int tail = 0;
  for (int k = m - 1; k >= 0; --k) {
    row[k].off = 0; row[k].size = (uint8_t)sz[k]; row[k].tail_next = (uint8_t)tail; row[k].g = (uint8_t)k;
    row[k].pad[0] = row[k].pad[1] = row[k].pad[2] = 0;
    tail += sz[k];
  }
  const uint32_t sl = sz[m - 1];
  auto pf_last = [&](int q, uint64_t& v, uint64_t& p) { last_level_prefix<PRUNE, INCL>(sl, (uint32_t)q, v, p); };
  uint32_t RV[CT] = {}, RP[CT] = {};
  auto pf_row = [&](int q, uint64_t& v, uint64_t& p) { v = RV[q]; p = RP[q]; };
  if (m == 3) {                       // level 1 against the closed-form level 2, prefix-summed
    uint64_t av = 0, ap = 0;
    for (int r = 1; r <= d; ++r) {
      uint64_t fv, fp;
      level_counts_f<PRUNE, INCL>(row[1], false, r, pf_last, fv, fp);
      av += fv; ap += fp;
      RV[r] = (uint32_t)av; RP[r] = (uint32_t)ap;
    }
  }
  uint2* out = rows + (size_t)ct_row(hdr, m, sz[0], sz[1], sz[2]) * CT;
  uint64_t av = 0, ap = 0;
  out[0] = make_uint2(0u, 0u);
  for (int r = 1; r <= d; ++r) {      // (every value < 2^32: at most 65^3 nodes per call, 64 calls)
    uint64_t fv, fp;
    if (m == 3) level_counts_f<PRUNE, INCL>(row[0], false, r, pf_row, fv, fp);
    else level_counts_f<PRUNE, INCL>(row[0], m == 1, r, pf_last, fv, fp);
    av += fv; ap += fp;
    out[r] = make_uint2((uint32_t)av, (uint32_t)ap);
  }
}

// Node-count tables for four and five output classes at pool widths up to
// CTM_K (the config-5 shape): per partition shape s0..s_{m-1} >= 1 with
// sum d <= CTM_K, a row of PF0(q), q = 0..CTM_K, as in count_table_kernel.
// Shapes are numbered by the colex rank of their partial sums
// t_i = s_0 + .. + s_i (1 <= t_0 < .. < t_{m-1} = d <= CTM_K):
// rank = sum_i C(t_i - 1, i + 1), m = 4 rows first.  237,336 rows, 62.7 MB
// per flag variant.  Without them each width runs the level recurrence over
// a u32 row on its own lane (one lane per width, work ~ m d, lanes idle).
constexpr int CTM_K = 32;
constexpr int CTM = CTM_K + 1;
constexpr int CTM_ROWS4 = 35960;                          // C(32, 4)
constexpr int CTM_ROWS = CTM_ROWS4 + 201376;              // + C(32, 5)

// C(a, k) for 0 <= a < CTM_K, k = 1..5 (0 when a < k: the product has a zero
// factor); constant divisors
__host__ __device__ __forceinline__ int binom_small(int a, int k) {
  switch (k) {
    case 1: return a;
    case 2: return a * (a - 1) / 2;
    case 3: return a * (a - 1) * (a - 2) / 6;
    case 4: return a * (a - 1) * (a - 2) * (a - 3) / 24;
    default: return a * (a - 1) * (a - 2) * (a - 3) * (a - 4) / 120;
  }
}

__host__ __device__ __forceinline__ int ctm_row(int m, const int* sz) {
  int t = 0, rank = m == 5 ? CTM_ROWS4 : 0;
#pragma unroll
  for (int i = 0; i < 5; ++i)
    if (i < m) { t += sz[i]; rank += binom_small(t - 1, i + 1); }
  return rank;
}

template <bool PRUNE, bool INCL>
__global__ void count_table_m_kernel(uint2* __restrict__ rows) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n4 = 32LL * 32 * 32 * 32, n5 = n4 * 32;
  int m, sz[5];
  int64_t u;
  if (t < n4) { m = 4; u = t; } else if (t < n4 + n5) { m = 5; u = t - n4; } else return;
  int d = 0;
  for (int i = m - 1; i >= 0; --i) { sz[i] = 1 + (int)(u & 31); u >>= 5; d += sz[i]; }
  if (d > CTM_K) return;
  LevelInfo row[5];
  int tail = 0;
  for (int k = m - 1; k >= 0; --k) {
    row[k].off = 0; row[k].size = (uint8_t)sz[k]; row[k].tail_next = (uint8_t)tail; row[k].g = (uint8_t)k;
    row[k].pad[0] = row[k].pad[1] = row[k].pad[2] = 0;
    tail += sz[k];
  }
  const uint32_t sl = sz[m - 1];
  auto pf_last = [&](int q, uint64_t& v, uint64_t& p) { last_level_prefix<PRUNE, INCL>(sl, (uint32_t)q, v, p); };
  uint32_t RV[CTM] = {}, RP[CTM] = {};
  auto pf_row = [&](int q, uint64_t& v, uint64_t& p) { v = RV[q]; p = RP[q]; };
  {                                   // level m-2 against the closed-form last level, prefix-summed
    uint64_t av = 0, ap = 0;
    for (int r = 1; r <= d; ++r) {
      uint64_t fv, fp;
      level_counts_f<PRUNE, INCL>(row[m - 2], false, r, pf_last, fv, fp);
      av += fv; ap += fp;
      RV[r] = (uint32_t)av; RP[r] = (uint32_t)ap;
    }
  }
  for (int k = m - 3; k >= 1; --k) {  // in place: F(k, r) reads PF_{k+1} at indices <= r
    for (int r = d; r >= 1; --r) {
      uint64_t fv, fp;
      level_counts_f<PRUNE, INCL>(row[k], false, r, pf_row, fv, fp);
      RV[r] = (uint32_t)fv; RP[r] = (uint32_t)fp;
    }
    uint64_t bv = 0, bp = 0;
    for (int r = 1; r <= d; ++r) {
      bv += RV[r]; bp += RP[r];
      RV[r] = (uint32_t)bv; RP[r] = (uint32_t)bp;
    }
  }
  uint2* out = rows + (size_t)ctm_row(m, sz) * CTM;
  uint64_t av = 0, ap = 0;
  out[0] = make_uint2(0u, 0u);
  for (int r = 1; r <= d; ++r) {      // (< 2^32: at most C(37, 5) nodes per call, 32 calls)
    uint64_t fv, fp;
    level_counts_f<PRUNE, INCL>(row[0], false, r, pf_row, fv, fp);
    av += fv; ap += fp;
    out[r] = make_uint2((uint32_t)av, (uint32_t)ap);
  }
}

// Unranking prefix tables in closed form for partitions of at most three
// levels: P_{k+1}[y] = #{count vectors of levels k+1 .. m-1 within their
// class sizes, summing to at most y - 1} (P[0] = 0), the values build_pq
// stores.  The last level admits one vector per sum up to its size; the
// level above the last (m = 3) counts pairs (c1, c2) with c1 + c2 <= x:
//   F(x) = (b + 1)(s2 + 1) + (a - b)(x + 1) - (a(a + 1) - b(b + 1)) / 2,
//   a = min(s1, x), b = min(a, x - s2) (or -1 when x < s2).
__device__ __forceinline__ uint32_t pq_closed(const LevelInfo* row, int m, int k, int y) {
  if (y <= 0) return 0u;
  const int x = y - 1;
  if (k + 1 == m - 1) return (uint32_t)(min(x, (int)row[m - 1].size) + 1);
  const int s1 = row[k + 1].size, s2 = row[k + 2].size;   // k + 1 == m - 2, m == 3
  const int a = min(s1, x);
  const int b = x - s2 >= 0 ? min(a, x - s2) : -1;
  return (uint32_t)((b + 1) * (s2 + 1) + (a - b) * (x + 1) - (a * (a + 1) - b * (b + 1)) / 2);
}

template <bool PRUNE, bool INCL, bool EXACT, int NI, int FK = 0>
__device__ bool search_v2(int& passed, int n, int Gi, unsigned char* smem, const Lay& L, const LevelInfo* lvl,
                          const uint8_t* ncls_d,
                          const int32_t* c_len, const double* c_w, const double* o_tau, double k2, double k3,
                          double slot_base, bool has_cap, int padded, int64_t* traj, bool& found, int& zf,
                          int& dwin, int& kwin, uint64_t& W0, uint64_t& W1, int& best, uint64_t& tot_v,
                          uint64_t& tot_p, const CountsMode& cm, const uint2* ctab, const uint8_t* sizes) {
  const int lane = threadIdx.x & 31;
  constexpr bool V8 = FK > 0 && FK % 100 <= 8;   // count vectors fit one u64
  // per-level loops unrolled to a compiled-in bound of at most three classes
  // (config 2); five (config 5) unrolled measured 5 % slower
  constexpr int FGM = (FK > 0 && FK % 100 <= 3) ? FK % 100 : 0;
  uint64_t cm_before = 0;   // counts mode: count vectors tried in completed windows
  const double INF = __longlong_as_double(0x7ff0000000000000LL);
  uint32_t* pq = (uint32_t*)(smem + L.pq);
  uint32_t* pre = (uint32_t*)(smem + L.pre);
  uint64_t* pre64 = (uint64_t*)(smem + L.pre + 4 * 64);
  uint64_t* pfv = (uint64_t*)(smem + L.pf);
  uint64_t* pfp = pfv + (size_t)Gi * (n + 1);
  const uint64_t* pm = (const uint64_t*)(smem + L.pm);     // width masks (NI <= 2, setup)
  using WMask = typename std::conditional<NI == 1, uint32_t, uint64_t>::type;
  auto wm_ffs = [](WMask b) -> int { return NI == 1 ? __ffs((unsigned)b) - 1 : __ffsll((long long)b) - 1; };
  const int LV = Gi > 1 ? Gi - 1 : 1;
  const int W = n + 2;

  // ---- U: unranking tables, built lazily for pool widths d that have a
  //      call surviving the skip test.  For level k >= 1 of partition d,
  //      PQ_k[x + 1] = #{(c_k..c_{m-1}) : bounds, sum <= x}  (prefix of Q_k).
  uint64_t built = 0;       // bit d-1: tables of width d are ready
  auto build_pq = [&](int d) -> bool {
    const int m = ncls_d[d - 1];
    if (m < 2) return true;
    const LevelInfo* row = lvl + (size_t)(d - 1) * Gi;
    uint32_t* base = pq + (size_t)(d - 1) * LV * W;
    // levels m-1 and m-2 are closed forms (pq_closed); tables for m-3 .. 1
    bool ovf = false;
    for (int k = m - 3; k >= 1; --k) {
      const uint32_t* Pn = base + (size_t)k * W;        // level k+1
      uint32_t* Pk = base + (size_t)(k - 1) * W;        // level k
      const int sk = row[k].size;
      const bool closed = k + 1 >= m - 2;
      bool o2 = false;
      warp_prefix1<NI + 1>(n,
          [&](int r) -> uint64_t {
            int lo = r - sk - 1;
            if (closed) return (uint64_t)pq_closed(row, m, k, r + 1) - (lo >= 0 ? (uint64_t)pq_closed(row, m, k, lo + 1) : 0);
            return (uint64_t)Pn[r + 1] - (lo >= 0 ? (uint64_t)Pn[lo + 1] : 0);
          },
          [&](int r, uint64_t a) {
            if (a > 0x7fffffffULL) o2 = true;
            Pk[r + 1] = (uint32_t)a;
          });
      if (lane == 0) Pk[0] = 0;
      ovf |= __any_sync(EB_FULL, o2);
      __syncwarp();
    }
    return !ovf;
  };

  // ---- S: the call sequence (z from n down, d from z up) in windows of 32
  //      calls, lane = call: skip test, then the surviving calls' leaves in
  //      sequence order, 32 per step, first passing leaf wins.
  found = false;
  const int total_calls = n * (n + 1) / 2;
  EB_STAT(0, 1);
  // Whole targets z first: the greedy leaf of the widest pool (d = n) has the
  // least memory and latency of any width's greedy leaf (more short requests
  // to choose from), and every width d >= z has a cap no larger than width
  // z's (tau descends with d).  If it fails width z's caps by the margin, no
  // call (z, d) can contain a passing leaf, so the call sequence starts at
  // the largest z that survives (lanes = z).  Counts mode needs every call.
  // Exact per-leaf tau (dftsp.py:128): a leaf's tau is the least of its z
  // members' deadlines among the first d by tau, so it is at most the z-th
  // largest, o_tau[z - 1]; min(o_tau[z - 1] - k3 z, slot_budget(z)) thus
  // bounds every leaf cap of target z from above, for every width.  (With a
  // NaN deadline the tau ranks are not a permutation: slot budget only.)
  // A -inf normalized deadline (an infinite waiting time) makes every cap
  // that includes it -inf, and leq(lat, -inf) is TRUE (its tolerance
  // 1e-9 * max(1, |a|, |b|) is then infinite): the leaf check is not
  // monotone in the cap there, so no latency-based skip is sound -- only the
  // memory skips stay (lat_free).  tau ranks are a permutation (NaN taus are
  // refused in setup), so o_tau[n - 1] is the least.
  const bool lat_free = o_tau[n - 1] == -INF;
  bool tau_ok = !lat_free;
  if (EXACT) {
    bool nan = false;
    for (int t = lane; t < n; t += 32) nan |= !(o_tau[t] == o_tau[t]);
    tau_ok = tau_ok && !__any_sync(EB_FULL, nan);
  }
  int c_first = 0;
  if (!cm.on) {
    const LevelInfo* rown = lvl + (size_t)(n - 1) * Gi;
    const int mn = ncls_d[n - 1];
    int zhi = 0;
    for (int z = lane + 1; z <= n; z += 32) {
      const double k3z = mul(k3, i2d(z));
      const double slot_cap = has_cap ? sub(slot_base, k3z) : INF;
      const double mem_cap = sub(k2, i2d((int64_t)padded * z));
      int rem = z;
      int64_t mem = 0;
      double lat = 0.0;
#pragma unroll
      for (int k = 0; k < (FGM ? FGM : mn); ++k) {   // FGM > 0: unrolled
        if (k >= mn || rem <= 0) break;
        const LevelInfo li = rown[k];
        const int cc = min(rem, (int)li.size);
        mem += (int64_t)cc * c_len[li.g];
        lat = add(lat, mul(i2d(cc), c_w[li.g]));
        rem -= cc;
      }
      const double lat_cap = lat_free ? INF : (EXACT && !tau_ok) ? slot_cap : pymin(sub(o_tau[z - 1], k3z), slot_cap);
      if (!(fails_with_margin(i2d(mem), mem_cap) || fails_with_margin(mul(lat, 0.999999999999), lat_cap)))
        zhi = z;
    }
    zhi = __reduce_max_sync(EB_FULL, zhi);
    c_first = zhi > 0 ? (n - zhi) * (n - zhi + 1) / 2 : total_calls;
  }
  for (int c0 = c_first; c0 < total_calls && !found; c0 += 32) {
    const int c = c0 + lane;
    int z = 0, d = 0;
    bool live = false;
    EB_STAT(1, 1);
    if (c < total_calls) {
      call_zd(n, c, z, d);
      const double k3z = mul(k3, i2d(z));                            // coeff.k3 * z
      const double slot_cap = has_cap ? sub(slot_base, k3z) : INF;  // slot_budget(z)
      const double mem_cap = sub(k2, i2d((int64_t)padded * z));      // mem_budget(z)
      const int m = ncls_d[d - 1];
      const LevelInfo* row = lvl + (size_t)(d - 1) * Gi;
      // sound skip: greedy (first) leaf fails memory or latency by a margin
      int rem = z;
      int64_t mem = 0;
      double lat = 0.0;
#pragma unroll
      for (int k = 0; k < (FGM ? FGM : m); ++k) {   // FGM > 0: unrolled
        if (k >= m || rem <= 0) break;
        const LevelInfo li = row[k];
        const int cc = min(rem, (int)li.size);
        mem += (int64_t)cc * c_len[li.g];
        lat = add(lat, mul(i2d(cc), c_w[li.g]));
        rem -= cc;
      }
      // (non-exact: the call's own cap, exact for all its leaves, -inf included)
      const double lat_cap = EXACT ? (lat_free ? INF : tau_ok ? pymin(sub(o_tau[z - 1], k3z), slot_cap) : slot_cap)
                                   : pymin(sub(o_tau[d - 1], k3z), slot_cap);
      live = !(fails_with_margin(i2d(mem), mem_cap) || fails_with_margin(mul(lat, 0.999999999999), lat_cap));
      if (EXACT && tau_ok && live && !cm.on) {
        // Exact tau: a member t whose own deadline fails the greedy latency
        // (o_tau[t] - k3 z < lat by the margin) is in no passing leaf, so a
        // passing leaf takes at most lim_k of class k (its members before the
        // first such one, in key order among the first d).  The greedy fill of
        // that box bounds every in-box leaf's memory and latency from below.
        const double lat_m = mul(lat, 0.999999999999);
        int r2 = z;
        int64_t mem2 = 0;
        double lat2 = 0.0;
        for (int k = 0; k < m && r2 > 0; ++k) {
          const LevelInfo li = row[k];
          int lim = 0;
          if constexpr (NI <= 2) {
            WMask bits = (WMask)pm[d - 1] & ((WMask)~(WMask)0 << cm.c_start[li.g]);
            for (int seen = 0; seen < (int)li.size && lim < r2; ++seen) {
              const int t = cm.c_list[wm_ffs(bits)];
              bits &= bits - 1;
              if (fails_with_margin(lat_m, sub(o_tau[t], k3z))) break;
              ++lim;
            }
          } else {
            for (int p = cm.c_start[li.g], seen = 0; seen < (int)li.size && lim < r2; ++p) {
              const int t = cm.c_list[p];
              if (t >= d) continue;
              ++seen;
              if (fails_with_margin(lat_m, sub(o_tau[t], k3z))) break;
              ++lim;
            }
          }
          mem2 += (int64_t)lim * c_len[li.g];
          lat2 = add(lat2, mul(i2d(lim), c_w[li.g]));
          r2 -= lim;
        }
        live = r2 == 0 && !(fails_with_margin(i2d(mem2), mem_cap) ||
                            fails_with_margin(mul(lat2, 0.999999999999), lat_cap));
      }
    }
    // unranking tables for surviving widths (once per width); counts mode
    // needs every call's vector count, skipped or not
    {
      const bool need = live || (cm.on && c < total_calls);
      const uint64_t bit = need ? (1ULL << (d - 1)) : 0ULL;
      uint64_t want = (uint64_t)__reduce_or_sync(EB_FULL, (unsigned)bit) |
                      ((uint64_t)__reduce_or_sync(EB_FULL, (unsigned)(bit >> 32)) << 32);
      want &= ~built;
      if (Gi < 4) want = 0;                                     // <= 3 levels everywhere: closed form
      bool ok = true;
      while (want) {
        const int dd = __ffsll((long long)want);
        want &= want - 1;
        if (ncls_d[dd - 1] >= 4) ok &= build_pq(dd);             // <= 3 levels: closed form (pq_closed)
        EB_STAT(5, 1);
        built |= 1ULL << (dd - 1);
      }
      if (!ok) return false;
    }
    uint32_t cnt = 0, nall = 0;
    if (live || (cm.on && c < total_calls)) {
      const LevelInfo* row = lvl + (size_t)(d - 1) * Gi;
      if (ncls_d[d - 1] == 1) {
        nall = (z <= row[0].size) ? 1u : 0u;
      } else {
        const uint32_t* P1 = pq + (size_t)(d - 1) * LV * W;        // level 1
        const int m1 = ncls_d[d - 1];
        const int hi0 = min(z, (int)row[0].size), lo0 = max(0, z - (int)row[0].tail_next);
        if (hi0 < lo0) nall = 0u;
        else if (m1 <= 3) nall = pq_closed(row, m1, 0, z - lo0 + 1) - pq_closed(row, m1, 0, z - hi0);
        else nall = P1[z - lo0 + 1] - P1[z - hi0];
      }
      cnt = live ? nall : 0u;
    }
    uint64_t nall_before = 0, nall_tot = 0;   // counts mode: vectors of earlier calls / whole window
    if (cm.on) {
      uint64_t ia = nall;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        uint64_t t = __shfl_up_sync(EB_FULL, ia, o);
        if (lane >= o) ia += t;
      }
      nall_before = ia - nall;
      nall_tot = __shfl_sync(EB_FULL, ia, 31);
    }
    uint32_t inc = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t t = __shfl_up_sync(EB_FULL, inc, o);
      if (lane >= o) inc += t;
    }
    const uint32_t T = __shfl_sync(EB_FULL, inc, 31);
#ifdef EB_STATS
    { const unsigned lv = __ballot_sync(EB_FULL, live); EB_STAT(6, __popc(lv)); }
#endif
    EB_STAT(2, T > 0);
    EB_STAT(4, T);
    if (T == 0) { cm_before += nall_tot; continue; }
    pre[lane] = inc - cnt;
    pre[32 + lane] = (uint32_t)((z << 8) | d);                      // call of this slot
    pre64[lane] = nall_before;
    __syncwarp();
    for (uint32_t b0 = 0; b0 < T; b0 += 32) {
      const uint32_t g = b0 + lane;
      EB_STAT(3, 1);
      bool pass = false;
      int klast = 0, zz = 0, dd = 0, slot = 0;
      uint32_t i0 = 0;
      uint64_t V0 = 0, V1 = 0;
      if (g < T) {
        int a = 0, bnd = 31;                                       // largest slot with pre[slot] <= g
        while (a < bnd) {
          int mid = (a + bnd + 1) >> 1;
          if (pre[mid] <= g) a = mid; else bnd = mid - 1;
        }
        const uint32_t zd = pre[32 + a];
        zz = (int)(zd >> 8);
        dd = (int)(zd & 0xff);
        uint32_t i = g - pre[a];
        slot = a;
        i0 = i;
        const double k3z = mul(k3, i2d(zz));
        const double slot_cap = has_cap ? sub(slot_base, k3z) : INF;
        const double mem_cap = sub(k2, i2d((int64_t)padded * zz));
        const int m = ncls_d[dd - 1];
        const LevelInfo* row = lvl + (size_t)(dd - 1) * Gi;
        const uint32_t* base = pq + (size_t)(dd - 1) * LV * W;
        int r = zz;
        double u = 0.0, dl = 0.0, lat = 0.0, tau = INF;
        int64_t mem = 0;
#pragma unroll
        for (int k = 0; k < (FGM ? FGM : m); ++k) {   // FGM > 0: unrolled
          if (FGM && k >= m) break;
          const LevelInfo li = row[k];
          int cc;
          if (k == m - 1) {
            cc = r;
          } else if (k + 1 == m - 1) {
            // one level below: exactly one vector per remaining sum, so the
            // i-th leaf takes hi - i here (the closed-form search's answer)
            cc = min(r, (int)li.size) - (int)i;
            i = 0;
          } else if (k + 1 == m - 2) {
            // two levels below: e(x) = #pairs (c1, c2) <= (s1, s2) summing to
            // x; scan x from the largest count down (the leaf sits in the
            // first few groups), the same answer as the prefix search
            const int s1 = row[k + 1].size, s2 = row[k + 2].size;
            int x = r - min(r, (int)li.size);
            for (;;) {
              const uint32_t e = (uint32_t)(min(x, s1) - max(0, x - s2) + 1);
              if (e > i) break;
              i -= e;
              ++x;
            }
            cc = r - x;
          } else {                                                 // unrank level k
            const uint32_t* P = base + (size_t)k * W;              // level k+1 prefix
            // levels with three or more below: the unranking tables
            auto Pv = [&](int y) -> uint32_t { return P[y]; };
            const int hi = min(r, (int)li.size), lo = max(0, r - (int)li.tail_next);
            const uint32_t pb = Pv(r - hi);
            int xa = r - hi, xz = r - lo;
            while (xa < xz) {
              int mid = (xa + xz) >> 1;
              if (Pv(mid + 1) - pb > i) xz = mid; else xa = mid + 1;
            }
            i -= Pv(xa) - pb;
            cc = r - xa;
          }
          if (cc) { setV<V8>(V0, V1, k, cc); klast = k; }
          // SearchTables.build's up[k][cc] / dn[k][cc] / tau_min_prefix[k][cc]
          // (dftsp.py:119-128): the same sequential folds over the class's
          // first cc members among the dd first by tau, in key order
          double cu = 0.0, cdn = 0.0, tm = INF;
          if constexpr (NI <= 2) {
            // the class's members inside the pool, in key order: set bits of
            // the width mask from the class start on
            WMask bits = (WMask)pm[dd - 1] & ((WMask)~(WMask)0 << cm.c_start[li.g]);
            for (int q = 0; q < cc; ++q) {
              const int p = wm_ffs(bits);
              bits &= bits - 1;
              const double2 kd = cm.c_kd[p];                    // no tau-rank indirection
              cu = add(cu, kd.x);
              cdn = add(cdn, kd.y);
              if (EXACT) tm = pymin(tm, o_tau[cm.c_list[p]]);
            }
          } else {
            for (int p = cm.c_start[li.g], taken = 0; taken < cc; ++p) {
              const int t = cm.c_list[p];
              if (t < dd) {
                cu = add(cu, cm.o_key[t]);
                cdn = add(cdn, cm.o_dnt[t]);
                if (EXACT) tm = pymin(tm, o_tau[t]);
                ++taken;
              }
            }
          }
          u = add(u, cu);                                          // up_acc + up[k][x]
          dl = add(dl, cdn);
          mem += (int64_t)cc * c_len[li.g];
          lat = add(lat, mul(i2d(cc), c_w[li.g]));
          if (EXACT && cc) tau = pymin(tau, tm);
          r -= cc;
        }
        const double cap = EXACT ? pymin(sub(tau, k3z), slot_cap) : pymin(sub(o_tau[dd - 1], k3z), slot_cap);
        if (!cm.on) {
          pass = leq(u, 1.0) && leq(dl, 1.0) && leq(i2d(mem), mem_cap) && leq(lat, cap);
        } else {
          // check_knapsack(recover_subset(part, counts), coeff, z, tau_min):
          // sequential fold over the recovered members (class order, then
          // cheapest-uplink order among the first dd by tau rank)
          double up2 = 0.0, dn2 = 0.0, lat2 = 0.0;
          int64_t mem2 = 0;
          for (int k = 0; k < m; ++k) {
            const LevelInfo li = row[k];
            const int want = getV<V8>(V0, V1, k);
            if constexpr (NI <= 2) {
              WMask bits = (WMask)pm[dd - 1] & ((WMask)~(WMask)0 << cm.c_start[li.g]);
              for (int q = 0; q < want; ++q) {
                const int t = cm.c_list[wm_ffs(bits)];
                bits &= bits - 1;
                up2 = add(up2, cm.o_key[t]);                       // up += k_up * s
                dn2 = add(dn2, cm.o_dnt[t]);                       // dn += k_down * n
                mem2 += c_len[li.g];                               // mem += n
                lat2 = add(lat2, c_w[li.g]);                       // lat += latency_weight(n)
              }
            } else {
              int taken = 0;
              for (int p = cm.c_start[li.g]; taken < want; ++p) {
                const int t = cm.c_list[p];
                if (t >= dd) continue;
                up2 = add(up2, cm.o_key[t]);                       // up += k_up * s
                dn2 = add(dn2, cm.o_dnt[t]);                       // dn += k_down * n
                mem2 += c_len[li.g];                               // mem += n
                lat2 = add(lat2, c_w[li.g]);                       // lat += latency_weight(n)
                ++taken;
              }
            }
          }
          const double cap2 = pymin(sub(o_tau[dd - 1], k3z), slot_cap);   // min(tau_min, slot_budget(z))
          pass = leq(up2, 1.0) && leq(dn2, 1.0) && leq(i2d(mem2), mem_cap) && leq(lat2, cap2);
        }
      }
      const unsigned bal = __ballot_sync(EB_FULL, pass);
      if (bal) {
        const int src = __ffs(bal) - 1;
        found = true;
        if (cm.on) {
          const int ws = __shfl_sync(EB_FULL, slot, src);
          const uint32_t wi = __shfl_sync(EB_FULL, i0, src);
          tot_v = cm_before + pre64[ws] + wi + 1;
        }
        zf = __shfl_sync(EB_FULL, zz, src);
        dwin = __shfl_sync(EB_FULL, dd, src);
        kwin = __shfl_sync(EB_FULL, klast, src);
        W0 = __shfl_sync(EB_FULL, V0, src);
        W1 = __shfl_sync(EB_FULL, V1, src);
        break;
      }
    }
    if (!found) cm_before += nall_tot;
    __syncwarp();
  }
  best = found ? (n - zf) * (n - zf + 1) / 2 + (dwin - zf) : INT_MAX;
  EB_STAT(7, found ? best + 1 : total_calls);

  phase_barrier<2>(passed);
  if (cm.on) {                       // nodes = count vectors tried; no pruning
    if (!found) tot_v = cm_before;
    tot_p = 0;
    return true;
  }
  // ---- C: node counts.  Calls (z, d) counted: z > zf (all d >= z), and
  //      z == zf with d < dwin; plus the winner's partial count.
  //      Lanes = pool widths d: each runs the level recurrence for its own
  //      partition sequentially over r in one u32 row, in place (F(k, r)
  //      reads PF_{k+1} only at indices <= r, so r descends, then a running
  //      prefix), inside the prefix-table region that is free once the search
  //      is done.  The winner's width (it also needs every level for the
  //      partial count) takes the warp-scan path below.
  uint64_t my_v = 0, my_p = 0;
  {
    bool ovf = false;
    uint32_t* rows = (uint32_t*)(smem + L.pq);    // unranking tables are dead now
    const int W2 = 2 * (n + 1);
    for (int dbase = found ? zf : 1; dbase <= n; dbase += 32) {
      const int d = dbase + lane;
      if (d > n || (found && d == dwin)) continue;
      const int m = ncls_d[d - 1];
      const LevelInfo* row = lvl + (size_t)(d - 1) * Gi;
      uint32_t* RV = rows + (size_t)lane * W2;
      uint32_t* RP = RV + (n + 1);
      // deepest level in closed form; level m-2 against it, fused with its
      // running prefix; levels m-3 .. 1 in place over the u32 row (F(k, r)
      // reads PF_{k+1} only at indices <= r, so r descends, then a prefix).
      // Prefix sums are monotone, so checking the last one bounds the row.
      if (ctab != nullptr && m <= 3 && d <= EB_MAX_K && !traj) {     // tabulated shape: two lookups
        const int lo = found ? (d > dwin ? zf + 1 : zf) : 1;
        if (lo <= d) {
          const uint2* T = (const uint2*)((const unsigned char*)ctab + CT_HDR_BYTES) +
                           (size_t)ct_row_closed(m, row[0].size, m > 1 ? row[1].size : 0, m > 2 ? row[2].size : 0) * CT;
          const uint2 a = T[d], b = T[lo - 1];
          my_v += (uint64_t)(a.x - b.x) + (uint64_t)(d - lo + 1);    // + one root per call
          my_p += (uint64_t)(a.y - b.y);
        }
        continue;
      }
      const uint2* ctab_m = (ctab != nullptr && (m == 4 || m == 5) && d <= CTM_K && !traj)
                                ? *(const uint2* const*)((const unsigned char*)ctab + CT_MPTR_OFF) : nullptr;
      if (ctab_m != nullptr) {                                        // four/five classes
        const int lo = found ? (d > dwin ? zf + 1 : zf) : 1;
        if (lo <= d) {
          int t = 0, rank = m == 5 ? CTM_ROWS4 : 0;                  // ctm_row, sizes from the row
#pragma unroll
          for (int i = 0; i < 5; ++i)
            if (i < m) { t += row[i].size; rank += binom_small(t - 1, i + 1); }
          const uint2* T = ctab_m + (size_t)rank * CTM;
          const uint2 a = T[d], b = T[lo - 1];
          my_v += (uint64_t)(a.x - b.x) + (uint64_t)(d - lo + 1);
          my_p += (uint64_t)(a.y - b.y);
        }
        continue;
      }
      const uint32_t sl = row[m - 1].size;
      auto pf_last = [&](int q, uint64_t& v, uint64_t& p) { last_level_prefix<PRUNE, INCL>(sl, (uint32_t)q, v, p); };
      auto pf_row = [&](int q, uint64_t& v, uint64_t& p) { v = RV[q]; p = RP[q]; };
      if (m >= 4) {
        const LevelInfo li = row[m - 2];
        uint64_t av = 0, ap = 0;
        RV[0] = RP[0] = 0;
        for (int r = 1; r <= d; ++r) {
          uint64_t fv, fp;
          level_counts_f<PRUNE, INCL>(li, false, r, pf_last, fv, fp);
          av += fv;
          ap += fp;
          RV[r] = (uint32_t)av;
          RP[r] = (uint32_t)ap;
        }
        ovf |= (av | ap) > 0x7fffffffULL;
        for (int k = m - 3; k >= 1; --k) {
          const LevelInfo lk = row[k];
          for (int r = d; r >= 1; --r) {
            uint64_t fv, fp;
            level_counts_f<PRUNE, INCL>(lk, false, r, pf_row, fv, fp);
            RV[r] = (uint32_t)fv;
            RP[r] = (uint32_t)fp;
          }
          uint64_t bv = 0, bp = 0;
          for (int r = 1; r <= d; ++r) {
            bv += RV[r];
            bp += RP[r];
            RV[r] = (uint32_t)bv;
            RP[r] = (uint32_t)bp;
          }
          ovf |= (bv | bp) > 0x7fffffffULL;
        }
      }
      const LevelInfo l0 = row[0];
      auto level0 = [&](auto pf) {
        for (int r = found ? zf : 1; r <= d; ++r) {
          if (found && r == zf && d > dwin) continue;                // after the winning call
          uint64_t fv, fp;
          level_counts_f<PRUNE, INCL>(l0, m == 1, r, pf, fv, fp);
          fv += 1;                                                   // the root
          my_v += fv;
          my_p += fp;
          if (traj) {
            int64_t* tr = traj + 4 * (int64_t)((n - r) * (n - r + 1) / 2 + (d - r));
            tr[0] = r; tr[1] = d; tr[2] = (int64_t)fv; tr[3] = (int64_t)fp;
          }
        }
      };
      if (m >= 4) {
        level0(pf_row);
      } else if (m == 3) {
        // Level 0 reads PF1 at r - xs and at r - xb - 1, two indices that
        // never decrease with r: stream both prefix sums of F(1, .) (closed
        // form against the last level) instead of storing a row, in u64.
        // level_counts_f asks for the first, then the second, per r.
        const LevelInfo l1 = row[1];
        uint64_t va = 0, pa = 0, vb = 0, pb = 0;
        int qa = 0, qb = 0;
        bool second = false;
        auto adv = [&](int q, int& qq, uint64_t& v, uint64_t& p) {
          for (; qq < q;) {
            ++qq;
            uint64_t fv, fp;
            level_counts_f<PRUNE, INCL>(l1, false, qq, pf_last, fv, fp);
            v += fv;
            p += fp;
          }
        };
        auto pf_stream = [&](int q, uint64_t& v, uint64_t& p) {
          if (!second) { adv(q, qa, va, pa); v = va; p = pa; }
          else { adv(q, qb, vb, pb); v = vb; p = pb; }
          second = !second;
        };
        level0(pf_stream);
      } else {
        level0(pf_last);                                             // m == 2 (m == 1 never reads pf)
      }
    }
    if (__any_sync(EB_FULL, ovf)) return false;                    // exact literal-walk pass instead
    __syncwarp();
  }
  for (int d = dwin; found && d == dwin; ++d) {
    const int m = ncls_d[d - 1];
    const LevelInfo* row = lvl + (size_t)(d - 1) * Gi;
    const uint2* ctab_m = (ctab != nullptr && (m == 4 || m == 5) && d <= CTM_K && !traj)
                              ? *(const uint2* const*)((const unsigned char*)ctab + CT_MPTR_OFF) : nullptr;
    if (ctab != nullptr && !traj && ((m <= 3 && d <= EB_MAX_K) || ctab_m != nullptr)) {
      // Tabulated shape: the calls r > zf of the winning width are one
      // difference of the partition's row (as for the other widths), and the
      // winner's partial count reads PF_{j+1} -- the prefix sums of the level
      // below j -- from the row of the suffix partition (levels j+1 .. m-1):
      // F(j+1, .) depends only on the suffix's sizes and tails, which is what
      // that row tabulates.  The indices stay below the suffix's total (the
      // path reaches the winning leaf), inside the row.
      if (lane == 0) {
        const uint2* CT0 = (const uint2*)((const unsigned char*)ctab + CT_HDR_BYTES);
        auto trow = [&](int j0, int ms) -> const uint2* {     // levels j0 .. j0 + ms - 1
          if (ms <= 3)
            return CT0 + (size_t)ct_row_closed(ms, row[j0].size, ms > 1 ? row[j0 + 1].size : 0,
                                               ms > 2 ? row[j0 + 2].size : 0) * CT;
          int t = 0, rank = ms == 5 ? CTM_ROWS4 : 0;         // ctm_row over the sizes
          for (int i = 0; i < ms; ++i) { t += row[j0 + i].size; rank += binom_small(t - 1, i + 1); }
          return ctab_m + (size_t)rank * CTM;
        };
        const uint2* T = trow(0, m);
        my_v += (uint64_t)(T[d].x - T[zf].x) + (uint64_t)(d - zf);      // + one root per call
        my_p += (uint64_t)(T[d].y - T[zf].y);
        uint64_t fv = 1, fp = 0;
        int rr = zf;
        for (int j = 0; j < kwin; ++j) {
          const int c = getV<V8>(W0, W1, j);
          const int x0 = min(rr, (int)row[j].size);
          const int xb = (x0 == rr) ? x0 - 1 : x0;
          fv += (uint64_t)(x0 - c) + 1;
          if (xb >= c + 1) {
            const uint2* S = trow(j + 1, m - j - 1);                     // suffix levels (>= 1)
            fv += (uint64_t)(S[rr - c - 1].x - S[rr - xb - 1].x);
            fp += (uint64_t)(S[rr - c - 1].y - S[rr - xb - 1].y);
          }
          rr -= c;
        }
        my_v += fv + 1;                                                  // the leaf itself
        my_p += fp;
      }
      continue;
    }
    const int kc = m - 1;    // all levels (the partial count walks them)
    for (int k = kc; k >= 1; --k) {
      const uint64_t* NV = pfv + (size_t)(k + 1) * (n + 1);
      const uint64_t* NP = pfp + (size_t)(k + 1) * (n + 1);
      uint64_t* KV = pfv + (size_t)k * (n + 1);
      uint64_t* KP = pfp + (size_t)k * (n + 1);
      const LevelInfo li = row[k];
      const bool last = (k == m - 1);
      if (last) {
        for (int r = lane; r <= n; r += 32) {
          uint64_t v, p;
          last_level_prefix<PRUNE, INCL>(li.size, (uint32_t)r, v, p);
          KV[r] = v;
          KP[r] = p;
        }
      } else {
        warp_prefix2<NI + 1>(n,
            [&](int r, uint64_t& a, uint64_t& b) {
              if (r == 0) { a = b = 0; return; }
              level_counts<PRUNE, INCL>(li, false, r, NV, NP, a, b);
            },
            [&](int r, uint64_t a, uint64_t b) { KV[r] = a; KP[r] = b; });
      }
      __syncwarp();
    }
    const LevelInfo l0 = row[0];
    for (int r = 1 + lane; r <= d; r += 32) {
      const bool win = found && r == zf && d == dwin;
      const bool counted = !found || r > zf || (r == zf && d < dwin);
      if (!win && !counted) continue;
      uint64_t fv, fp;
      if (!win) {
        level_counts<PRUNE, INCL>(l0, m == 1, r, pfv + (size_t)(n + 1), pfp + (size_t)(n + 1), fv, fp);
        fv += 1;                                                   // the root
      } else {
        // nodes before the winning leaf: root, then per level j < kwin the
        // earlier siblings x in (c_j, x0_j] with their full subtrees, the path
        // node c_j; finally the leaf itself (first node of level kwin).
        fv = 1;
        fp = 0;
        int rr = r;
        for (int j = 0; j < kwin; ++j) {
          const LevelInfo lj = row[j];
          const int c = getV<V8>(W0, W1, j);
          const int x0 = min(rr, (int)lj.size);
          const int xb = (x0 == rr) ? x0 - 1 : x0;
          fv += (uint64_t)(x0 - c) + 1;
          if (xb >= c + 1) {
            const uint64_t* SV = pfv + (size_t)(j + 1) * (n + 1);
            const uint64_t* SP = pfp + (size_t)(j + 1) * (n + 1);
            fv += SV[rr - c - 1] - SV[rr - xb - 1];
            fp += SP[rr - c - 1] - SP[rr - xb - 1];
          }
          rr -= c;
        }
        fv += 1;
      }
      my_v += fv;
      my_p += fp;
      if (traj) {
        int64_t* tr = traj + 4 * (int64_t)((n - r) * (n - r + 1) / 2 + (d - r));
        tr[0] = r; tr[1] = d; tr[2] = (int64_t)fv; tr[3] = (int64_t)fp;
      }
    }
    __syncwarp();
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    my_v += __shfl_xor_sync(EB_FULL, my_v, o);
    my_p += __shfl_xor_sync(EB_FULL, my_p, o);
  }
  tot_v = my_v;
  tot_p = my_p;
  return true;
}

// Error / empty exit of one instance (kept out of line: one copy serves
// every early-exit site, which keeps the kernel's instruction footprint small).
// Per-context constants of the search, derived with the reference's exact
// operations once per context -- per block for the lockstep kernels' first
// EB_DC_CACHE contexts, per warp otherwise -- instead of once per instance.
// The integer polynomials of the padded length are expanded (exact
// integers): gen_base(s) = gb0 + fd4 s, flops_initial(s) = s (fa + fb s).
struct DCtx {
  Ctx c;
  int64_t m1, kv, gb0, fd4, fa, fb;
  double headroom, k2, k5, slot_base;
  double sb_up, sb_dn;                      // T_up * B_up, T_dn * B_dn (radio.py:75, :83)
  double g_a, g_b, g_c, g_w, g_m;           // overflow-guard polynomials (estimates, 4x margin)
};
#define EB_DC_CACHE 8

__device__ __noinline__ void derive_dctx(const eb_context* p, DCtx& D) {
  const Ctx C = load_ctx(p);
  D.c = C;
  const int64_t L = C.m.L, d = C.m.d, f = C.m.ffn;
  D.m1 = weight_bytes(C.m);                                  // costs.py:62-67
  D.kv = kv_per_token(C.m);                                  // costs.py:70-72
  D.gb0 = 8 * d * d + 4 * d * f;                             // feasibility.py:155 without the s term
  D.fd4 = 4 * d;
  D.fa = L * (8 * d * d + 4 * d * f);                        // costs.py:87-97 expanded in s
  D.fb = 4 * L * d;
  D.headroom = sub(div(C.M, C.alpha), i2d(D.m1));            // feasibility.py:144
  D.k2 = div(D.headroom, i2d(D.kv));                         // feasibility.py:152
  D.k5 = i2d(2 * L * d);                                     // feasibility.py:159
  D.slot_base = C.has_cap ? div(mul(C.cap_s, C.C), C.beta) : 0.0;   // feasibility.py:124
  D.sb_up = mul(C.T_up, C.B_up);
  D.sb_dn = mul(C.T_dn, C.B_dn);
  const double Ld = (double)L, dd = (double)d, fd = (double)f, bp = (double)C.m.bpp;
  D.g_a = Ld * (8.0 * dd * dd + 4.0 * dd * fd);
  D.g_b = Ld * 4.0 * dd;
  D.g_c = Ld * 2.0 * dd;
  D.g_w = Ld * (4.0 * bp * dd * (double)C.m.head_dim * (double)C.m.heads + 2.0 * bp * dd * fd);
  D.g_m = 2.0 * bp * Ld * dd;
}

// uplink / downlink fractions per token (radio.py:71-84) with the slot x
// band products of the context precomputed (same operations, same order)
__device__ __forceinline__ int k_up_d(const DCtx& D, double gain, double pup, double* out) {
  const Ctx& c = D.c;
  if (pup <= 0.0 || gain <= 0.0 || c.N0_up <= 0.0) { *out = 0.0; return EB_ERR_NONPOSITIVE_LINK; }
  const double eff = spectral_efficiency(pup, gain, c.N0_up);
  if (eff <= 0.0) { *out = 0.0; return EB_ERR_UPLINK_EFF_ZERO; }    // radio.py:74
  *out = div(c.fbits, mul(D.sb_up, eff));
  return 0;
}
__device__ __forceinline__ int k_dn_d(const DCtx& D, double gain, double* out) {
  const Ctx& c = D.c;
  if (c.P_dn <= 0.0 || gain <= 0.0 || c.N0_dn <= 0.0) { *out = 0.0; return EB_ERR_NONPOSITIVE_LINK; }
  const double eff = spectral_efficiency(c.P_dn, gain, c.N0_dn);
  if (eff <= 0.0) { *out = 0.0; return EB_ERR_DOWNLINK_EFF_ZERO; }  // radio.py:82
  *out = div(c.fbits, mul(D.sb_dn, eff));
  return 0;
}

__device__ __noinline__ void write_status(const eb_dftsp_result& O, int64_t inst, int64_t r0, int n, int st,
                                          int err) {
  const int lane = threadIdx.x & 31;
  if (lane == 0) {
    O.status[inst] = st;
    if (O.error_index) O.error_index[inst] = err;
    O.z_found[inst] = 0;
    O.nodes_visited[inst] = 0;
    O.nodes_pruned[inst] = 0;
    if (O.n_classes) O.n_classes[inst] = 0;
    if (O.traj_len) O.traj_len[inst] = 0;
    if (O.solution_mask) O.solution_mask[inst] = 0ULL;
  }
  if (O.metrics && lane < EB_N_METRICS) O.metrics[inst * EB_N_METRICS + lane] = 0.0;
  if (lane < EB_MAX_CLASSES) {
    if (O.counts) O.counts[inst * EB_MAX_CLASSES + lane] = 0;
    if (O.class_lengths) O.class_lengths[inst * EB_MAX_CLASSES + lane] = 0;
  }
  if (O.solution)
    for (int j = lane; j < n; j += 32) O.solution[r0 + j] = -1;
}

// FK > 0: the launch's layout is make_lay(FK / 100, FK % 100, EXACT, v2)
// (K bound, class bound), known at compile time -- shared-memory offsets
// become immediates; 0: A.lay.
template <bool PRUNE, bool INCL, bool EXACT, int ALGO, int NI, int FK = 0>
__device__ void solve_instance(const DftspArgs& A, int64_t inst, unsigned char* smem, int& passed,
                               const DCtx* dcache, int ncache, DCtx* dslot,
                               bool have_meta = false, int64_t m_row0 = 0, int64_t m_row1 = 0, int m_ci = 0) {
  const int lane = threadIdx.x & 31;
  constexpr bool V8 = FK > 0 && FK % 100 <= 8;   // count vectors fit one u64
  const int K = A.K, G = A.G;
  constexpr Lay LF = make_lay(FK > 0 ? FK / 100 : 1, FK > 0 ? FK % 100 : 1, EXACT, ALGO == 2);
  const Lay& L = FK > 0 ? LF : A.lay;       // computed once on the host (make_lay)
  double* a_tau = (double*)(smem + L.a_tau);
  double* a_key = (double*)(smem + L.a_key);
  int64_t* a_id = (int64_t*)(smem + L.a_id);
  int32_t* a_len = (int32_t*)(smem + L.a_len);
  double* o_tau = (double*)(smem + L.o_tau);
  double* o_key = (double*)(smem + L.o_key);
  double* o_dnt = (double*)(smem + L.o_dnt);
  double* o_ws = (double*)(smem + L.o_ws);
  double* o_dl = (double*)(smem + L.o_dl);
  int64_t* o_id = (int64_t*)(smem + L.o_id);
  int32_t* o_s = (int32_t*)(smem + L.o_s);
  int32_t* o_len = (int32_t*)(smem + L.o_len);
  uint8_t* o_local = smem + L.o_local;
  uint8_t* o_g = smem + L.o_g;
  uint8_t* o_kr = smem + L.o_kr;
  int32_t* c_len = (int32_t*)(smem + L.c_len);
  double* c_w = (double*)(smem + L.c_w);
  int32_t* c_start = (int32_t*)(smem + L.c_start);
  int32_t* c_cnt = (int32_t*)(smem + L.c_cnt);
  uint8_t* c_list = smem + L.c_list;
  uint8_t* sizes = smem + L.sizes;
  uint8_t* ncls_d = smem + L.ncls;
  LevelInfo* lvl = (LevelInfo*)(smem + L.lvl);
  // per-width prefix tables: the literal walk only (v2 folds on the fly)
  double* t_up = ALGO == 1 ? (double*)(smem + L.t_up) : nullptr;
  double* t_dn = ALGO == 1 ? (double*)(smem + L.t_dn) : nullptr;
  double* t_tau = (ALGO == 1 && EXACT) ? (double*)(smem + L.t_tau) : nullptr;
  uint64_t* ring_v = (uint64_t*)(smem + L.ring_v);
  uint64_t* ring_p = (uint64_t*)(smem + L.ring_p);
  uint8_t* ring_done = smem + L.ring_done;
  uint8_t* sol = smem + L.sol;

  const eb_dftsp_result& O = A.out;
  // meta (lockstep kernel): offsets[inst], offsets[inst + 1] and the
  // context index, loaded a round ahead
  const int64_t row0 = have_meta ? m_row0 : A.offsets[inst];
  const int n = (int)((have_meta ? m_row1 : A.offsets[inst + 1]) - row0);
  const int64_t r0 = row0 - A.req_base;

  auto put_status = [&](int st, int err) { write_status(O, inst, r0, n, st, err); };

  int ci = have_meta ? m_ci : (A.ctx_index ? A.ctx_index[inst] : 0);
  if (ci < 0 || ci >= A.n_ctx) { put_status(EB_ERR_INVALID_ARG, -1); return; }
  if (n == 0) { put_status(EB_OK, -1); return; }     // dftsp.py:253-254
  if (n > K || n > 32 * NI) { put_status(EB_ERR_K_TOO_LARGE, -1); return; }
  const DCtx* D = dcache + ci;
  if (ci >= ncache) {
    if (lane == 0) derive_dctx(&A.ctxs[ci], *dslot);
    __syncwarp();
    D = dslot;
  }
  const Ctx& C = D->c;

  // ---------------- setup: per request (lanes over i = lane, lane+32) -----
  int s_i[NI], len_i[NI];
  int64_t id_i[NI];
  double dl_i[NI], w_i[NI], g_i[NI], p_i[NI];
  int padded = 0;
#pragma unroll
  for (int h = 0; h < NI; ++h) {
    int i = lane + 32 * h;
    id_i[h] = 0;
    if (i < n) {
      int64_t r = r0 + i;
      s_i[h] = A.req.prompt_tokens[r];
      len_i[h] = A.req.output_tokens[r];
      id_i[h] = A.req.id[r];
      dl_i[h] = A.req.deadline_s[r];
      w_i[h] = A.req.waiting_s[r];
      g_i[h] = A.req.channel_gain[r];
      p_i[h] = A.req.uplink_power_w[r];
      a_id[i] = id_i[h];
      a_len[i] = len_i[h];
      padded = max(padded, s_i[h]);
    }
  }
  padded = __reduce_max_sync(EB_FULL, padded);             // dftsp.py:255
  __syncwarp();
  // NaN deadline / waiting / gain / power: the reference then orders the
  // pool by CPython's sort on unordered keys (dftsp.py:257, :81), which no
  // rank-based order reproduces -- a documented status instead (DESIGN.md §1,
  // pinned by tests/golden/edge.npz).
  {
    int err_nan = INT_MAX;
#pragma unroll
    for (int h = 0; h < NI; ++h) {
      const int i = lane + 32 * h;
      if (i < n && (isnan(dl_i[h]) || isnan(w_i[h]) || isnan(g_i[h]) || isnan(p_i[h]))) err_nan = min(err_nan, i);
    }
    err_nan = __reduce_min_sync(EB_FULL, err_nan);
    if (err_nan != INT_MAX) { put_status(EB_ERR_NAN_INPUT, err_nan); return; }
  }
  // Duplicate ids (coefficients are keyed by id, feasibility.py:164-166).
  int err_dup = INT_MAX;
  const unsigned active = (n >= 32) ? EB_FULL : ((1u << n) - 1u);
  if constexpr (NI == 1) {
    // one request per lane: lanes holding the same id, via a match
    const unsigned long long key = (lane < n) ? (unsigned long long)id_i[0] : ~0ULL;
    const unsigned same = __match_any_sync(EB_FULL, key) & active;
    if (lane < n && (same & lanemask_lt())) err_dup = lane;
  } else {
    // within each 32-request slice by a match; against the earlier slices by
    // a branch-free scan
#pragma unroll
    for (int h = 0; h < NI; ++h) {
      const int i = lane + 32 * h;
      const int left = n - 32 * h;
      const unsigned act_h = left >= 32 ? EB_FULL : (left > 0 ? ((1u << left) - 1u) : 0u);
      const unsigned long long key = (i < n) ? (unsigned long long)id_i[h] : ~0ULL;
      const unsigned same = __match_any_sync(EB_FULL, key) & act_h;
      bool dup = i < n && (same & lanemask_lt());
      if (h > 0 && i < n)
        for (int j = 0; j < 32 * h; ++j) dup |= (a_id[j] == id_i[h]);
      if (dup) err_dup = min(err_dup, i);
    }
  }
  err_dup = __reduce_min_sync(EB_FULL, err_dup);
  if (err_dup != INT_MAX) { put_status(EB_ERR_DUPLICATE_ID, err_dup); return; }
  // ids rising along the rows (the common layout): the solution's id order
  // is then its row order (finish)
  bool ids_rise;
  {
    bool rise = true;
#pragma unroll
    for (int h = 0; h < NI; ++h) {
      int64_t nx = __shfl_down_sync(EB_FULL, id_i[h], 1);
      if (h + 1 < NI) {
        const int64_t nx2 = __shfl_sync(EB_FULL, id_i[h + 1 < NI ? h + 1 : h], 0);
        if (lane == 31) nx = nx2;
      }
      if (lane + 32 * h + 1 < n) rise &= id_i[h] < nx;
    }
    ids_rise = __all_sync(EB_FULL, rise);
  }

  // The exact integer cost model runs in int64: refuse instances whose
  // FLOP / byte counts could leave its range (double estimate, 4x margin).
  {
    int nmx = 0;
#pragma unroll
    for (int h = 0; h < NI; ++h)
      if (lane + 32 * h < n) nmx = max(nmx, len_i[h]);
    nmx = __reduce_max_sync(EB_FULL, nmx);
    const double s = (double)padded, o = (double)nmx;
    const double fi = s * (D->g_a + D->g_b * s);              // flops_initial(s)
    const double far = o * (D->g_a + D->g_b * s + D->g_c * o); // flops_autoregressive(s, o)
    const double mem = D->g_w + D->g_m * (s + o) * (double)n;
    if ((double)n * (fi + far) > 0x1p61 || mem > 0x1p61) { put_status(EB_ERR_OVERFLOW, -1); return; }
  }

  // derive_coefficients feasibility.py:133-167
  const int64_t m1 = D->m1;
  if (D->headroom < 0) { put_status(EB_ERR_WEIGHTS_DO_NOT_FIT, -1); return; }
  const int64_t kv = D->kv;
  const int64_t gb = D->gb0 + D->fd4 * padded;                        // gen_base(padded)
  const int64_t fi_pad = (int64_t)padded * (D->fa + D->fb * padded);  // flops_initial(padded)
  const double k2 = D->k2;
  const double k3 = i2d(fi_pad - C.m.L * gb);
  const double k4 = i2d(C.m.L * (gb - 2 * C.m.d));
  const double k5 = D->k5;
  const double slot_base = D->slot_base;                              // feasibility.py:124

  double key_i[NI], dnt_i[NI], tau_i[NI];
  int err_link = INT_MAX, err_code = 0;
#pragma unroll
  for (int h = 0; h < NI; ++h) {
    int i = lane + 32 * h;
    key_i[h] = dnt_i[h] = tau_i[h] = 0.0;
    if (i < n) {
      double ku, kd;
      int st = k_up_d(*D, g_i[h], p_i[h], &ku);
      if (!st) st = k_dn_d(*D, g_i[h], &kd);
      if (st) {
        if (i < err_link) { err_link = i; err_code = st; }
      } else {
        key_i[h] = mul(i2d(s_i[h]), ku);       // min_uplink_fraction radio.py:94 (== k_up * s)
        dnt_i[h] = mul(kd, i2d(len_i[h]));     // dftsp.py:127  k_down * n
        tau_i[h] = tau_base_of(C, dl_i[h], w_i[h]);
        a_tau[i] = tau_i[h];
        a_key[i] = key_i[h];
      }
    }
  }
  {
    int e = __reduce_min_sync(EB_FULL, err_link);
    if (e != INT_MAX) {
      int code = __shfl_sync(EB_FULL, err_code, e & 31);
      // lane (e & 31) holds item e in slot h = e >> 5; err_code is that lane's min
      put_status(code, e);
      return;
    }
  }
  {
    // a NaN normalized deadline from finite-looking inputs (an infinite
    // deadline minus an infinite wait): the same undefined order as NaN inputs
    int e = INT_MAX;
#pragma unroll
    for (int h = 0; h < NI; ++h)
      if (lane + 32 * h < n && isnan(tau_i[h])) e = min(e, lane + 32 * h);
    e = __reduce_min_sync(EB_FULL, e);
    if (e != INT_MAX) { put_status(EB_ERR_NAN_INPUT, e); return; }
  }
  __syncwarp();

  // order = sorted by (-tau_base, id) (dftsp.py:257); classes by ascending
  // output length with within-class order (key, id) (dftsp.py:71-82).
  int t_i[NI], gcls_i[NI], kr_i[NI];
  bool first_i[NI];
  unsigned peers = 0;     // NI == 1: lanes with my output length
  unsigned tau_ties = 0;  // NI == 1: other lanes with my tau
  if constexpr (NI == 1) {
    peers = __match_any_sync(EB_FULL, lane < n ? len_i[0] : -1) & active;
    const double tz = tau_i[0] == 0.0 ? 0.0 : tau_i[0];
    tau_ties = __match_any_sync(EB_FULL, lane < n ? (unsigned long long)__double_as_longlong(tz) : ~0ULL) & active &
               ~(1u << lane);
  }
#pragma unroll
  for (int h = 0; h < NI; ++h) {
    int i = lane + 32 * h;
    t_i[h] = gcls_i[h] = kr_i[h] = 0;
    first_i[h] = false;
    if (i < n) {
      int t = 0;
      bool first = true;
      if constexpr (NI == 1) {
        // tau rank: requests with a larger tau, then equal-tau requests with a
        // smaller id (lanes holding the same tau, by a match; -0.0 is
        // folded onto +0.0 so that equal doubles match)
        const double2* a_tau2 = (const double2*)a_tau;
        int j = 0;
#pragma unroll 2
        for (; j + 1 < n; j += 2) {
          const double2 v = a_tau2[j >> 1];
          t += (int)(v.x > tau_i[h]) + (int)(v.y > tau_i[h]);
        }
        if (j < n) t += (int)(a_tau[j] > tau_i[h]);
        first = (peers & lanemask_lt()) == 0;
      } else {
        // one branch-free pass: tau rank, class leadership, within-class rank
        int kr = 0, earlier = 0;
        for (int j = 0; j < n; ++j) {
          const double tj = a_tau[j], kj = a_key[j];
          const int idlt = (int)(a_id[j] < id_i[h]);
          const int same = (int)(a_len[j] == len_i[h]);
          t += (int)(tj > tau_i[h]) | ((int)(tj == tau_i[h]) & idlt);
          earlier |= (int)(j < i) & same;
          kr += same & ((int)(kj < key_i[h]) | ((int)(kj == key_i[h]) & idlt));
        }
        first = !earlier;
        kr_i[h] = kr;
      }
      if constexpr (NI == 1)
        for (unsigned m = tau_ties; m; m &= m - 1) t += (int)(a_id[__ffs(m) - 1] < id_i[h]);
      t_i[h] = t;
      first_i[h] = first;
    }
  }
  // class index = number of distinct lengths below mine
  unsigned fmask[NI];     // class leaders: bit (i & 31) of word i >> 5
  int Gi = 0;
#pragma unroll
  for (int h = 0; h < NI; ++h) {
    fmask[h] = __ballot_sync(EB_FULL, first_i[h]);
    Gi += __popc(fmask[h]);
  }
  if (Gi > G || Gi > EB_MAX_CLASSES) { put_status(EB_ERR_TOO_MANY_CLASSES, -1); return; }
  // Ladder check: the first off-ladder request in tau order (dftsp.py:63-70).
  int bad_t = INT_MAX, bad_i = -1;
  if (A.prm.ladder_len > 0) {
#pragma unroll
    for (int h = 0; h < NI; ++h) {
      int i = lane + 32 * h;
      if (i < n) {
        bool ok = false;
#pragma unroll
        if constexpr (FK > 0) {
          // the compiled-in class bound is the ladder length bound (G = ladder_len)
#pragma unroll
          for (int q = 0; q < FK % 100; ++q) ok |= (q < A.prm.ladder_len) && A.prm.ladder[q] == len_i[h];
        } else {
          for (int q = 0; q < A.prm.ladder_len; ++q) ok |= A.prm.ladder[q] == len_i[h];
        }
        if (!ok && t_i[h] < bad_t) { bad_t = t_i[h]; bad_i = i; }
      }
    }
  }
  {
    int bt = __reduce_min_sync(EB_FULL, bad_t);
    if (bt != INT_MAX) {
      unsigned who = __ballot_sync(EB_FULL, bad_t == bt);
      int bi = __shfl_sync(EB_FULL, bad_i, __ffs(who) - 1);
      put_status(EB_ERR_OFF_LADDER, bi);
      return;
    }
  }
  unsigned key_ties = 0;   // NI == 1: other lanes with my key (within-class order ties)
  if constexpr (NI == 1) {
    const double kz = key_i[0] == 0.0 ? 0.0 : key_i[0];
    key_ties = __match_any_sync(EB_FULL, lane < n ? (unsigned long long)__double_as_longlong(kz) : ~0ULL) & active &
               ~(1u << lane);
  }
#pragma unroll
  for (int h = 0; h < NI; ++h) {
    int i = lane + 32 * h;
    if (i < n) {
      int g = 0, kr = 0;
      if constexpr (NI == 1) {
        // class index: class leaders with a shorter output; rank among peers
        if constexpr (FK > 0) {
          // at most FK % 100 class leaders
          unsigned fm = fmask[0];
#pragma unroll
          for (int q = 0; q < FK % 100; ++q) {
            if (fm) { g += a_len[__ffs(fm) - 1] < len_i[h]; fm &= fm - 1; }
          }
        } else {
          for (unsigned fm = fmask[0]; fm; fm &= fm - 1) g += a_len[__ffs(fm) - 1] < len_i[h];
        }
        // within-class key rank: two peers per step (independent chains)
        unsigned pm = peers & ~(1u << lane);
        int kr2 = 0;
        while (pm) {
          const int j0 = __ffs(pm) - 1;
          pm &= pm - 1;
          kr += (int)(a_key[j0] < key_i[h]);
          if (pm) {
            const int j1 = __ffs(pm) - 1;
            pm &= pm - 1;
            kr2 += (int)(a_key[j1] < key_i[h]);
          }
        }
        kr += kr2;
        for (unsigned pm = peers & key_ties; pm; pm &= pm - 1) kr += (int)(a_id[__ffs(pm) - 1] < id_i[h]);
      } else {
        // class index: leaders with a shorter output (kr came with the ranks)
#pragma unroll
        for (int q = 0; q < NI; ++q)
          for (unsigned fm = fmask[q]; fm; fm &= fm - 1) g += a_len[32 * q + __ffs(fm) - 1] < len_i[h];
        kr = kr_i[h];
      }
      gcls_i[h] = g;
      kr_i[h] = kr;
      int t = t_i[h];
      o_tau[t] = tau_i[h];
      o_key[t] = key_i[h];
      o_dnt[t] = dnt_i[h];
      o_ws[t] = add(w_i[h], C.slots);   // r.waiting_s + slots (feasibility.py:222)
      o_dl[t] = dl_i[h];
      o_id[t] = id_i[h];
      o_s[t] = s_i[h];
      o_len[t] = len_i[h];
      o_local[t] = (uint8_t)i;
      o_g[t] = (uint8_t)g;
      o_kr[t] = (uint8_t)kr;
      if (first_i[h]) {
        c_len[g] = len_i[h];
        double fn = i2d(len_i[h]);
        c_w[g] = add(mul(k4, fn), mul(mul(k5, fn), fn));   // latency_weight feasibility.py:108
      }
    }
  }
  {
    // class sizes and starts: one ballot per class and 32-request slice
    int acc = 0, my_start = 0, my_cnt = 0;
    for (int g = 0; g < Gi; ++g) {
      int cg = 0;
#pragma unroll
      for (int h = 0; h < NI; ++h) cg += __popc(__ballot_sync(EB_FULL, lane + 32 * h < n && gcls_i[h] == g));
      if (lane == g) { my_start = acc; my_cnt = cg; }
      acc += cg;
    }
    if (lane < Gi) { c_start[lane] = my_start; c_cnt[lane] = my_cnt; }
    if (lane == 0) c_start[Gi] = acc;
  }
  __syncwarp();
#pragma unroll
  for (int h = 0; h < NI; ++h) {
    int i = lane + 32 * h;
    if (i < n) {
      const int p = c_start[gcls_i[h]] + kr_i[h];
      c_list[p] = (uint8_t)t_i[h];
      if constexpr (ALGO == 2 && NI <= 2) ((double2*)(smem + L.c_kd))[p] = make_double2(key_i[h], dnt_i[h]);
    }
  }
  __syncwarp();
  if constexpr (ALGO == 2 && NI <= 2) {
    // width masks: pm[d - 1] = the class-list positions of the d first
    // requests in tau order (an OR-scan over tau ranks), so a leaf's walk
    // over a class visits only the members inside its pool.  `sol` is free
    // until the finish phase: it holds each tau rank's position meanwhile.
    uint64_t* pm = (uint64_t*)(smem + L.pm);
#pragma unroll
    for (int h = 0; h < NI; ++h) {
      const int i = lane + 32 * h;
      if (i < n) sol[t_i[h]] = (uint8_t)(c_start[gcls_i[h]] + kr_i[h]);
    }
    __syncwarp();
    uint64_t carry = 0;
#pragma unroll
    for (int h = 0; h < NI; ++h) {
      const int t = lane + 32 * h;
      uint64_t v = t < n ? (1ULL << sol[t]) : 0ULL;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint64_t u = __shfl_up_sync(EB_FULL, v, o);
        if (lane >= o) v |= u;
      }
      v |= carry;
      if (t < n) pm[t] = v;
      carry = __shfl_sync(EB_FULL, v, 31);
    }
    __syncwarp();
  }

  // ---------------- per pool width d: class sizes, levels, tables --------
  const int nDG = n * Gi;
  (void)nDG;
  if constexpr (NI == 1 && FK > 0) {
    // Compiled-in class bound (FG): lane = tau rank t = width d - 1 computes
    // its width's class sizes by one ballot per class and builds that width's
    // level row from registers (the general path below stores the sizes and
    // reads them back on the same lane).
    constexpr int FG = FK % 100;
    const int t = lane, d = lane + 1;
    const int gt = t < n ? o_g[t] : -1;
    const unsigned below = (2u << lane) - 1u;
    int szr[FG];
#pragma unroll
    for (int g = 0; g < FG; ++g) szr[g] = __popc(__ballot_sync(EB_FULL, gt == g) & below);
    if (t < n) {
      const int base = (d - 1) * d / 2 + (d - 1) * Gi;
      LevelInfo* row = lvl + (size_t)(d - 1) * Gi;
      int k = 0, start = 0, kn = 0;
#pragma unroll
      for (int g = 0; g < FG; ++g) {
        if (g < Gi) {
          const int sz = szr[g];
          sizes[t * Gi + g] = (uint8_t)sz;
          if (g == gt) kn = k;        // level of the class the d-th request joined
          if (sz > 0) {
            LevelInfo li;
            li.off = (uint16_t)(base + start);
            li.size = (uint8_t)sz;
            li.tail_next = 0;
            li.g = (uint8_t)g;
            li.pad[0] = li.pad[1] = li.pad[2] = 0;
            row[k++] = li;
          }
          start += sz + 1;
        }
      }
      ncls_d[d - 1] = (uint8_t)k;
      int tail = 0;
      for (int q = k - 1; q >= 0; --q) { row[q].tail_next = (uint8_t)tail; tail += row[q].size; }
      row[0].pad[0] = (uint8_t)kn;
    }
  } else {
  {
      // sizes[d][g] = members of class g among the d first in tau order: one
      // ballot per class and 32-rank slice over lanes = tau ranks, then lanes =
      // d count the bits below d (earlier slices whole)
  #pragma unroll
      for (int h = 0; h < NI; ++h) {
        const int t = lane + 32 * h;                            // tau rank; width d = t + 1
        const int gt = t < n ? o_g[t] : -1;
        const unsigned below = (t < n) ? ((2u << lane) - 1u) : 0u;
        for (int g = 0; g < Gi; ++g) {
          int full = 0;                                         // class g in slices before h
  #pragma unroll
          for (int q = 0; q < h; ++q) {
            const int tq = lane + 32 * q;
            full += __popc(__ballot_sync(EB_FULL, tq < n && o_g[tq] == g));
          }
          const unsigned mg = __ballot_sync(EB_FULL, gt == g);
          if (t < n) sizes[t * Gi + g] = (uint8_t)(full + __popc(mg & below));
        }
      }
    }
    __syncwarp();
    for (int d = lane + 1; d <= n; d += 32) {
      int base = (d - 1) * d / 2 + (d - 1) * Gi;
      int k = 0, start = 0;
      LevelInfo* row = lvl + (size_t)(d - 1) * Gi;
      // level of the class the d-th request (tau order) joined: the count
      // recurrence of width d differs from width d-1 only at that level and
      // above (row[0].pad[0]; meaningful when the class count is unchanged)
      const int gn = o_g[d - 1];
      int kn = 0;
      for (int g = 0; g < Gi; ++g) {
        int sz = sizes[(d - 1) * Gi + g];
        if (g == gn) kn = k;
        if (sz > 0) {
          LevelInfo li;
          li.off = (uint16_t)(base + start);
          li.size = (uint8_t)sz;
          li.tail_next = 0;
          li.g = (uint8_t)g;
          li.pad[0] = li.pad[1] = li.pad[2] = 0;
          row[k++] = li;
        }
        start += sz + 1;
      }
      ncls_d[d - 1] = (uint8_t)k;
      int tail = 0;
      for (int q = k - 1; q >= 0; --q) { row[q].tail_next = (uint8_t)tail; tail += row[q].size; }
      row[0].pad[0] = (uint8_t)kn;
    }
  }
  if constexpr (ALGO == 1) {
    // the literal walk reads every width's tables; the leaf-parallel search
    // builds them lazily for the widths that have a live call (search_v2)
    for (int w = lane; w < nDG; w += 32)
      build_width_tables<EXACT>(w / Gi + 1, w % Gi, Gi, sizes, c_start, c_list, o_key, o_dnt, o_tau, t_up, t_dn,
                                t_tau);
  }
  if constexpr (ALGO == 1) { ring_done[lane] = 0; ring_done[lane + 32] = 0; }
  __syncwarp();

  phase_barrier<ALGO>(passed);
  // ---------------- search ------------------------------------------------
  const int total_calls = n * (n + 1) / 2;
  const bool collect = A.prm.collect_trajectory && O.traj && O.traj_offsets;
  int64_t* traj = collect ? O.traj + 4 * (O.traj_offsets[inst] - A.traj_base) : nullptr;
  int best = INT_MAX;                // sequence index of the winning dfs call
  uint64_t tot_v = 0, tot_p = 0;
  bool found = false;
  int zf = 0, dwin = 0, kwin = 0;
  uint64_t W0 = 0, W1 = 0;
  if constexpr (ALGO == 2) {
    if (!search_v2<PRUNE, INCL, EXACT, NI, FK>(passed, n, Gi, smem, L, lvl, ncls_d, c_len, c_w, o_tau, k2, k3,
                                       slot_base, C.has_cap, padded, traj, found, zf, dwin, kwin, W0, W1, best,
                                       tot_v, tot_p,
                                       CountsMode{A.prm.exhaustive_counts != 0, c_start, c_list, o_key, o_dnt,
                                                  ALGO == 2 && NI <= 2 ? (const double2*)(smem + L.c_kd) : nullptr},
                                       A.ctab, sizes)) {
      // leaf counts overflow the u32 unranking tables: hand the instance to
      // the literal walk (second pass of launch_dftsp)
      put_status(EB_STATUS_FALLBACK, -1);
      if (lane == 0) atomicAdd(A.counter + 1, 1);
      return;
    }
  } else {
  int next_call = 0, fold = 0;
  tot_v = 0; tot_p = 0;

  Lane S;
  S.z = S.k = S.x = S.sel = S.ncl = 0;
  S.V0 = S.V1 = 0;
  S.vis = S.prn = 0;
  int c = -1, d = 0;
  Tables T;
  T.row = lvl; T.up = t_up; T.dn = t_dn; T.tau = t_tau; T.len = c_len; T.w = c_w;
  int succ_c = INT_MAX, succ_k = 0, succ_d = 0, succ_z = 0;
  uint64_t succ_V0 = 0, succ_V1 = 0;

  auto finish_call = [&](int outcome) {
    int slot = c % RING;
    ring_v[slot] = S.vis; ring_p[slot] = S.prn; ring_done[slot] = 1;
    if (traj) {
      int64_t* tr = traj + 4 * (int64_t)c;
      tr[0] = S.z; tr[1] = d; tr[2] = (int64_t)S.vis; tr[3] = (int64_t)S.prn;
    }
    if (outcome == 2) { succ_c = c; succ_k = S.k; succ_d = d; succ_z = S.z; succ_V0 = S.V0; succ_V1 = S.V1; }
    c = -1;
  };

  for (;;) {
    // 1. hand out calls to idle lanes (in sequence order, lowest lane first)
    int limit = min(total_calls, best);
    limit = min(limit, fold + RING);
    unsigned want = __ballot_sync(EB_FULL, c < 0);
    if (c < 0) {
      int my = next_call + __popc(want & lanemask_lt());
      if (my < limit) {
        c = my;
        int z;
        call_zd(n, c, z, d);
        T.row = lvl + (size_t)(d - 1) * Gi;
        double tau_min = sub(o_tau[d - 1], mul(k3, i2d(z)));       // bases[d-1] - k3*z (dftsp.py:267)
        if (dfs_begin<PRUNE, INCL, EXACT>(S, T, z, d, ncls_d[d - 1], k3, slot_base, C.has_cap, tau_min, k2,
                                          padded))
          finish_call(1);
      }
    }
    next_call += max(0, min(__popc(want), limit - next_call));

    // 2. one node of each running call
    if (c >= 0) {
      int outcome = dfs_step<PRUNE, INCL, EXACT>(S, T);
      if (outcome) finish_call(outcome);
    }

    // 3. first success in sequence order; abort speculative calls behind it
    best = __reduce_min_sync(EB_FULL, succ_c);
    if (c > best) c = -1;
    __syncwarp();
    // 4. fold completed calls in sequence order (uniform across the warp)
    for (;;) {
      int lim = (best == INT_MAX) ? total_calls : best + 1;
      if (fold >= lim || fold >= next_call) break;
      int slot = fold % RING;
      if (!ring_done[slot]) break;
      tot_v += ring_v[slot];
      tot_p += ring_p[slot];
      ++fold;
      __syncwarp();
      if (lane == 0) ring_done[slot] = 0;
      __syncwarp();
    }
    if (best != INT_MAX ? fold > best : fold >= total_calls) break;
  }
  found = best != INT_MAX;
  if (found) {
    unsigned who = __ballot_sync(EB_FULL, succ_c == best);
    int src = __ffs(who) - 1;
    zf = __shfl_sync(EB_FULL, succ_z, src);
    dwin = __shfl_sync(EB_FULL, succ_d, src);
    kwin = __shfl_sync(EB_FULL, succ_k, src);
    W0 = __shfl_sync(EB_FULL, succ_V0, src);
    W1 = __shfl_sync(EB_FULL, succ_V1, src);
  }
  }  // v1

  if constexpr (ALGO == 1) phase_barrier<1>(passed);   // (ALGO 2 passed its own)
  phase_barrier<ALGO>(passed);
  // ---------------- finish ------------------------------------------------
  int status = EB_OK;
  double met[EB_N_METRICS];
#pragma unroll
  for (int q = 0; q < EB_N_METRICS; ++q) met[q] = 0.0;
  met[EB_MET_PADDED] = (double)padded;
  const LevelInfo* wrow = lvl + (size_t)(dwin > 0 ? dwin - 1 : 0) * Gi;
  const int wncls = found ? ncls_d[dwin - 1] : 0;
  if (found) {
    // recover_subset (dftsp.py:85-93) in recover order, then check_direct
    // (feasibility.py:192-223) exactly as dftsp.py:276 calls it.
    if constexpr (NI == 1) {
      // lanes = class-list positions p (class-major, within-class key order):
      // member t = c_list[p] of class g is taken iff t < dwin and fewer than
      // count[level of g] earlier members of g qualify; its slot is the
      // counts of earlier levels plus that rank (same order as the loop below)
      const int t = lane < n ? c_list[lane] : 0;
      const int g = lane < n ? o_g[t] : 0;
      const bool in = lane < n && t < dwin;
      const unsigned inm = __ballot_sync(EB_FULL, in);
      const unsigned present = __reduce_or_sync(EB_FULL, in ? (1u << g) : 0u);
      if (in) {
        const int cs = c_start[g];
        const int rk = __popc(inm & ((1u << lane) - 1u) & ~((1u << cs) - 1u));
        const int kk = __popc(present & ((1u << g) - 1u));
        const int cnt = (kk <= kwin) ? getV<V8>(W0, W1, kk) : 0;
        if (rk < cnt) {
          sol[sumV_below(W0, W1, kk) + rk] = (uint8_t)t;     // kk <= kwin here (cnt > 0)
        }
      }
    } else if constexpr (NI == 2) {
      // the same over two 32-position slices of the class lists
      int tt[2], gg[2];
      bool inb[2];
      unsigned inm[2], present = 0;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int p = lane + 32 * h;
        tt[h] = p < n ? c_list[p] : 0;
        gg[h] = p < n ? o_g[tt[h]] : 0;
        inb[h] = p < n && tt[h] < dwin;
        inm[h] = __ballot_sync(EB_FULL, inb[h]);
        present |= __reduce_or_sync(EB_FULL, inb[h] ? (1u << gg[h]) : 0u);
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (!inb[h]) continue;
        const int p = lane + 32 * h, g = gg[h], cs = c_start[g];
        int rk = 0;                                    // qualifying positions in [cs, p)
#pragma unroll
        for (int w = 0; w < 2; ++w) {
          const int lo = max(cs - 32 * w, 0), hi = min(p - 32 * w, 32);
          if (hi > lo) {
            const unsigned upto = hi == 32 ? EB_FULL : ((1u << hi) - 1u);
            rk += __popc(inm[w] & upto & ~((1u << lo) - 1u));
          }
        }
        const int kk = __popc(present & ((1u << g) - 1u));
        const int cnt = (kk <= kwin) ? getV<V8>(W0, W1, kk) : 0;
        if (rk < cnt) {
          sol[sumV_below(W0, W1, kk) + rk] = (uint8_t)tt[h];   // kk <= kwin here (cnt > 0)
        }
      }
    } else if (lane == 0) {
      int q = 0;
      for (int kk = 0; kk < wncls; ++kk) {
        int cnt = (kk <= kwin) ? getV<V8>(W0, W1, kk) : 0;
        int g = wrow[kk].g;
        int taken = 0;
        for (int p = c_start[g]; p < c_start[g + 1] && taken < cnt; ++p) {
          int t = c_list[p];
          if (t < dwin) { sol[q++] = (uint8_t)t; ++taken; }
        }
      }
    }
    __syncwarp();
    // Lanes = member slots j = lane + 32 h of the subset (recover order).
    // Integer sums are order-free: sum_j flops_autoregressive(s, n_j) =
    // L * (base(s) * S1 + 2 d * S2) with S1 = sum (n_j - 1), S2 = sum
    // (n_j - 1) n_j -- the same integers as the per-member closed forms, so
    // one pair of reductions serves both paddings.
    int t_m[NI], loc_m[NI];
    double key_m[NI], dnt_m[NI];
    int64_t s1 = 0, s2 = 0;
    int pb = 0;
#pragma unroll
    for (int h = 0; h < NI; ++h) {
      const int j = lane + 32 * h;
      t_m[h] = 0;
      loc_m[h] = -1;
      key_m[h] = dnt_m[h] = 0.0;
      if (j < zf) {
        const int t = sol[j];
        const int64_t ln = o_len[t];
        t_m[h] = t;
        loc_m[h] = o_local[t];
        key_m[h] = o_key[t];
        dnt_m[h] = o_dnt[t];
        s1 += ln - 1;
        s2 += (ln - 1) * ln;
        pb = max(pb, o_s[t]);
      }
    }
    s1 = warp_sum_i64(s1);
    s2 = warp_sum_i64(s2);
    const int64_t sn = s1 + zf;                                        // sum of output tokens
    const int64_t fl_pool = (int64_t)zf * fi_pad + C.m.L * (gb * s1 + 2 * C.m.d * s2);
    const double compute_s = compute_seconds(C, fl_pool);
    bool late = false;                                                 // per-member deadline checks
#pragma unroll
    for (int h = 0; h < NI; ++h)
      if (lane + 32 * h < zf) late |= !leq(add(o_ws[t_m[h]], compute_s), o_dl[t_m[h]]);
    late = __any_sync(EB_FULL, late);
    // check_direct's folds in subset order (feasibility.py:203-205): every
    // lane runs the same left fold over the members' registers
    double up = 0.0, dn = 0.0;
#pragma unroll
    for (int h = 0; h < NI; ++h) {
      const int zh = min(zf - 32 * h, 32);
      for (int j = 0; j < zh; ++j) {
        up = add(up, __shfl_sync(EB_FULL, key_m[h], j));     // r.prompt_tokens * k_up
        dn = add(dn, __shfl_sync(EB_FULL, dnt_m[h], j));     // r.output_tokens * k_down
      }
    }
    const int64_t mem = m1 + kv * (int64_t)padded * zf + kv * sn;
    bool ok = leq(up, 1.0) && leq(dn, 1.0) && leq(mul(C.alpha, i2d(mem)), C.M);
    if (ok && C.has_cap) ok = leq(compute_s, C.cap_s);
    if (ok && late) ok = false;
    if (!ok) status = EB_ERR_REVERIFY;
    if (O.metrics) {
      // batch_cost at the batch's own padding (sim.py:372-376)
      pb = __reduce_max_sync(EB_FULL, pb);
      const int64_t mem_b = m1 + kv * (int64_t)pb * zf + kv * sn;
      const int64_t fl_batch = (int64_t)zf * ((int64_t)pb * (D->fa + D->fb * pb)) +
                               C.m.L * ((D->gb0 + D->fd4 * pb) * s1 + 2 * C.m.d * s2);
      met[EB_MET_UP_SUM] = up;
      met[EB_MET_DN_SUM] = dn;
      met[EB_MET_MEM_POOLPAD] = mul(C.alpha, i2d(mem));
      met[EB_MET_LAT_POOLPAD] = compute_s;
      met[EB_MET_MEM_BATCHPAD] = mul(C.alpha, i2d(mem_b));
      met[EB_MET_LAT_BATCHPAD] = compute_seconds(C, fl_batch);
      met[EB_MET_WIN_D] = (double)dwin;
    }
    // the subset's rows as a bit set over local row positions (rows < 64)
    uint32_t rows_lo = 0, rows_hi = 0;
#pragma unroll
    for (int h = 0; h < NI; ++h) {
      const int loc = loc_m[h];
      rows_lo |= (loc >= 0 && loc < 32) ? (1u << loc) : 0u;
      rows_hi |= (loc >= 32 && loc < 64) ? (1u << (loc - 32)) : 0u;
    }
    rows_lo = __reduce_or_sync(EB_FULL, rows_lo);
    if (NI > 1) rows_hi = __reduce_or_sync(EB_FULL, rows_hi);
    // solution sorted by request id (dftsp.py:281)
    if (status == EB_OK && O.solution) {
      if (NI <= 2 && ids_rise) {
        // ids rise along the rows: id order is row order, so a member's
        // slot is the number of member rows before it
#pragma unroll
        for (int h = 0; h < NI; ++h) {
          const int i = lane + 32 * h;
          const uint32_t word = h ? rows_hi : rows_lo;
          if (i < n && ((word >> lane) & 1u))
            O.solution[r0 + (h ? __popc(rows_lo) : 0) + __popc(word & lanemask_lt())] = i;
        }
      } else {
#pragma unroll
        for (int h = 0; h < NI; ++h) {
          const int j = lane + 32 * h;
          if (j < zf) {
            const int64_t idv = o_id[t_m[h]];
            int rank = 0;
            for (int q = 0; q < zf; ++q) rank += o_id[sol[q]] < idv;
            O.solution[r0 + rank] = loc_m[h];
          }
        }
      }
    }
    if (status == EB_OK && O.solution_mask && lane == 0)
      O.solution_mask[inst] = n <= 64 ? (((uint64_t)rows_hi << 32) | rows_lo) : 0ULL;
  }
  if (O.solution_mask && lane == 0 && (!found || status != EB_OK)) O.solution_mask[inst] = 0ULL;
  // rows past the batch are unused: mark them
  if (O.solution)
    for (int j = lane; j < n; j += 32)
      if (!found || status != EB_OK || j >= zf) O.solution[r0 + j] = -1;
  if (lane == 0) {
    O.status[inst] = status;
    if (O.error_index) O.error_index[inst] = -1;
    O.z_found[inst] = (found && status == EB_OK) ? zf : 0;
    O.nodes_visited[inst] = (int64_t)tot_v;
    O.nodes_pruned[inst] = (int64_t)tot_p;
    if (O.n_classes) O.n_classes[inst] = (found && status == EB_OK) ? wncls : 0;
    if (O.traj_len) O.traj_len[inst] = found ? best + 1 : total_calls;
    if (O.metrics)
      for (int q = 0; q < EB_N_METRICS; ++q) O.metrics[inst * EB_N_METRICS + q] = met[q];
  }
  if (lane < EB_MAX_CLASSES) {
    bool live = found && status == EB_OK && lane < wncls;
    int cnt = 0, clen = 0;
    if (live) {
      cnt = (lane <= kwin) ? getV<V8>(W0, W1, lane) : 0;
      clen = c_len[wrow[lane].g];
    }
    if (O.counts) O.counts[inst * EB_MAX_CLASSES + lane] = cnt;
    if (O.class_lengths) O.class_lengths[inst * EB_MAX_CLASSES + lane] = clen;
  }
}

template <bool PRUNE, bool INCL, bool EXACT, int ALGO, int NI>
__global__ void __launch_bounds__(128, 4) dftsp_kernel(const __grid_constant__ DftspArgs A) {
  extern __shared__ __align__(16) unsigned char smem_all[];
  __shared__ DCtx s_dw[4];
  const int warp = threadIdx.x >> 5;
  unsigned char* smem = smem_all + warp * A.warp_bytes;
  // second (fallback) pass: only instances v2 flagged, and nothing at all
  // when none were flagged
  if (A.fallback_pass && *(volatile int*)(A.counter + 1) == 0) return;
  for (;;) {
    int64_t inst = 0;
    if ((threadIdx.x & 31) == 0) inst = atomicAdd(A.counter, 1);
    inst = __shfl_sync(EB_FULL, inst, 0);
    if (inst >= A.n_inst) break;
    if (A.fallback_pass && A.out.status[inst] != EB_STATUS_FALLBACK) continue;
    int passed = 0;
    solve_instance<PRUNE, INCL, EXACT, ALGO, NI>(A, inst, smem, passed, nullptr, 0, &s_dw[warp]);
    __syncwarp();
  }
}

// Wide instances (EB_MAX_K < n <= EB_MAX_K_DFTSP candidates, e.g. a
// simulator queue with the prefilter off): one warp per block, literal node
// walk, up to 8 requests per lane; the per-instance tables (O(n^2) prefix
// sums) live in shared memory when they fit and in a global scratch slab
// per block otherwise.  Instances come from an atomic counter; the narrow
// ones were solved by the main pass.
template <bool PRUNE, bool INCL, bool EXACT>
__global__ void __launch_bounds__(32, 1) dftsp_wide_kernel(const __grid_constant__ DftspArgs A, unsigned char* gscratch) {
  extern __shared__ __align__(16) unsigned char smem_all[];
  __shared__ DCtx s_dw;
  unsigned char* smem = gscratch ? gscratch + (size_t)blockIdx.x * A.warp_bytes : smem_all;
  for (;;) {
    int64_t inst = 0;
    if (threadIdx.x == 0) inst = atomicAdd(A.counter, 1);
    inst = __shfl_sync(EB_FULL, inst, 0);
    if (inst >= A.n_inst) break;
    const int64_t n = A.offsets[inst + 1] - A.offsets[inst];
    if (n <= EB_MAX_K || n > EB_MAX_K_DFTSP) continue;
    if (A.fallback_pass && A.out.status[inst] != EB_STATUS_FALLBACK) continue;   // after the v2 wide pass
    int passed = 0;
    solve_instance<PRUNE, INCL, EXACT, 1, (EB_MAX_K_DFTSP + 31) / 32>(A, inst, smem, passed, nullptr, 0, &s_dw);
    __syncwarp();
  }
}

// Lockstep variant (leaf-parallel algorithm): the block takes one instance
// per warp per round and all warps cross the same phase barriers.
#ifndef EB_LOCK_THREADS
#define EB_LOCK_THREADS 512
#endif
#ifndef EB_LOCK_MINB
#define EB_LOCK_MINB 1
#endif
template <bool PRUNE, bool INCL, bool EXACT, int NI, int FK = 0>
__device__ __forceinline__ void lock_loop(const DftspArgs& A) {
  extern __shared__ __align__(16) unsigned char smem_all[];
  __shared__ int s_q[3];           // round bases, two rounds ahead (ring of 3)
  __shared__ DCtx s_dc[EB_DC_CACHE];   // derived constants of the first contexts
  // per warp: a context past the cache (<= 16 warps per block; the config-2
  // shapes launch at most 8, and the 2.5 KB saved lets three config-2 blocks
  // fit the 132 KB shared-memory carveout, leaving 124 KB of L1)
  __shared__ DCtx s_dw[(FK == 2003 || FK == 3203) ? 8 : 16];
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  constexpr size_t WB = al8(make_lay(FK > 0 ? FK / 100 : 1, FK > 0 ? FK % 100 : 1, EXACT, true).total);
  unsigned char* smem = smem_all + warp * (FK > 0 ? WB : A.warp_bytes);
  const int64_t total = A.list_count ? (int64_t)*A.list_count : A.n_inst;
  auto inst_of = [&](int64_t slot) -> int64_t { return A.inst_list ? (int64_t)A.inst_list[slot] : slot; };
  // offsets / context index of a round's instance, loaded one round early so
  // the load latency hides behind the current round
  // (scalars, so the loads stay in flight in registers until used)
  auto meta_of = [&](int64_t slot, int64_t& r0, int64_t& r1, int& ci) {
    if (slot < total) {
      const int64_t i = inst_of(slot);
      r0 = A.offsets[i];
      r1 = A.offsets[i + 1];
      ci = A.ctx_index ? A.ctx_index[i] : 0;
    }
  };
  if (threadIdx.x == 0) { s_q[0] = atomicAdd(A.counter, nw); s_q[1] = atomicAdd(A.counter, nw); }
  const int ncache = A.n_ctx < EB_DC_CACHE ? A.n_ctx : EB_DC_CACHE;
  if (threadIdx.x < ncache) derive_dctx(&A.ctxs[threadIdx.x], s_dc[threadIdx.x]);
  __syncthreads();
  int64_t base = s_q[0], nxt = s_q[1];
  int64_t c0 = 0, c1 = 0, a0 = 0, a1 = 0;
  int cci = 0, aci = 0;
  meta_of(base + warp, c0, c1, cci);
  for (int r = 0;; ++r) {
    if (base >= total) break;
    if (threadIdx.x == 0) s_q[(r + 2) % 3] = atomicAdd(A.counter, nw);   // read after this round's barriers
    meta_of(nxt + warp, a0, a1, aci);
    const int64_t slot = base + warp;
    int passed = 0;
    if (slot < total)
      solve_instance<PRUNE, INCL, EXACT, 2, NI, FK>(A, inst_of(slot), smem, passed, s_dc, ncache, &s_dw[warp], true, c0,
                                                   c1, cci);
    __syncwarp();
    for (; passed < 3; ++passed)
      if ((EB_LOCK_BARRIERS >> passed) & 1) __syncthreads();
    base = nxt;
    nxt = s_q[(r + 2) % 3];
    c0 = a0; c1 = a1; cci = aci;
  }
}

// The config-2 shape (FK = 3203) runs at 80 registers and 24 warps per SM:
// 211 M against 184 M inst/s at 128 registers and 16 warps (spills are 132 B
// per thread, L1-resident); config 5 (2005) measured the opposite (83 M at 80
// registers against 97 M), so the other variants keep 128.
// Config 2's shape (K <= 20, three classes, default flags) with its own
// compiled-in layout: 4.8 instead of 6.5 KB of shared memory per warp, which
// leaves the L1 more room for the 80-register build's spills.
#ifndef EB_FK2003
#define EB_FK2003 1
#endif
#ifndef EB_LOCK3203_THREADS
#define EB_LOCK3203_THREADS 256
#endif
static_assert(EB_LOCK3203_THREADS <= 256, "s_dw holds 8 warps for the FK 2003/3203 kernels");
#ifndef EB_LOCK3203_MINB
#define EB_LOCK3203_MINB 3
#endif
#ifndef EB_LOCK2005_THREADS
#define EB_LOCK2005_THREADS EB_LOCK_THREADS
#endif
#ifndef EB_LOCK2005_MINB
#define EB_LOCK2005_MINB EB_LOCK_MINB
#endif
#ifndef EB_LOCK6403_THREADS
#define EB_LOCK6403_THREADS EB_LOCK_THREADS
#endif
#ifndef EB_LOCK6403_MINB
#define EB_LOCK6403_MINB EB_LOCK_MINB
#endif
template <bool PRUNE, bool INCL, bool EXACT, int NI, int FK = 0>
__global__ void __launch_bounds__((FK == 3203 || FK == 2003) ? EB_LOCK3203_THREADS : FK == 2005 ? EB_LOCK2005_THREADS
                                  : FK == 6403 ? EB_LOCK6403_THREADS : EB_LOCK_THREADS,
                                  (FK == 3203 || FK == 2003) ? EB_LOCK3203_MINB : FK == 2005 ? EB_LOCK2005_MINB
                                  : FK == 6403 ? EB_LOCK6403_MINB : EB_LOCK_MINB)
    dftsp_lock_kernel(const __grid_constant__ DftspArgs A) {
  lock_loop<PRUNE, INCL, EXACT, NI, FK>(A);
}

// Wide instances (EB_MAX_K < n <= EB_MAX_K_DFTSP) with at most three classes
// on the leaf-parallel search: up to 8 requests per lane, no unranking
// tables (closed form), count rows past the table range; few warps per SM
// (the per-warp footprint is O(K)), so the full register file per thread.
// NI = 4 serves pools of at most 128 candidates with half the per-lane
// arrays (fewer registers, more resident warps); NI = 8 the rest.
#ifndef EB_WIDE4_THREADS
#define EB_WIDE4_THREADS 128
#endif
#ifndef EB_WIDE4_MINB
#define EB_WIDE4_MINB 3
#endif
template <bool PRUNE, bool INCL, bool EXACT>
__global__ void __launch_bounds__(64, 1) dftsp_lock_wide_kernel(const __grid_constant__ DftspArgs A) {
  lock_loop<PRUNE, INCL, EXACT, (EB_MAX_K_DFTSP + 31) / 32>(A);
}
template <bool PRUNE, bool INCL, bool EXACT>
__global__ void __launch_bounds__(EB_WIDE4_THREADS, EB_WIDE4_MINB) dftsp_lock_wide4_kernel(const __grid_constant__ DftspArgs A) {
  lock_loop<PRUNE, INCL, EXACT, 4>(A);
}

// Indices of the instances wider than EB_MAX_K (order irrelevant).
__global__ void wide_list_kernel(int64_t n, const int64_t* __restrict__ off, int32_t* __restrict__ list,
                                 int* __restrict__ count) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t sz = off[i + 1] - off[i];
    if (sz > EB_MAX_K && sz <= EB_MAX_K_DFTSP) list[atomicAdd(count, 1)] = (int32_t)i;
  }
}


// Single dfs() call on a caller-built partition (dfs(z, part, coeff, tau_min)
// dftsp.py:135-234): builds SearchTables (dftsp.py:110-132) in shared memory
// and runs the same dfs_begin/dfs_step as the batched search.
template <bool PRUNE, bool INCL, bool EXACT>
__global__ void dfs_single_kernel(int z, int ncls, const int32_t* sizes, const int32_t* lengths,
                                  const int32_t* prompt, const double* k_up, const double* k_dn,
                                  const double* deadline, const double* waiting, const double* co,
                                  int64_t padded, int has_tau, double tau_min, int32_t* res) {
  __shared__ LevelInfo row[EB_MAX_CLASSES];
  __shared__ double up[EB_MAX_K + EB_MAX_CLASSES], dn[EB_MAX_K + EB_MAX_CLASSES],
      tau[EB_MAX_K + EB_MAX_CLASSES], w[EB_MAX_CLASSES];
  __shared__ int32_t len[EB_MAX_CLASSES];
  if (threadIdx.x != 0) return;
  const double k2 = co[0], k3 = co[1], k4 = co[2], k5 = co[3], sb = co[4];
  const double slots = co[5], Cf = co[6], beta = co[7];
  int off = 0, m = 0, tail0 = 0;
  for (int k = 0; k < ncls; ++k) tail0 += sizes[k];
  int tail = tail0;
  for (int k = 0; k < ncls; ++k) {
    int sz = sizes[k];
    tail -= sz;
    row[k].off = (uint16_t)off; row[k].size = (uint8_t)sz; row[k].tail_next = (uint8_t)tail;
    row[k].g = (uint8_t)k; row[k].pad[0] = row[k].pad[1] = row[k].pad[2] = 0;
    len[k] = lengths[k];
    double fn = i2d(lengths[k]);
    w[k] = add(mul(k4, fn), mul(mul(k5, fn), fn));              // latency_weight
    double cu = 0.0, cd = 0.0, tm = __longlong_as_double(0x7ff0000000000000LL);
    up[off] = cu; dn[off] = cd; tau[off] = tm;
    for (int q = 0; q < sz; ++q, ++m) {
      cu = add(cu, mul(k_up[m], i2d(prompt[m])));             // cu[-1] + k_up * s     (dftsp.py:126)
      cd = add(cd, mul(k_dn[m], fn));                          // cd[-1] + k_down * n   (dftsp.py:127)
      double tb = div(mul(sub(sub(deadline[m], waiting[m]), slots), Cf), beta);  // tau_base :110-114
      tm = pymin(tm, tb);
      up[off + q + 1] = cu; dn[off + q + 1] = cd; tau[off + q + 1] = tm;
    }
    off += sz + 1;
  }
  Tables T;
  T.row = row; T.up = up; T.dn = dn; T.tau = tau; T.len = len; T.w = w;
  Lane s;
  s.k = 0; s.V0 = s.V1 = 0;
  const bool has_cap = sb == sb;   // NaN marks slot_cap_s None
  int r = dfs_begin<PRUNE, INCL, EXACT>(s, T, z, tail0, ncls, k3, has_cap ? sb : 0.0, has_cap,
                                        has_tau ? tau_min : 0.0, k2, padded);
  while (r == 0) r = dfs_step<PRUNE, INCL, EXACT>(s, T);
  res[0] = (r == 2);
  res[1] = (r == 2) ? s.k : -1;
  for (int k = 0; k < EB_MAX_CLASSES; ++k) res[2 + k] = (r == 2 && k < ncls && k <= s.k) ? getV(s.V0, s.V1, k) : 0;
  int64_t v = (int64_t)s.vis, p = (int64_t)s.prn;
  *(int64_t*)(res + 2 + EB_MAX_CLASSES) = v;
  *(int64_t*)(res + 2 + EB_MAX_CLASSES + 2) = p;
}

}  // namespace

// ---------------------------------------------------------------------------
// Host-side launcher (device pointers, caller's stream).
// ---------------------------------------------------------------------------
size_t dftsp_warp_bytes(int K, int G, bool exact) { return make_lay(K, G, exact, true).total; }

#ifdef EB_STATS
extern "C" int eb_debug_stats(unsigned long long* out, int reset) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, g_stats, sizeof(unsigned long long) * 16);
  if (reset) { unsigned long long z[16] = {0}; cudaMemcpyToSymbol(g_stats, z, sizeof(z)); }
  return 0;
}
#endif

static int launch_one(eb_handle* h, cudaStream_t st, void (*kern)(DftspArgs), const DftspArgs& A, int warps,
                      size_t smem, int64_t n_inst) {
  // occupancy per (kernel, block, smem), cached per thread (the host
  // pipeline launches every kernel once per chunk).  The dynamic shared
  // memory attribute is set on every launch: the block-width search of
  // launch_dftsp moves it too.
  struct Occ { void (*k)(DftspArgs); int warps; size_t smem; int per_sm; int dev; };
  static thread_local Occ occ[16];
  static thread_local int nocc = 0;
  EB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = -1;
  for (int i = 0; i < nocc && i < 16; ++i)
    if (occ[i].k == kern && occ[i].warps == warps && occ[i].smem == smem && occ[i].dev == h->device) {
      per_sm = occ[i].per_sm;
      break;
    }
  if (per_sm < 0) {
    EB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * warps, smem));
    occ[nocc % 16] = Occ{kern, warps, smem, per_sm, h->device};
    ++nocc;
  }
  if (per_sm < 1) per_sm = 1;
  int64_t want = (n_inst + warps - 1) / warps;
  int64_t grid = (int64_t)per_sm * h->num_sms;
  if (grid > want) grid = want;
  kern<<<(unsigned)grid, 32 * warps, smem, st>>>(A);
  EB_CUDA(cudaGetLastError());
  h->launches += 1;
  return EB_OK;
}

// Second pass over instances wider than EB_MAX_K (see dftsp_wide_kernel).
static int launch_wide(eb_handle* h, cudaStream_t st, const DftspArgs& A0, int K_all, int64_t n_wide,
                       int fallback_only = 0) {
  DftspArgs W = A0;
  const int Kw = K_all < EB_MAX_K_DFTSP ? K_all : EB_MAX_K_DFTSP;
  W.K = Kw;
  W.G = A0.prm.ladder_len > 0 ? A0.prm.ladder_len : (Kw < EB_MAX_CLASSES ? Kw : EB_MAX_CLASSES);
  W.fallback_pass = fallback_only;
  W.inst_list = nullptr;
  W.list_count = nullptr;
  const bool exact = A0.prm.exact_tau != 0;
  W.lay = make_lay(Kw, W.G, exact, false);
  W.warp_bytes = al8(W.lay.total);
  const size_t smem_cap = 227 * 1024;
  const bool in_smem = W.warp_bytes <= smem_cap;
  int64_t grid = n_wide > 0 ? n_wide : W.n_inst;
  if (grid > 4 * (int64_t)h->num_sms) grid = 4 * (int64_t)h->num_sms;
  if (grid < 1) grid = 1;
  void (*kern)(DftspArgs, unsigned char*);
  const bool P = W.prm.pruning != 0, I = W.prm.inclusive_bound != 0;
  if (P) {
    if (I) kern = exact ? dftsp_wide_kernel<true, true, true> : dftsp_wide_kernel<true, true, false>;
    else kern = exact ? dftsp_wide_kernel<true, false, true> : dftsp_wide_kernel<true, false, false>;
  } else {
    if (I) kern = exact ? dftsp_wide_kernel<false, true, true> : dftsp_wide_kernel<false, true, false>;
    else kern = exact ? dftsp_wide_kernel<false, false, true> : dftsp_wide_kernel<false, false, false>;
  }
  unsigned char* scratch = nullptr;
  size_t smem = 0;
  if (in_smem) {
    smem = W.warp_bytes;
    EB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  } else {
    EB_CUDA(cudaMallocAsync((void**)&scratch, (size_t)grid * W.warp_bytes, st));
  }
  EB_CUDA(cudaMemsetAsync(W.counter, 0, sizeof(int), st));
  kern<<<(unsigned)grid, 32, smem, st>>>(W, scratch);
  EB_CUDA(cudaGetLastError());
  h->launches += 1;
  if (scratch) EB_CUDA(cudaFreeAsync(scratch, st));
  return EB_OK;
}

// Instances wider than EB_MAX_K: the leaf-parallel search when every
// partition has at most three levels (ladder of <= 3 lengths) and the O(K)
// per-warp footprint fits; the literal walk otherwise, and for any instance
// whose u32 count rows overflow.
static int launch_wide_v2(eb_handle* h, cudaStream_t st, const DftspArgs& A0, int K_all, int64_t n_wide) {
  const int Kw = K_all < EB_MAX_K_DFTSP ? K_all : EB_MAX_K_DFTSP;
  const int G = A0.prm.ladder_len > 0 ? A0.prm.ladder_len : (Kw < EB_MAX_CLASSES ? Kw : EB_MAX_CLASSES);
  const bool exact = A0.prm.exact_tau != 0;
  const size_t smem_cap = 227 * 1024;
  const Lay lay = make_lay(Kw, G, exact, true);
  if (G > 3 || al8(lay.total) > smem_cap || A0.prm.collect_trajectory) return launch_wide(h, st, A0, K_all, n_wide);
  DftspArgs W = A0;
  W.K = Kw;
  W.G = G;
  W.lay = lay;
  W.warp_bytes = al8(lay.total);
  W.fallback_pass = 0;
  int* buf = nullptr;                                // [0] queue, [1] fallback count, [2] list count, list
  EB_CUDA(cudaMallocAsync((void**)&buf, sizeof(int) * (4 + (size_t)W.n_inst), st));
  EB_CUDA(cudaMemsetAsync(buf, 0, 4 * sizeof(int), st));
  {
    int blocks = (int)((W.n_inst + 255) / 256);
    if (blocks > 4 * h->num_sms) blocks = 4 * h->num_sms;
    if (blocks < 1) blocks = 1;
    wide_list_kernel<<<blocks, 256, 0, st>>>(W.n_inst, W.offsets, buf + 4, buf + 2);
    EB_CUDA(cudaGetLastError());
    h->launches += 1;
  }
  W.counter = buf;
  W.inst_list = buf + 4;
  W.list_count = buf + 2;
  void (*kern)(DftspArgs);
  const bool P = W.prm.pruning != 0, I = W.prm.inclusive_bound != 0;
#define EB_PICKW(KN)                                                                                   \
  if (P) {                                                                                             \
    if (I) kern = exact ? KN<true, true, true> : KN<true, true, false>;                                \
    else kern = exact ? KN<true, false, true> : KN<true, false, false>;                                \
  } else {                                                                                             \
    if (I) kern = exact ? KN<false, true, true> : KN<false, true, false>;                              \
    else kern = exact ? KN<false, false, true> : KN<false, false, false>;                              \
  }
  const bool ni4 = Kw <= 128;
  if (ni4) { EB_PICKW(dftsp_lock_wide4_kernel) } else { EB_PICKW(dftsp_lock_wide_kernel) }
#undef EB_PICKW
  int warps = (int)(smem_cap / W.warp_bytes);
  const int wmax = ni4 ? EB_WIDE4_THREADS / 32 : 2;
  if (warps > wmax) warps = wmax;
  const int64_t n_launch = n_wide > 0 ? n_wide : W.n_inst;        // grid bound only
  int rc = launch_one(h, st, kern, W, warps, W.warp_bytes * warps, n_launch);
  if (rc) return rc;
  // literal walk for instances whose count rows overflowed (status flagged)
  DftspArgs F = A0;
  F.counter = buf;
  EB_CUDA(cudaMemsetAsync(buf, 0, sizeof(int), st));
  rc = launch_wide(h, st, F, K_all, n_wide, 1);
  if (rc) return rc;
  EB_CUDA(cudaFreeAsync(buf, st));
  return EB_OK;
}

int launch_dftsp(eb_handle* h, cudaStream_t st, const eb_context* d_ctxs, int n_ctx,
                 const eb_search_params& prm, int64_t n_inst, const int64_t* d_off,
                 const int32_t* d_ctx_index, int64_t req_base, const eb_requests& d_req,
                 int K, const eb_dftsp_result& d_out, int64_t traj_base, int* d_counter, int64_t n_wide) {
  if (n_inst <= 0) return EB_OK;
  const int K_all = K;                // widest instance: a wide pass follows when > EB_MAX_K
  if (K > EB_MAX_K) K = EB_MAX_K;
  int G = prm.ladder_len > 0 ? prm.ladder_len : (K < EB_MAX_CLASSES ? K : EB_MAX_CLASSES);
  if (G < 1) G = 1;
  const bool exact = prm.exact_tau != 0;
  DftspArgs A;
  A.ctxs = d_ctxs; A.n_ctx = n_ctx; A.prm = prm; A.n_inst = n_inst; A.offsets = d_off;
  A.ctx_index = d_ctx_index; A.req_base = req_base; A.req = d_req; A.K = K; A.G = G;
  A.out = d_out; A.traj_base = traj_base; A.counter = d_counter; A.fallback_pass = 0;
  A.ctab = nullptr;
  A.inst_list = nullptr;
  A.list_count = nullptr;
  // algorithm: 2 = leaf-parallel (default) unless its tables do not fit two
  // warps per block, 1 = literal lanes-per-call (also v2's in-kernel fallback)
  int algo = prm.algorithm;
  const size_t smem_cap = 227 * 1024;
  if (prm.exhaustive_counts) {
    // counts mode exists only in the leaf-parallel search
    if (prm.exact_tau || al8(make_lay(K, G, exact, true).total) > smem_cap) {
      set_error("exhaustive counts mode needs the leaf-parallel search (K=%d too large)", K);
      return EB_ERR_K_TOO_LARGE;
    }
    algo = 2;
  }
  if (algo != 1 && al8(make_lay(K, G, exact, true).total) * 2 > smem_cap) algo = 1;
  if (algo != 1) algo = 2;
  // Leaf-parallel kernels with the layout compiled in (FK = 100 K + G):
  // K <= 32 with the paper's three-class ladder (every flag set), and with
  // pruning on, K <= 20 with four or five classes (config 5) and K = 33..64
  // with three classes (config 3's wide end).
  const bool P = prm.pruning != 0, I = prm.inclusive_bound != 0;
  int fk = 0;
  if (algo == 2) {
    if (EB_FK2003 && P && !I && !exact && K <= 20 && G <= 3) fk = 2003;
    else if (K <= 32 && G <= 3) fk = 3203;
    else if (P && K <= 20 && G <= 5) fk = 2005;
    else if (P && K <= 64 && G <= 3) fk = 6403;
  }
  A.lay = fk ? make_lay(fk / 100, fk % 100, exact, true) : make_lay(K, G, exact, algo == 2);
  A.warp_bytes = al8(A.lay.total);
  int warps = (int)(smem_cap / A.warp_bytes);
  if (warps > 4) warps = 4;
  if (warps < 1) { set_error("instance size K=%d needs %zu B shared memory per warp", K, A.warp_bytes); return EB_ERR_K_TOO_LARGE; }
  size_t smem = A.warp_bytes * warps;
  void (*kern)(DftspArgs);
#define EB_PICK3(AL, NI)                                                                           \
  if (P) {                                                                                         \
    if (I) kern = exact ? dftsp_kernel<true, true, true, AL, NI> : dftsp_kernel<true, true, false, AL, NI>;   \
    else kern = exact ? dftsp_kernel<true, false, true, AL, NI> : dftsp_kernel<true, false, false, AL, NI>;   \
  } else {                                                                                         \
    if (I) kern = exact ? dftsp_kernel<false, true, true, AL, NI> : dftsp_kernel<false, true, false, AL, NI>; \
    else kern = exact ? dftsp_kernel<false, false, true, AL, NI> : dftsp_kernel<false, false, false, AL, NI>; \
  }
#define EB_PICK(AL) if (K <= 32) { EB_PICK3(AL, 1) } else { EB_PICK3(AL, 2) }
#define EB_PICKL3(NI, FK)                                                                              \
  if (P) {                                                                                             \
    if (I) kern = exact ? dftsp_lock_kernel<true, true, true, NI, FK> : dftsp_lock_kernel<true, true, false, NI, FK>;   \
    else kern = exact ? dftsp_lock_kernel<true, false, true, NI, FK> : dftsp_lock_kernel<true, false, false, NI, FK>;   \
  } else {                                                                                             \
    if (I) kern = exact ? dftsp_lock_kernel<false, true, true, NI, FK> : dftsp_lock_kernel<false, true, false, NI, FK>; \
    else kern = exact ? dftsp_lock_kernel<false, false, true, NI, FK> : dftsp_lock_kernel<false, false, false, NI, FK>; \
  }
  if (algo == 2) {
    // Lockstep blocks (one instance per warp, phases shared by the block).
    // Block width: the most resident warps per SM for this kernel's
    // registers and this instance size's shared memory (occupancy API,
    // cached per kernel and per-warp footprint), preferring wider blocks
    // (measured at K=20: 4 -> 44.4, 8 -> 51.6, 16 -> 50.4 M inst/s).  Wide
    // instances (K = 21..64) thus get e.g. two 5-warp blocks instead of one
    // 8-warp block.  EB_LOCK_WARPS caps the width (tuning).
    int cap_w = 8;
    if (const char* e = getenv("EB_LOCK_WARPS")) { int v = atoi(e); if (v >= 1 && v <= 16) cap_w = v; }
#define EB_PICKLP(NI, FK)                                                                              \
  kern = I ? (exact ? dftsp_lock_kernel<true, true, true, NI, FK> : dftsp_lock_kernel<true, true, false, NI, FK>)    \
           : (exact ? dftsp_lock_kernel<true, false, true, NI, FK> : dftsp_lock_kernel<true, false, false, NI, FK>);
    if (fk == 2003) { kern = dftsp_lock_kernel<true, false, false, 1, 2003>; }
    else if (fk == 3203) { EB_PICKL3(1, 3203) }
    else if (fk == 2005) { EB_PICKLP(1, 2005) }
    else if (fk == 6403) { EB_PICKLP(2, 6403) }
    else if (K <= 32) { EB_PICKL3(1, 0) } else { EB_PICKL3(2, 0) }
#undef EB_PICKLP

    {
      struct WCache { void (*k)(DftspArgs); size_t wb; int cap; int dev; int w; };
      static thread_local WCache wc[8];
      static thread_local int nwc = 0;
      int best_w = -1;
      for (int i = 0; i < nwc && i < 8; ++i)
        if (wc[i].k == kern && wc[i].wb == A.warp_bytes && wc[i].cap == cap_w && wc[i].dev == h->device) {
          best_w = wc[i].w;
          break;
        }
      if (best_w < 0) {
        int best_res = 0;
        best_w = 1;
        cudaFuncAttributes fa;                 // never wider than the launch bounds allow
        EB_CUDA(cudaFuncGetAttributes(&fa, kern));
        const int wlim = cap_w < fa.maxThreadsPerBlock / 32 ? cap_w : fa.maxThreadsPerBlock / 32;
        for (int w = 1; w <= wlim; ++w) {
          const size_t sm = A.warp_bytes * w;
          if (sm > smem_cap) break;
          if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) != cudaSuccess) {
            cudaGetLastError();                 // beyond this kernel's limit: stop widening
            break;
          }
          int blocks = 0;
          EB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, kern, 32 * w, sm));
          const int res = blocks * w;
          if (res >= best_res) { best_res = res; best_w = w; }
        }
        wc[nwc % 8] = WCache{kern, A.warp_bytes, cap_w, h->device, best_w};
        ++nwc;
      }
      warps = best_w;
    }
    smem = A.warp_bytes * warps;
  } else {
    EB_PICK(1)
  }
#undef EB_PICKL3
  A.fallback_pass = 0;
  if (algo == 2 && K <= EB_MAX_K && !prm.exhaustive_counts) {
    const int v = !P ? 0 : (I ? 2 : 1);
    if (!h->ctab[v]) {
      // built once per handle and flag variant; synchronous, so kernels on
      // the other pipeline streams never see a partial table
      void* t = nullptr;
      EB_CUDA(cudaMalloc(&t, CT_HDR_BYTES + (size_t)CT_ROWS * CT * sizeof(uint2)));
      uint32_t hdr[CT_HDR];
      ct_header(hdr);
      for (int s0 = 1; s0 <= 62; ++s0)                 // the device uses the closed form
        for (int s1 = 1; s0 + s1 <= 63; ++s1)
          if (ct_row(hdr, 3, s0, s1, 1) != ct_row_closed(3, s0, s1, 1)) {
            set_error("count table numbering mismatch");
            return EB_ERR_CUDA;
          }
      EB_CUDA(cudaMemcpyAsync(t, hdr, sizeof(hdr), cudaMemcpyHostToDevice, st));
      EB_CUDA(cudaMemsetAsync((unsigned char*)t + CT_MPTR_OFF, 0, 8, st));
      void (*bk)(const uint32_t*, uint2*) = !P ? count_table_kernel<false, false>
                                               : (I ? count_table_kernel<true, true> : count_table_kernel<true, false>);
      const int nthr = 64 * 64 * 64 + 64 * 64 + 64;
      bk<<<(nthr + 255) / 256, 256, 0, st>>>((const uint32_t*)t, (uint2*)((unsigned char*)t + CT_HDR_BYTES));
      EB_CUDA(cudaGetLastError());
      h->launches += 1;
      EB_CUDA(cudaStreamSynchronize(st));
      h->ctab[v] = t;
    }
    A.ctab = (const uint2*)h->ctab[v];
    if (G >= 4) {
      if (!h->ctab_m[v]) {
        void* t = nullptr;
        EB_CUDA(cudaMalloc(&t, (size_t)CTM_ROWS * CTM * sizeof(uint2)));
        void (*bk)(uint2*) = !P ? count_table_m_kernel<false, false>
                                : (I ? count_table_m_kernel<true, true> : count_table_m_kernel<true, false>);
        const int64_t nthr = 32LL * 32 * 32 * 32 * 33;
        bk<<<(unsigned)((nthr + 255) / 256), 256, 0, st>>>((uint2*)t);
        EB_CUDA(cudaGetLastError());
        h->launches += 1;
        EB_CUDA(cudaStreamSynchronize(st));
        h->ctab_m[v] = t;
        EB_CUDA(cudaMemcpy((unsigned char*)h->ctab[v] + CT_MPTR_OFF, &h->ctab_m[v], 8, cudaMemcpyHostToDevice));
      }
    }
  }
  EB_CUDA(cudaMemsetAsync(d_counter, 0, 2 * sizeof(int), st));
  int rc = launch_one(h, st, kern, A, warps, smem, n_inst);
  if (rc) return rc;
  if (algo == 2) {
  // literal-walk pass for any instance whose leaf counts overflowed u32
  DftspArgs B = A;
  B.fallback_pass = 1;
  B.lay = make_lay(K, G, exact, false);
  B.warp_bytes = al8(B.lay.total);
  int wb = (int)(smem_cap / B.warp_bytes);
  if (wb > 4) wb = 4;
  EB_PICK(1)
  EB_CUDA(cudaMemsetAsync(d_counter, 0, sizeof(int), st));
  rc = launch_one(h, st, kern, B, wb, B.warp_bytes * wb, n_inst);
  if (rc) return rc;
  }
#undef EB_PICK
#undef EB_PICK3
  if (K_all > EB_MAX_K) {
    if (prm.exhaustive_counts) {
      set_error("exhaustive counts mode supports at most %d candidates", EB_MAX_K);
      return EB_ERR_K_TOO_LARGE;
    }
    return launch_wide_v2(h, st, A, K_all, n_wide);
  }
  return EB_OK;
}

int launch_dfs_single(eb_handle* h, cudaStream_t st, int z, int ncls, const int32_t* sizes,
                      const int32_t* lengths, const int32_t* prompt, const double* ku, const double* kd,
                      const double* dl, const double* wt, const double* co, int64_t padded, int has_tau,
                      double tau_min, const eb_search_params& prm, int32_t* res) {
  void (*kern)(int, int, const int32_t*, const int32_t*, const int32_t*, const double*, const double*,
               const double*, const double*, const double*, int64_t, int, double, int32_t*);
  const bool P = prm.pruning != 0, I = prm.inclusive_bound != 0, E = prm.exact_tau != 0;
  if (P) {
    if (I) kern = E ? dfs_single_kernel<true, true, true> : dfs_single_kernel<true, true, false>;
    else kern = E ? dfs_single_kernel<true, false, true> : dfs_single_kernel<true, false, false>;
  } else {
    if (I) kern = E ? dfs_single_kernel<false, true, true> : dfs_single_kernel<false, true, false>;
    else kern = E ? dfs_single_kernel<false, false, true> : dfs_single_kernel<false, false, false>;
  }
  kern<<<1, 32, 0, st>>>(z, ncls, sizes, lengths, prompt, ku, kd, dl, wt, co, padded, has_tau, tau_min, res);
  EB_CUDA(cudaGetLastError());
  h->launches += 1;
  return EB_OK;
}

}  // namespace eb
