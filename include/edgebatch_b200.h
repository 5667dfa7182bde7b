/*
 * edgebatch_b200.h -- C ABI of the B200-native DFTSP / brute-force batch
 * scheduling solver (arXiv 2405.07140 reference, package `edgebatch`).
 *
 * Plain C: fixed-width integers, doubles and pointers only; no torch, no C++
 * types.  Every entry point returns an eb_status.  Nothing throws across the
 * ABI.  Per-instance failures (the reference's ValueError / RuntimeError
 * cases) are reported per instance in `status[]` so a batch never aborts.
 *
 * Each entry point replaces one reference interface; the reference citation
 * (path:line under /root/reference) is given beside it.  The Python shim in
 * paper_2405_07140_b200/ binds these with ctypes and re-raises the reference's
 * exception types and messages; INTEGRATION.md shows that binding.
 *
 * Memory: every batched call takes `mem` = EB_MEM_HOST (pointers are host
 * memory; the library stages through pinned buffers on its own stream,
 * overlapping copies with compute) or EB_MEM_DEVICE (pointers are device
 * memory on the handle's GPU; the call is asynchronous on `stream` unless
 * stated otherwise).
 */
#ifndef EDGEBATCH_B200_H
#define EDGEBATCH_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EB_ABI_VERSION 2   /* 2: wire format (eb_dftsp_batch_packed), solution masks */
#define EB_MAX_K 64          /* candidates per instance (u64 subset masks)   */
#define EB_MAX_K_DFTSP 255   /* dftsp instances: > EB_MAX_K take a wide pass   */
#define EB_MAX_CLASSES 16    /* output-length classes per instance           */
#define EB_N_METRICS 8       /* doubles per instance in eb_dftsp_result.metrics */

typedef enum eb_status {
  EB_OK = 0,
  EB_ERR_INVALID_ARG = 1,          /* null pointer, bad size, bad flag               */
  EB_ERR_CUDA = 2,                 /* CUDA runtime failure (eb_last_error())          */
  EB_ERR_K_TOO_LARGE = 3,          /* instance larger than the entry point's limit or the call's k_max */
  EB_ERR_TOO_MANY_CLASSES = 4,     /* more than EB_MAX_CLASSES distinct output lengths */
  EB_ERR_NO_DEVICE = 5,
  /* Reference exceptions, per instance (status[] value; error_index[] names
   * the offending request by its local index within the instance):        */
  EB_ERR_WEIGHTS_DO_NOT_FIT = 10,  /* WeightsDoNotFitError  feasibility.py:145-150  */
  EB_ERR_UPLINK_EFF_ZERO = 11,     /* ValueError            radio.py:74-75          */
  EB_ERR_DOWNLINK_EFF_ZERO = 12,   /* ValueError            radio.py:82-83          */
  EB_ERR_OFF_LADDER = 13,          /* ValueError            dftsp.py:63-70          */
  EB_ERR_REVERIFY = 14,            /* RuntimeError          dftsp.py:276-280        */
  EB_ERR_DUPLICATE_ID = 15,        /* ids must be unique within a pool (coefficients are keyed by id, feasibility.py:164-166) */
  EB_ERR_CAP_EXCEEDED = 16,        /* ValueError            dftsp.py:302-303        */
  EB_ERR_OVERFLOW = 17,            /* exact integer FLOP count would exceed int64    */
  EB_ERR_BAD_MODE = 18,            /* ValueError            dftsp.py:314-315        */
  EB_ERR_PADDED_TOO_SMALL = 19,    /* ValueError            feasibility.py:142-143  */
  EB_ERR_NONPOSITIVE_LINK = 20,    /* ValueError            radio.py:63-64 (power, gain or noise <= 0) */
  EB_ERR_NAN_INPUT = 21            /* dftsp only: a NaN deadline/waiting/gain/power; the reference then orders
                                      the pool by CPython's sort on unordered keys (not reproduced) */
} eb_status;

typedef enum eb_mem { EB_MEM_HOST = 0, EB_MEM_DEVICE = 1 } eb_mem;

/* One serving context: EdgeContext (feasibility.py:59-71) flattened, with the
 * model's PPL degradation under the profile (catalog.py:131-143).  All
 * 8-byte fields, so the layout has no padding. */
typedef struct eb_context {
  /* LlmSpec catalog.py:15-39 */
  int64_t layers, hidden_dim, head_count, head_dim, ffn_dim, bytes_per_param;
  /* QuantProfile catalog.py:42-66 (alpha scales memory, beta latency) */
  double alpha, beta, delta_ppl;
  /* RadioConfig radio.py:16-43 (SI units; dBm already converted) */
  double uplink_band_hz, downlink_band_hz, downlink_power_w, noise_density_w_hz;
  double uplink_slot_s, downlink_slot_s;
  int64_t bits_per_token;
  /* NodeCompute costs.py:18-36 (aggregate C and M) */
  double flops_per_s, memory_bytes;
  int64_t gpu_count;
  /* EdgeContext.slot_cap_s; has_slot_cap == 0 means None */
  int64_t has_slot_cap;
  double slot_cap_s;
} eb_context;

/* Requests as structure-of-arrays (Request feasibility.py:33-56 with
 * UserLink radio.py:46-57).  Entry j belongs to instance i iff
 * offsets[i] <= j < offsets[i+1].  `tolerance` may be NULL for calls that
 * do not use it (dftsp, exhaustive, check_direct). */
typedef struct eb_requests {
  const int64_t *id;
  const int32_t *prompt_tokens;
  const int32_t *output_tokens;
  const double *deadline_s;
  const double *waiting_s;
  const double *tolerance;
  const double *channel_gain;
  const double *uplink_power_w;
} eb_requests;

/* A batch of independent scheduling instances (one `dftsp(candidates, ctx)`
 * call each).  `k_max` bounds offsets[i+1]-offsets[i]; it sizes shared
 * memory (EB_MEM_DEVICE callers must supply it; EB_MEM_HOST computes it if 0). */
typedef struct eb_batch {
  int64_t n_inst;
  int64_t n_req;              /* == offsets[n_inst] */
  const int64_t *offsets;     /* n_inst + 1 */
  const int32_t *ctx_index;   /* n_inst, or NULL = context 0 for all */
  eb_requests req;
  int32_t k_max;
  int32_t _pad;
} eb_batch;

/* dftsp() keyword arguments, dftsp.py:237-239. */
typedef struct eb_search_params {
  int32_t pruning;            /* default 1 */
  int32_t inclusive_bound;    /* default 0 */
  int32_t exact_tau;          /* default 0 */
  int32_t collect_trajectory; /* default 0 */
  int32_t ladder_len;         /* 0 = ladder None */
  int32_t ladder[EB_MAX_CLASSES];
  /* Device algorithm (results are identical): 0 = auto (leaf-parallel when
   * its tables fit), 1 = one dfs call per lane (literal node walk),
   * 2 = leaf-parallel enumeration with combinatorial node counts. */
  int32_t algorithm;
  /* 1 = run exhaustive_optimal(mode="counts") (dftsp.py:316-332) instead of
   * dftsp: same count-vector sequence, check_knapsack per vector, nodes =
   * vectors tried (nodes_pruned = 0, counts not reported). */
  int32_t exhaustive_counts;
} eb_search_params;

/* Indices into eb_dftsp_result.metrics[i*EB_N_METRICS + m]. */
enum {
  EB_MET_UP_SUM = 0,          /* sum rho_up of the batch, check_direct order (feasibility.py:203-205) */
  EB_MET_DN_SUM = 1,          /* sum rho_dn */
  EB_MET_MEM_POOLPAD = 2,     /* alpha * memory bytes at the pool's padded length (what the search checked) */
  EB_MET_LAT_POOLPAD = 3,     /* compute seconds at the pool's padded length */
  EB_MET_MEM_BATCHPAD = 4,    /* batch_cost memory at the batch's own padding (sim.py:372-376) */
  EB_MET_LAT_BATCHPAD = 5,    /* batch_cost latency at the batch's own padding */
  EB_MET_PADDED = 6,          /* pool padded length (dftsp.py:255) */
  EB_MET_WIN_D = 7            /* pool width d of the winning search (0 if none) */
};

/* Output of eb_dftsp_batch; SearchOutcome dftsp.py:42-51.  All arrays are
 * caller-allocated in the call's memory space.  Optional arrays may be NULL. */
typedef struct eb_dftsp_result {
  int32_t *status;           /* n_inst: eb_status                               */
  int32_t *error_index;      /* n_inst: offending local request index or -1     */
  int32_t *z_found;          /* n_inst                                          */
  int64_t *nodes_visited;    /* n_inst                                          */
  int64_t *nodes_pruned;     /* n_inst                                          */
  int32_t *n_classes;        /* n_inst: len(counts) = classes of the winning partition */
  int32_t *counts;           /* n_inst * EB_MAX_CLASSES                          */
  int32_t *class_lengths;    /* n_inst * EB_MAX_CLASSES: output length of each counted class */
  int32_t *solution;         /* n_req: at offsets[i], z_found local indices sorted by request id */
  double *metrics;           /* optional: n_inst * EB_N_METRICS                  */
  /* Optional trajectory (collect_trajectory): rows of (z, d, visited, pruned)
   * per dfs call; instance i owns rows [traj_offsets[i], traj_offsets[i+1]),
   * which must hold K*(K+1)/2 rows for K = its size. */
  const int64_t *traj_offsets; /* n_inst + 1 */
  int64_t *traj;             /* rows * 4 */
  int32_t *traj_len;         /* n_inst */
  /* Optional: n_inst selection masks, bit j = local request j scheduled
   * (instances of at most 64 requests; 0 for wider ones).  With ids that
   * rise along the rows the mask's bit order is the solution's id order, so
   * a caller can take it instead of `solution` (8 B per instance instead of
   * 4 B per request). */
  uint64_t *solution_mask;
} eb_dftsp_result;

typedef struct eb_handle eb_handle;

/* ---- library / handle ------------------------------------------------- */
int32_t eb_abi_version(void);
const char *eb_status_string(int32_t status);
const char *eb_last_error(void);                 /* thread-local detail string */
/* Per-thread handle: device, stream, pinned staging and scratch.  No global
 * mutable state outside handles. */
int32_t eb_handle_create(int32_t device, eb_handle **out);
int32_t eb_handle_destroy(eb_handle *h);
/* Stream the handle launches on (cudaStream_t as void*); may be replaced. */
int32_t eb_handle_set_stream(eb_handle *h, void *stream);
int32_t eb_synchronize(eb_handle *h);
/* Kernels launched by this handle since creation (evidence counter). */
int64_t eb_kernel_launches(eb_handle *h);
/* Live roofline denominators (bench.py): FP64 add rate (DADD/s over every SM)
 * and warp-instruction issue rate (independent IMAD + LOP3 chains) measured on
 * the handle's GPU at its current clocks.  No reference counterpart. */
int32_t eb_probe_peaks(eb_handle *h, double *fp64_ops_per_s, double *warp_inst_per_s);

/* ---- K3: instance-parallel DFTSP -------------------------------------
 * Replaces dftsp() dftsp.py:237-285 (with derive_coefficients
 * feasibility.py:133-167, partition dftsp.py:54-82, SearchTables.build
 * dftsp.py:110-132, dfs dftsp.py:135-234 and the check_direct
 * re-verification dftsp.py:276-280) for n_inst independent instances.
 * Bit-exact: solution ids, counts, z_found, nodes_visited, nodes_pruned. */
int32_t eb_dftsp_batch(eb_handle *h, const eb_context *ctxs, int32_t n_ctx,
                       const eb_search_params *params, const eb_batch *batch,
                       eb_dftsp_result *out, int32_t mem);

/* ---- K3 over the compact wire format ------------------------------------
 * Same search and results as eb_dftsp_batch (dftsp.py:237-285), for host
 * callers whose request columns fit narrower types.  Fewer bytes cross
 * PCIe per request: 4 (id, or none) + 2 + 2 (tokens, or one dictionary
 * byte) + 3 x 8 (deadline, waiting, gain), plus 8 for uplink power unless it
 * is uniform.  That is 25-32 B instead of eb_requests' 48 B.  Each chunk is copied in this layout and widened on
 * the device by a copy kernel into eb_requests columns, so the search
 * reads exactly the values the wide call would.  Every narrowing is
 * lossless: Request.id (feasibility.py:35) and the token counts
 * (feasibility.py:36-37) are Python ints.  The caller checks they fit
 * (paper_2405_07140_b200/soa.py pack_wire does). */
typedef struct eb_requests_packed {
  /* NULL: ids are the request positions (row indices).  The search only
   * compares ids within an instance (tie-breaks dftsp.py:78,257; the
   * duplicate check; the solution's id order dftsp.py:281), so any
   * increasing numbering of an instance's rows gives identical results;
   * this is how Monte Carlo instances number their candidates. */
  const int32_t *id;
  const uint16_t *prompt_tokens;
  const uint16_t *output_tokens;
  const double *deadline_s;
  const double *waiting_s;
  const double *channel_gain;
  const double *uplink_power_w;   /* n_req values, or 1 if uplink_power_uniform */
  int32_t uplink_power_uniform;   /* 1: every request has uplink_power_w[0]     */
  /* Dictionary-coded token counts (when token_codes != NULL the two token
   * columns are not read): code = prompt index | output index << 4 into the
   * two value tables (at most 16 distinct values each), one byte per
   * request instead of four. */
  int32_t n_dict;                 /* 0, or the table length (<= 16) */
  const uint8_t *token_codes;
  int32_t prompt_dict[16];
  int32_t output_dict[16];
} eb_requests_packed;

typedef struct eb_batch_packed {
  int64_t n_inst;
  int64_t n_req;              /* == offsets[n_inst] */
  const int64_t *offsets;     /* n_inst + 1, or NULL: every instance has k_max requests */
  const int32_t *ctx_index;   /* n_inst, or NULL = context 0 for all */
  eb_requests_packed req;
  int32_t k_max;              /* required: max offsets[i+1]-offsets[i] (<= EB_MAX_K) */
  int32_t _pad;
} eb_batch_packed;

/* Host memory only (mem must be EB_MEM_HOST): the wire format exists to cut
 * host->device bytes.  Device-resident callers use eb_dftsp_batch. */
int32_t eb_dftsp_batch_packed(eb_handle *h, const eb_context *ctxs, int32_t n_ctx,
                              const eb_search_params *params, const eb_batch_packed *batch,
                              eb_dftsp_result *out, int32_t mem);

/* ---- K3': one dfs() call on a prepared partition ----------------------
 * Replaces dfs(z, part, coeff, tau_min, ...) dftsp.py:135-234.  The
 * partition (ClassPartition dftsp.py:29-39) is given class-major: n_cls
 * classes with sizes[c] members and output length lengths[c]; per member,
 * in within-class order: prompt, k_up, k_down (KnapsackCoefficients
 * values), deadline_s, waiting_s.  coeff[8] = {k2, k3, k4, k5,
 * slot_base (slot_cap*C/beta, NaN when slot_cap_s is None),
 * uplink_slot+downlink_slot, C, beta}.  has_tau_min = 0 means None
 * (exact_tau only).  Builds SearchTables (dftsp.py:110-132) on the device.
 * Host memory, synchronous.  out_counts receives n_cls entries. */
int32_t eb_dfs_single(eb_handle *h, int32_t z, int32_t n_cls, const int32_t *sizes,
                      const int32_t *lengths, const int32_t *prompt, const double *k_up,
                      const double *k_down, const double *deadline_s,
                      const double *waiting_s, const double coeff[8], int64_t padded_len,
                      int32_t has_tau_min, double tau_min,
                      const eb_search_params *params, int32_t *out_found,
                      int32_t *out_counts, int64_t *out_visited, int64_t *out_pruned);

/* ---- K4: brute-force subset enumeration --------------------------------
 * Replaces exhaustive_optimal(mode="subsets") dftsp.py:288-313: per
 * instance, the largest z with a feasible subset and the lexicographically
 * first such subset in itertools.combinations order (pool order).  Outputs
 * z, its lexicographic rank within C(K,z), the subset (local indices, pool
 * order) and nodes_visited = sum_{z'>z} C(K,z') + lexrank + 1 (2^K - 1 if
 * none, 0 if empty).  `cap`: pools larger than cap get EB_ERR_CAP_EXCEEDED. */
int32_t eb_exhaustive_batch(eb_handle *h, const eb_context *ctxs, int32_t n_ctx,
                            const eb_batch *batch, int32_t cap,
                            int32_t *status, int32_t *z_found, int64_t *lexrank,
                            int64_t *nodes_visited, uint64_t *subset_mask,
                            int32_t mem);

/* Shardable level search for one instance (host memory, synchronous): the
 * smallest lexicographic rank r in [rank_lo, rank_hi) of a size-z subset
 * that passes check_direct, or -1.  Used to split 2^K across GPUs by rank
 * range; ranks index itertools.combinations(pool, z) order. */
int32_t eb_exhaustive_level_range(eb_handle *h, const eb_context *ctx,
                                  int32_t k, const eb_requests *req, int32_t z,
                                  int64_t rank_lo, int64_t rank_hi,
                                  int64_t *first_rank);

/* Levels worth searching for one instance (host memory, synchronous): bit
 * z-1 of *live_mask is set unless the sound level bounds the range search
 * applies (minimum memory, compute time, uplink, downlink and deadline over
 * all size-z subsets) prove that no size-z subset passes check_direct.  A
 * sharded search can skip the clear levels: eb_exhaustive_level_range would
 * return -1 for them. */
int32_t eb_exhaustive_live_levels(eb_handle *h, const eb_context *ctx, int32_t k,
                                  const eb_requests *req, uint64_t *live_mask);
/* Evidence counters of the brute-force kernels on this handle since its
 * creation: out[0] = combinations checked with the full check_direct,
 * out[1] = prefixes whose whole subtree the branch and bound skipped.
 * Synchronizes the handle's stream.  No reference counterpart. */
int32_t eb_exhaustive_counters(eb_handle *h, int64_t *out);

/* ---- K2: batched feasibility / cost ----------------------------------- */
/* check_direct(subset, ctx, padded_len) feasibility.py:192-223 for n_sub
 * subsets.  Subset s = request rows members[sub_off[s] .. sub_off[s+1]) of
 * `req` (summed in that order), evaluated under ctxs[sub_ctx[s]] (NULL = 0)
 * at padded_len[s].  out_ok[s] in {0,1}; out_metrics[s*4 + {0..3}] (optional)
 * = {up_sum, dn_sum, alpha*mem, compute_s}.  status[s] carries
 * EB_ERR_UPLINK_EFF_ZERO/... when a link math error would have raised. */
int32_t eb_check_direct_batch(eb_handle *h, const eb_context *ctxs, int32_t n_ctx,
                              const eb_requests *req, int64_t n_req_rows,
                              int64_t n_sub, const int64_t *sub_off,
                              const int32_t *members, const int32_t *sub_ctx,
                              const int64_t *padded_len, int32_t *status,
                              uint8_t *out_ok, double *out_metrics, int32_t mem);

/* check_knapsack(subset, coeff, z, tau_min) feasibility.py:170-189 for n_sub
 * subsets given their KnapsackCoefficients: member rows
 * [sub_off[s], sub_off[s+1]) carry (prompt, output, k_up, k_down) in subset
 * order; coeff[s*6 + {k2, k3, k4, k5, slot_base (NaN = no slot cap),
 * padded_len}]; z[s]; tau_min[s].  out_ok[s] in {0,1}. */
int32_t eb_check_knapsack_batch(eb_handle *h, int64_t n_sub, const int64_t *sub_off,
                                const int32_t *prompt, const int32_t *output,
                                const double *k_up, const double *k_down,
                                const double *coeff, const int32_t *z,
                                const double *tau_min, uint8_t *out_ok, int32_t mem);

/* K1: derive_coefficients feasibility.py:133-167 per instance at padded_len
 * (<=0 means pool max prompt): out_scalar[i*6 + {k2,k3,k4,k5,slot_base,padded}]
 * (slot_base = slot_cap*C/beta, NaN if None); per request row out_req[j*4 +
 * {k_up, k_down, tau_base, min_uplink_fraction}]. */
int32_t eb_coefficients_batch(eb_handle *h, const eb_context *ctxs, int32_t n_ctx,
                              const eb_batch *batch, const int64_t *padded_len,
                              int32_t *status, int32_t *error_index,
                              double *out_scalar, double *out_req, int32_t mem);

/* K1: per-request link math radio.py:64-101 under ctxs[req_ctx[j]]:
 * out[j*6 + {eta_up, eta_dn, k_up, k_down, rho_up_min, rho_dn_min}];
 * status[j] = EB_ERR_*_EFF_ZERO where the reference raises. */
int32_t eb_link_batch(eb_handle *h, const eb_context *ctxs, int32_t n_ctx,
                      const eb_requests *req, int64_t n_req, const int32_t *req_ctx,
                      int32_t *status, double *out, int32_t mem);

/* K1: the simulator's candidate filter sim.py:264-274: accuracy admission
 * catalog.py:146-155 (when accuracy_check) then check_direct((r,), ctx,
 * r.prompt_tokens) (when prefilter).  out_keep[j] in {0,1}. */
int32_t eb_admission_batch(eb_handle *h, const eb_context *ctxs, int32_t n_ctx,
                           const eb_batch *batch, int32_t accuracy_check,
                           int32_t prefilter, int32_t *status, uint8_t *out_keep,
                           int32_t mem);

/* batch_cost(spec, quant, plan, node, weight_copies) costs.py:131-148 for
 * n_plans plans: plan p = entries [plan_off[p], plan_off[p+1]) of
 * (prompt, output), padded_len[p], weight_copies[p] (NULL = 1), ctx
 * plan_ctx[p].  out[p*2 + {memory_bytes, latency_s}]. */
int32_t eb_batch_cost_batch(eb_handle *h, const eb_context *ctxs, int32_t n_ctx,
                            int64_t n_plans, const int64_t *plan_off,
                            const int32_t *prompt, const int32_t *output,
                            const int64_t *padded_len, const int64_t *weight_copies,
                            const int32_t *plan_ctx, double *out, int32_t mem);

/* ---- benchmark batching baselines (baselines.py) ------------------------ */
/* static_batch_size(spec, quant, node, slot_s, s_max, n_max) baselines.py:51-65
 * per context. */
int32_t eb_static_batch_size_batch(eb_handle *h, const eb_context *ctxs, int32_t n,
                                   const double *slot_s, const int64_t *s_max,
                                   const int64_t *n_max, int64_t *out_b, int32_t mem);

/* stb_schedule(queue, b, ctx, delta, accuracy_check) baselines.py:68-87 per
 * instance (queue = instance rows in order, delta = ctx.delta_ppl):
 * out_sel[j] = 1 if row j is scheduled. */
int32_t eb_stb_batch(eb_handle *h, const eb_context *ctxs, int32_t n_ctx,
                     const eb_batch *batch, const int64_t *b, int32_t accuracy_check,
                     int32_t *status, uint8_t *out_sel, int32_t mem);

/* nob_assign(queue, pool, now, ctx, delta, accuracy_check) baselines.py:90-121
 * per instance.  Device state busy_until[i*max_dev + g] (in/out) for
 * n_dev[i] devices (NULL = ctx gpu_count); per-device flops/memory =
 * flops_per_s/gpu_count and memory_bytes/gpu_count (NodeCompute per_gpu_*
 * costs.py:30-36, GpuPool.from_node baselines.py:37-39).  out_action[j]: 0 = not considered/skipped,
 * 1 = scheduled, 2 = dropped ("exceeds per-device memory");
 * out_completion[j] = completion time of scheduled rows; out_order[j] =
 * position in the scheduled list (-1 otherwise). */
int32_t eb_nob_batch(eb_handle *h, const eb_context *ctxs, int32_t n_ctx,
                     const eb_batch *batch, const double *now, int32_t accuracy_check,
                     const int32_t *n_dev, int32_t max_dev, double *busy_until, int32_t *status,
                     int8_t *out_action, double *out_completion, int32_t *out_order,
                     int32_t mem);

#ifdef __cplusplus
}
#endif
#endif /* EDGEBATCH_B200_H */
