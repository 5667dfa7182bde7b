// eb_capi.cu -- extern "C" entry points of include/edgebatch_b200.h.
//
// EB_MEM_DEVICE calls launch directly on the handle's stream.  EB_MEM_HOST
// calls stage through stream-ordered device allocations; eb_dftsp_batch
// splits large batches into instance chunks pipelined over three streams so
// host->device copies, the search kernel and device->host copies of
// neighbouring chunks overlap (pinned caller buffers give true overlap).
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <vector>

#include "eb_internal.cuh"

namespace eb {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
int cuda_fail(cudaError_t e, const char* what) {
  set_error("CUDA error %s (%s) at %s", cudaGetErrorName(e), cudaGetErrorString(e), what);
  return EB_ERR_CUDA;
}

// launchers defined in the kernel translation units
size_t dftsp_warp_bytes(int K, int G, bool exact);
int launch_dftsp(eb_handle*, cudaStream_t, const eb_context*, int, const eb_search_params&, int64_t,
                 const int64_t*, const int32_t*, int64_t, const eb_requests&, int, const eb_dftsp_result&,
                 int64_t, int*, int64_t);
int launch_dfs_single(eb_handle*, cudaStream_t, int, int, const int32_t*, const int32_t*, const int32_t*,
                      const double*, const double*, const double*, const double*, const double*, int64_t, int,
                      double, const eb_search_params&, int32_t*);
int binom_init(cudaStream_t);
int launch_exh_batch(eb_handle*, cudaStream_t, const eb_context*, int, int64_t, const int64_t*,
                     const int32_t*, int64_t, const eb_requests&, int, int32_t*, int32_t*, int64_t*,
                     int64_t*, uint64_t*);
int exh_range(eb_handle*, cudaStream_t, const eb_context&, const eb_requests&, int, int, int64_t, int64_t,
              unsigned long long*, int*, int64_t*, int*);
int exh_levels(eb_handle*, cudaStream_t, const eb_context&, const eb_requests&, int, unsigned long long*, int*,
               uint64_t*, int*);
int launch_link(eb_handle*, cudaStream_t, const eb_context*, int, const eb_requests&, int64_t,
                const int32_t*, int32_t*, double*);
int launch_coeff(eb_handle*, cudaStream_t, const eb_context*, int, int64_t, const int64_t*, const int32_t*,
                 int64_t, const eb_requests&, const int64_t*, int32_t*, int32_t*, double*, double*);
int launch_check_direct(eb_handle*, cudaStream_t, const eb_context*, int, const eb_requests&, int64_t,
                        const int64_t*, const int32_t*, const int32_t*, const int64_t*, int32_t*, uint8_t*,
                        double*);
int launch_check_knapsack(eb_handle*, cudaStream_t, int64_t, const int64_t*, const int32_t*, const int32_t*,
                          const double*, const double*, const double*, const int32_t*, const double*,
                          uint8_t*);
int launch_admission(eb_handle*, cudaStream_t, const eb_context*, int, int64_t, int64_t, const int64_t*,
                     const int32_t*, int64_t, const eb_requests&, int, int, int32_t*, uint8_t*);
int launch_batch_cost(eb_handle*, cudaStream_t, const eb_context*, int, int64_t, const int64_t*,
                      const int32_t*, const int32_t*, const int64_t*, const int64_t*, const int32_t*, double*);
int launch_static_b(eb_handle*, cudaStream_t, const eb_context*, int, const double*, const int64_t*,
                    const int64_t*, int64_t*);
int launch_stb(eb_handle*, cudaStream_t, const eb_context*, int, int64_t, const int64_t*, const int32_t*,
               int64_t, const eb_requests&, const int64_t*, int, int32_t*, uint8_t*);
int launch_nob(eb_handle*, cudaStream_t, const eb_context*, int, int64_t, const int64_t*, const int32_t*,
               int64_t, const eb_requests&, const double*, int, const int32_t*, int, double*, int32_t*, int8_t*,
               double*, int32_t*);

int ensure_dscratch(eb_handle* h, size_t bytes) {
  if (h->dscratch_bytes >= bytes) return EB_OK;
  if (h->dscratch) cudaFree(h->dscratch);
  h->dscratch = nullptr;
  h->dscratch_bytes = 0;
  EB_CUDA(cudaMalloc(&h->dscratch, bytes));
  h->dscratch_bytes = bytes;
  return EB_OK;
}
int ensure_pinned(eb_handle* h, size_t bytes) {
  if (h->pinned_bytes >= bytes) return EB_OK;
  if (h->pinned) cudaFreeHost(h->pinned);
  h->pinned = nullptr;
  h->pinned_bytes = 0;
  EB_CUDA(cudaMallocHost(&h->pinned, bytes));
  h->pinned_bytes = bytes;
  return EB_OK;
}

namespace {

// Collects stream-ordered device allocations of one host-memory call.
struct Stage {
  eb_handle* h;
  cudaStream_t st;
  std::vector<void*> bufs;
  int err = EB_OK;
  unsigned char* arena = nullptr;   // optional bump arena (no allocation calls per buffer)
  size_t cap = 0, used = 0;
  Stage(eb_handle* hh, cudaStream_t s) : h(hh), st(s) {}
  Stage(eb_handle* hh, cudaStream_t s, void* a, size_t bytes) : h(hh), st(s), arena((unsigned char*)a), cap(bytes) {}
  ~Stage() { for (void* p : bufs) cudaFreeAsync(p, st); }
  template <typename T>
  T* alloc(size_t count) {
    if (count == 0) count = 1;
    if (arena) {
      const size_t b = (count * sizeof(T) + 255) & ~(size_t)255;
      if (used + b <= cap) {
        T* q = (T*)(arena + used);
        used += b;
        return q;
      }
    }
    void* p = nullptr;
    cudaError_t e = cudaMallocAsync(&p, count * sizeof(T), st);
    if (e != cudaSuccess) { err = cuda_fail(e, "cudaMallocAsync"); return nullptr; }
    bufs.push_back(p);
    return (T*)p;
  }
  template <typename T>
  T* up(const T* host, size_t count) {
    if (!host) return nullptr;
    T* d = alloc<T>(count);
    if (!d) return nullptr;
    cudaError_t e = cudaMemcpyAsync(d, host, count * sizeof(T), cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) { err = cuda_fail(e, "H2D"); return nullptr; }
    return d;
  }
  template <typename T>
  T* out(const T* host, size_t count) { return host ? alloc<T>(count) : nullptr; }
  template <typename T>
  void down(T* host, const T* dev, size_t count) {
    if (!host || !dev || err) return;
    cudaError_t e = cudaMemcpyAsync(host, dev, count * sizeof(T), cudaMemcpyDeviceToHost, st);
    if (e != cudaSuccess) err = cuda_fail(e, "D2H");
  }
  int sync() {
    if (err) return err;
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "cudaStreamSynchronize");
    return EB_OK;
  }
};

eb_requests upload_req(Stage& S, const eb_requests& r, int64_t lo, int64_t n) {
  eb_requests d;
  d.id = r.id ? S.up(r.id + lo, n) : nullptr;
  d.prompt_tokens = S.up(r.prompt_tokens + lo, n);
  d.output_tokens = S.up(r.output_tokens + lo, n);
  d.deadline_s = r.deadline_s ? S.up(r.deadline_s + lo, n) : nullptr;
  d.waiting_s = r.waiting_s ? S.up(r.waiting_s + lo, n) : nullptr;
  d.tolerance = r.tolerance ? S.up(r.tolerance + lo, n) : nullptr;
  d.channel_gain = r.channel_gain ? S.up(r.channel_gain + lo, n) : nullptr;
  d.uplink_power_w = r.uplink_power_w ? S.up(r.uplink_power_w + lo, n) : nullptr;
  return d;
}

// Wire format -> eb_requests columns (lossless widening; uniform uplink
// power broadcast).  deadline/waiting/gain are already f64 and stay in place.
struct TokenDict { int32_t p[16], o[16]; };

__global__ void widen_wire_kernel(int64_t nr, int64_t row0, const int32_t* __restrict__ id32,
                                  const uint16_t* __restrict__ p16, const uint16_t* __restrict__ o16,
                                  const uint8_t* __restrict__ codes, const TokenDict dict,
                                  const double* __restrict__ pw, int uniform, int64_t* __restrict__ id64,
                                  int32_t* __restrict__ p32, int32_t* __restrict__ o32, double* __restrict__ pw64) {
  const double pw0 = uniform ? pw[0] : 0.0;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nr; j += (int64_t)gridDim.x * blockDim.x) {
    id64[j] = id32 ? (int64_t)id32[j] : row0 + j;      // NULL: ids are row positions
    if (codes) {
      const unsigned c = codes[j];
      p32[j] = dict.p[c & 15u];
      o32[j] = dict.o[c >> 4];
    } else {
      p32[j] = p16[j];
      o32[j] = o16[j];
    }
    pw64[j] = uniform ? pw0 : pw[j];
  }
}

// Uniform instance sizes: offsets of instances [i0, i0 + ni] are i * k.
__global__ void uniform_offsets_kernel(int64_t ni, int64_t i0, int k, int64_t* __restrict__ off) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= ni; i += (int64_t)gridDim.x * blockDim.x)
    off[i] = (i0 + i) * k;
}

// Upload policies of the DFTSP host pipeline: stage() issues the chunk's
// host->device copies on the upload stream (into the input arena); widen()
// runs on the chunk's compute stream once they have landed and returns the
// eb_requests columns the search reads.
struct WideUp {
  const eb_requests* r;
  static size_t row_bytes() { return 8 + 4 + 4 + 8 + 8 + 8 + 8 + 8; }
  eb_requests stage(Stage& S, int64_t lo, int64_t n) const { return upload_req(S, *r, lo, n); }
  eb_requests widen(Stage&, const eb_requests& d, int64_t, int64_t) const { return d; }
};

struct WireStaged {
  const int32_t* id32;
  const uint16_t *p16, *o16;
  const uint8_t* codes;
  const double *dl, *w, *g, *pw;
};

struct WireUp {
  const eb_requests_packed* r;
  static size_t row_bytes() { return 4 + 2 + 2 + 1 + 8 + 8 + 8 + 8; }
  WireStaged stage(Stage& S, int64_t lo, int64_t n) const {
    WireStaged d;
    d.id32 = r->id ? S.up(r->id + lo, n) : nullptr;
    if (r->token_codes) {
      d.codes = S.up(r->token_codes + lo, n);
      d.p16 = d.o16 = nullptr;
    } else {
      d.codes = nullptr;
      d.p16 = S.up(r->prompt_tokens + lo, n);
      d.o16 = S.up(r->output_tokens + lo, n);
    }
    d.dl = S.up(r->deadline_s + lo, n);
    d.w = S.up(r->waiting_s + lo, n);
    d.g = S.up(r->channel_gain + lo, n);
    d.pw = r->uplink_power_uniform ? S.up(r->uplink_power_w, 1) : S.up(r->uplink_power_w + lo, n);
    return d;
  }
  eb_requests widen(Stage& S, const WireStaged& d, int64_t lo, int64_t n) const {
    eb_requests q;
    memset(&q, 0, sizeof(q));
    int64_t* id64 = S.alloc<int64_t>(n);
    int32_t* p32 = S.alloc<int32_t>(n);
    int32_t* o32 = S.alloc<int32_t>(n);
    double* pw64 = S.alloc<double>(n);
    if (S.err) return q;
    int blocks = (int)((n + 255) / 256);
    if (blocks > 8 * S.h->num_sms) blocks = 8 * S.h->num_sms;
    if (blocks < 1) blocks = 1;
    TokenDict dict;
    for (int q = 0; q < 16; ++q) { dict.p[q] = r->prompt_dict[q]; dict.o[q] = r->output_dict[q]; }
    widen_wire_kernel<<<blocks, 256, 0, S.st>>>(n, lo, d.id32, d.p16, d.o16, d.codes, dict, d.pw,
                                                 r->uplink_power_uniform != 0, id64, p32, o32, pw64);
    ++S.h->launches;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { S.err = cuda_fail(e, "widen_wire_kernel"); return q; }
    q.id = id64;
    q.prompt_tokens = p32;
    q.output_tokens = o32;
    q.deadline_s = d.dl;
    q.waiting_s = d.w;
    q.channel_gain = d.g;
    q.uplink_power_w = pw64;
    return q;
  }
};

bool req_complete(const eb_requests& r, bool need_tol) {
  return r.id && r.prompt_tokens && r.output_tokens && r.deadline_s && r.waiting_s && r.channel_gain &&
         r.uplink_power_w && (!need_tol || r.tolerance);
}

// Host-memory DFTSP: instance chunks pipelined over an upload stream and the
// handle's three compute streams.  Every chunk's inputs get their own slice
// of the input arena, so the uploads run back to back on `up` (the PCIe
// bound) while chunk c computes on pipe[c % 3], waiting only for its own
// copies; outputs go back on the compute stream (the other copy direction).
// `upload` stages request rows [R0, R0+nr) (WideUp / WireUp).
template <typename Upload>
int dftsp_host_pipeline(eb_handle* h, const eb_context* ctxs, int n_ctx, const eb_search_params& prm, int64_t n,
                        const int64_t* offsets, const int32_t* ctx_index, int K, int64_t n_wide,
                        const eb_dftsp_result& out, const Upload& upload) {
  // offsets == NULL: every instance has K requests (wire format only)
  auto off_at = [&](int64_t i) -> int64_t { return offsets ? offsets[i] : i * (int64_t)K; };
  // Chunking: the first chunk's copy and the last chunk's search are the
  // exposed pipeline fill and drain, so chunk sizes ramp n/64, n/32, n/16,
  // ..., n/16, n/32, n/64.  Every chunk costs ~15 dependent copies and
  // launches (~0.2 ms of latency, measured by tools/host_overhead.py), so
  // chunks never go below 16384 instances (32768 in the middle).
  std::vector<int64_t> cut{0};
  {
    const int64_t full = (n + 15) / 16 > 32768 ? (n + 15) / 16 : 32768;
    const int64_t small = n / 64 > 16384 ? n / 64 : 16384;
    std::vector<int64_t> ramp;                       // n/64, n/32 (< full)
    for (int64_t s = small; s < full; s *= 2) ramp.push_back(s);
    int64_t head = 0;
    for (int64_t s : ramp) head += s;
    int64_t left = n;
    for (int64_t s : ramp) { if (left <= 0) break; cut.push_back(cut.back() + (s < left ? s : left)); left -= s; }
    // middle at `full`, keeping room for the mirrored ramp at the end
    while (left > head + full) { cut.push_back(cut.back() + full); left -= full; }
    if (left > head) { cut.push_back(cut.back() + (left - head)); left = head; }
    for (auto it = ramp.rbegin(); it != ramp.rend() && left > 0; ++it) {
      const int64_t s = *it < left ? *it : left;
      cut.push_back(cut.back() + s);
      left -= s;
    }
    if (cut.back() < n) cut.push_back(n);
  }
  const int nchunks = (int)cut.size() - 1;
  // The pipeline streams fork from / join back into the handle's stream so
  // events a caller records on that stream bracket the whole host->host call.
  EB_CUDA(cudaEventRecord(h->ev[0], h->stream));
  for (int i = 0; i < 3; ++i) EB_CUDA(cudaStreamWaitEvent(h->pipe[i], h->ev[0], 0));
  EB_CUDA(cudaStreamWaitEvent(h->up, h->ev[0], 0));
  // context table once per pipe stream (tiny)
  std::vector<Stage*> stages;
  int rc = EB_OK;
  // the context table once, through the pinned staging buffer (a pageable
  // copy would block the host), on pipe 0; the other pipes wait for it
  eb_context* d_ctx = nullptr;
  {
    const size_t cb = sizeof(eb_context) * (size_t)n_ctx;
    int e = ensure_pinned(h, cb);
    if (e) return e;
    memcpy(h->pinned, ctxs, cb);
    Stage* S0 = new Stage(h, h->pipe[0]);
    stages.push_back(S0);
    d_ctx = S0->up((const eb_context*)h->pinned, (size_t)n_ctx);
    if (S0->err) { rc = S0->err; }
    EB_CUDA(cudaEventRecord(h->ev[1], h->pipe[0]));
    EB_CUDA(cudaStreamWaitEvent(h->pipe[1], h->ev[1], 0));
    EB_CUDA(cudaStreamWaitEvent(h->pipe[2], h->ev[1], 0));
  }
  // one arena per pipeline stream, sized for its largest chunk: per instance
  // offsets, context index and outputs; per request the staged and widened
  // columns and the solution; per trajectory row 32 B; 256 B alignment slack
  // per buffer
  for (int c = 0; c < nchunks && rc == EB_OK; ++c) {
    const int64_t i0 = cut[c], i1 = cut[c + 1];
    size_t bytes = 48 * 256 + (size_t)(i1 - i0 + 1) * 320 + (size_t)(off_at(i1) - off_at(i0)) * 96;
    if (prm.collect_trajectory) bytes += (size_t)(out.traj_offsets[i1] - out.traj_offsets[i0]) * 32;
    const int sidx = c % 3;
    if (h->arena_bytes[sidx] < bytes) {
      if (h->arena[sidx]) cudaFreeAsync(h->arena[sidx], h->pipe[sidx]);
      h->arena[sidx] = nullptr;
      h->arena_bytes[sidx] = 0;
      cudaError_t e = cudaMallocAsync(&h->arena[sidx], bytes, h->pipe[sidx]);
      if (e != cudaSuccess) { rc = cuda_fail(e, "cudaMallocAsync(arena)"); break; }
      h->arena_bytes[sidx] = bytes;
    }
  }
  // input arena: every chunk's uploaded inputs (offsets, context index,
  // trajectory offsets, request columns), 256 B slack per buffer
  std::vector<size_t> in_off(nchunks + 1, 0);
  for (int c = 0; c < nchunks; ++c) {
    const int64_t i0 = cut[c], i1 = cut[c + 1];
    const size_t b = 16 * 256 + (size_t)(i1 - i0 + 1) * 20 + (size_t)(off_at(i1) - off_at(i0)) * Upload::row_bytes();
    in_off[c + 1] = in_off[c] + ((b + 255) & ~(size_t)255);     // slices stay 256 B aligned
  }
  if (rc == EB_OK && h->in_arena_bytes < in_off[nchunks]) {
    if (h->in_arena) cudaFreeAsync(h->in_arena, h->up);
    h->in_arena = nullptr;
    h->in_arena_bytes = 0;
    cudaError_t e = cudaMallocAsync(&h->in_arena, in_off[nchunks], h->up);
    if (e != cudaSuccess) rc = cuda_fail(e, "cudaMallocAsync(input arena)");
    else h->in_arena_bytes = in_off[nchunks];
  }
  for (int c = 0; c < nchunks && rc == EB_OK; ++c) {
    cudaStream_t st = h->pipe[c % 3];
    Stage* S = new Stage(h, st, h->arena[c % 3], h->arena_bytes[c % 3]);
    stages.push_back(S);
    Stage* U = new Stage(h, h->up, (unsigned char*)h->in_arena + in_off[c], in_off[c + 1] - in_off[c]);
    stages.push_back(U);
    const int64_t i0 = cut[c], i1 = cut[c + 1], ni = i1 - i0;
    const int64_t R0 = off_at(i0), R1 = off_at(i1), nr = R1 - R0;
    // uploads (stream `up`), then the compute stream waits for them
    const int64_t* d_off_up = offsets ? U->up(offsets + i0, (size_t)ni + 1) : nullptr;
    const int32_t* d_ci = ctx_index ? U->up(ctx_index + i0, (size_t)ni) : nullptr;
    const auto staged = upload.stage(*U, R0, nr);
    const int64_t* d_traj_off = prm.collect_trajectory ? U->up(out.traj_offsets + i0, (size_t)ni + 1) : nullptr;
    if (U->err) { rc = U->err; break; }
    {
      cudaEvent_t ev = h->cev[c % 64];
      cudaError_t e = cudaEventRecord(ev, h->up);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(st, ev, 0);
      if (e != cudaSuccess) { rc = cuda_fail(e, "chunk upload event"); break; }
    }
    const int64_t* d_off;
    if (offsets) {
      d_off = d_off_up;
    } else {
      int64_t* o = S->alloc<int64_t>((size_t)ni + 1);
      if (o) {
        int blocks = (int)((ni + 256) / 256);
        if (blocks > 4 * h->num_sms) blocks = 4 * h->num_sms;
        uniform_offsets_kernel<<<blocks, 256, 0, st>>>(ni, i0, K, o);
        ++h->launches;
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) S->err = cuda_fail(e, "uniform_offsets_kernel");
      }
      d_off = o;
    }
    eb_requests d_req = upload.widen(*S, staged, R0, nr);
    eb_dftsp_result d_out;
    memset(&d_out, 0, sizeof(d_out));
    d_out.status = S->alloc<int32_t>(ni);
    d_out.error_index = S->out(out.error_index, ni);
    d_out.z_found = S->alloc<int32_t>(ni);
    d_out.nodes_visited = S->alloc<int64_t>(ni);
    d_out.nodes_pruned = S->alloc<int64_t>(ni);
    d_out.n_classes = S->out(out.n_classes, ni);
    d_out.counts = S->out(out.counts, ni * EB_MAX_CLASSES);
    d_out.class_lengths = S->out(out.class_lengths, ni * EB_MAX_CLASSES);
    d_out.solution = S->out(out.solution, nr);
    d_out.metrics = S->out(out.metrics, ni * EB_N_METRICS);
    d_out.solution_mask = S->out(out.solution_mask, ni);
    int64_t T0 = 0;
    if (prm.collect_trajectory) {
      T0 = out.traj_offsets[i0];
      int64_t nt = out.traj_offsets[i1] - T0;
      d_out.traj_offsets = d_traj_off;
      d_out.traj = S->alloc<int64_t>((size_t)nt * 4);
      d_out.traj_len = S->out(out.traj_len, ni);
    }
    int* d_counter = S->alloc<int>(2);
    if (S->err) { rc = S->err; break; }
    rc = launch_dftsp(h, st, d_ctx, n_ctx, prm, ni, d_off, d_ci, R0, d_req, K, d_out, T0, d_counter, n_wide);
    if (rc) break;
    S->down(out.status + i0, d_out.status, ni);
    S->down(out.error_index ? out.error_index + i0 : nullptr, d_out.error_index, ni);
    S->down(out.z_found + i0, d_out.z_found, ni);
    S->down(out.nodes_visited + i0, d_out.nodes_visited, ni);
    S->down(out.nodes_pruned + i0, d_out.nodes_pruned, ni);
    S->down(out.n_classes ? out.n_classes + i0 : nullptr, d_out.n_classes, ni);
    S->down(out.counts ? out.counts + i0 * EB_MAX_CLASSES : nullptr, d_out.counts, ni * EB_MAX_CLASSES);
    S->down(out.class_lengths ? out.class_lengths + i0 * EB_MAX_CLASSES : nullptr, d_out.class_lengths,
            ni * EB_MAX_CLASSES);
    S->down(out.solution ? out.solution + R0 : nullptr, d_out.solution, nr);
    S->down(out.metrics ? out.metrics + i0 * EB_N_METRICS : nullptr, d_out.metrics, ni * EB_N_METRICS);
    S->down(out.solution_mask ? out.solution_mask + i0 : nullptr, d_out.solution_mask, ni);
    if (prm.collect_trajectory) {
      S->down(out.traj + 4 * T0, d_out.traj, (out.traj_offsets[i1] - T0) * 4);
      S->down(out.traj_len ? out.traj_len + i0 : nullptr, d_out.traj_len, ni);
    }
    if (S->err) { rc = S->err; break; }
  }
  for (Stage* S : stages) {
    int s2 = S->sync();
    if (!rc) rc = s2;
  }
  for (Stage* S : stages) delete S;   // stream-ordered frees
  // join the pipeline back into the handle's stream (every call checked:
  // the first failure is the one reported)
  auto keep = [&](cudaError_t e, const char* what) { if (e != cudaSuccess && rc == EB_OK) rc = cuda_fail(e, what); };
  for (int i = 0; i < 3; ++i) {
    keep(cudaEventRecord(h->ev[i], h->pipe[i]), "join: cudaEventRecord");
    keep(cudaStreamWaitEvent(h->stream, h->ev[i], 0), "join: cudaStreamWaitEvent");
  }
  keep(cudaEventRecord(h->cev[0], h->up), "join: cudaEventRecord(up)");
  keep(cudaStreamWaitEvent(h->stream, h->cev[0], 0), "join: cudaStreamWaitEvent(up)");
  for (int i = 0; i < 3; ++i) keep(cudaStreamSynchronize(h->pipe[i]), "join: cudaStreamSynchronize");
  keep(cudaStreamSynchronize(h->up), "join: cudaStreamSynchronize(up)");
  return rc;
}


}  // namespace
}  // namespace eb

using namespace eb;

extern "C" {

int32_t eb_abi_version(void) { return EB_ABI_VERSION; }

const char* eb_status_string(int32_t s) {
  switch (s) {
    case EB_OK: return "ok";
    case EB_ERR_INVALID_ARG: return "invalid argument";
    case EB_ERR_CUDA: return "CUDA error";
    case EB_ERR_K_TOO_LARGE: return "instance too large";
    case EB_ERR_TOO_MANY_CLASSES: return "too many output-length classes";
    case EB_ERR_NO_DEVICE: return "no CUDA device";
    case EB_ERR_WEIGHTS_DO_NOT_FIT: return "weights do not fit";
    case EB_ERR_UPLINK_EFF_ZERO: return "uplink spectral efficiency is zero";
    case EB_ERR_DOWNLINK_EFF_ZERO: return "downlink spectral efficiency is zero";
    case EB_ERR_OFF_LADDER: return "output length not on the class ladder";
    case EB_ERR_REVERIFY: return "reduced-form solution failed direct re-verification";
    case EB_ERR_DUPLICATE_ID: return "duplicate request id";
    case EB_ERR_CAP_EXCEEDED: return "pool size exceeds the exhaustive cap";
    case EB_ERR_OVERFLOW: return "integer cost model would overflow int64";
    case EB_ERR_BAD_MODE: return "unknown exhaustive mode";
    case EB_ERR_PADDED_TOO_SMALL: return "padded_len must cover every candidate prompt";
    case EB_ERR_NONPOSITIVE_LINK: return "power, gain and noise must be strictly positive";
    case EB_ERR_NAN_INPUT: return "NaN deadline, waiting time, gain or power: the reference's candidate order is undefined";
    default: return "unknown status";
  }
}

const char* eb_last_error(void) { return g_err; }

int32_t eb_handle_create(int32_t device, eb_handle** out) {
  if (!out) return EB_ERR_INVALID_ARG;
  *out = nullptr;
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0) {
    set_error("no CUDA device: %s", e == cudaSuccess ? "count 0" : cudaGetErrorString(e));
    return EB_ERR_NO_DEVICE;
  }
  if (device < 0 || device >= count) return EB_ERR_INVALID_ARG;
  EB_CUDA(cudaSetDevice(device));
  eb_handle* h = new eb_handle();
  memset(h, 0, sizeof(*h));
  h->device = device;
  EB_CUDA(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
  h->own_stream = true;
  for (int i = 0; i < 3; ++i) {
    EB_CUDA(cudaStreamCreateWithFlags(&h->pipe[i], cudaStreamNonBlocking));
    EB_CUDA(cudaEventCreateWithFlags(&h->ev[i], cudaEventDisableTiming));
  }
  EB_CUDA(cudaStreamCreateWithFlags(&h->up, cudaStreamNonBlocking));
  for (int i = 0; i < 64; ++i) EB_CUDA(cudaEventCreateWithFlags(&h->cev[i], cudaEventDisableTiming));
  EB_CUDA(cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, device));
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  EB_CUDA(cudaMalloc(&h->exh_stats, 2 * sizeof(unsigned long long)));
  EB_CUDA(cudaMemsetAsync(h->exh_stats, 0, 2 * sizeof(unsigned long long), h->stream));
  int st = binom_init(h->stream);
  if (st) { delete h; return st; }
  EB_CUDA(cudaStreamSynchronize(h->stream));
  h->launches = 1;
  *out = h;
  return EB_OK;
}

int32_t eb_handle_destroy(eb_handle* h) {
  if (!h) return EB_OK;
  cudaSetDevice(h->device);
  cudaDeviceSynchronize();
  if (h->own_stream) cudaStreamDestroy(h->stream);
  for (int i = 0; i < 3; ++i) { cudaStreamDestroy(h->pipe[i]); cudaEventDestroy(h->ev[i]); }
  cudaStreamDestroy(h->up);
  for (int i = 0; i < 64; ++i) cudaEventDestroy(h->cev[i]);
  if (h->in_arena) cudaFree(h->in_arena);
  if (h->dscratch) cudaFree(h->dscratch);
  if (h->exh_stats) cudaFree(h->exh_stats);
  if (h->pinned) cudaFreeHost(h->pinned);
  for (int i = 0; i < 3; ++i) {
    if (h->ctab[i]) cudaFree(h->ctab[i]);
    if (h->ctab_m[i]) cudaFree(h->ctab_m[i]);
    if (h->arena[i]) cudaFree(h->arena[i]);
  }
  delete h;
  return EB_OK;
}

int32_t eb_handle_set_stream(eb_handle* h, void* stream) {
  if (!h) return EB_ERR_INVALID_ARG;
  if (h->own_stream) cudaStreamDestroy(h->stream);
  h->stream = (cudaStream_t)stream;
  h->own_stream = false;
  return EB_OK;
}

int32_t eb_synchronize(eb_handle* h) {
  if (!h) return EB_ERR_INVALID_ARG;
  EB_CUDA(cudaSetDevice(h->device));
  EB_CUDA(cudaStreamSynchronize(h->stream));
  for (int i = 0; i < 3; ++i) EB_CUDA(cudaStreamSynchronize(h->pipe[i]));
  return EB_OK;
}

int64_t eb_kernel_launches(eb_handle* h) { return h ? h->launches : -1; }

int32_t eb_exhaustive_counters(eb_handle* h, int64_t* out) {
  if (!h || !out) return EB_ERR_INVALID_ARG;
  EB_CUDA(cudaSetDevice(h->device));
  unsigned long long v[2];
  EB_CUDA(cudaMemcpyAsync(v, h->exh_stats, sizeof(v), cudaMemcpyDeviceToHost, h->stream));
  EB_CUDA(cudaStreamSynchronize(h->stream));
  out[0] = (int64_t)v[0];
  out[1] = (int64_t)v[1];
  return EB_OK;
}

// ---------------------------------------------------------------------------
int32_t eb_dftsp_batch(eb_handle* h, const eb_context* ctxs, int32_t n_ctx, const eb_search_params* prm,
                       const eb_batch* b, eb_dftsp_result* out, int32_t mem) {
  if (!h || !ctxs || n_ctx < 1 || !prm || !b || !out || !out->status || !out->z_found ||
      !out->nodes_visited || !out->nodes_pruned || b->n_inst < 0 || !b->offsets)
    return EB_ERR_INVALID_ARG;
  if (prm->ladder_len < 0 || prm->ladder_len > EB_MAX_CLASSES) return EB_ERR_INVALID_ARG;
  if (!req_complete(b->req, false)) return EB_ERR_INVALID_ARG;
  if (prm->collect_trajectory && (!out->traj || !out->traj_offsets)) return EB_ERR_INVALID_ARG;
  EB_CUDA(cudaSetDevice(h->device));
  if (b->n_inst == 0) return EB_OK;

  if (mem == EB_MEM_DEVICE) {
    int K = b->k_max;
    if (K < 1 || K > EB_MAX_K_DFTSP) return EB_ERR_INVALID_ARG;
    int st = ensure_dscratch(h, 256);
    if (st) return st;
    return launch_dftsp(h, h->stream, ctxs, n_ctx, *prm, b->n_inst, b->offsets, b->ctx_index, 0, b->req, K,
                        *out, 0, (int*)h->dscratch, -1);
  }
  if (mem != EB_MEM_HOST) return EB_ERR_INVALID_ARG;

  // ---- host memory: validate, then pipeline instance chunks -------------
  // (the int64 range of the exact cost model is checked per instance on the
  // device, status EB_ERR_OVERFLOW; only k_max is needed here)
  const int64_t n = b->n_inst;
  // (the widest instance sizes the kernels; instances wider than EB_MAX_K
  // take the wide pass, counted here to size its grid)
  int K = b->k_max;
  int64_t n_wide = 0;
  if (K <= 0 || K > EB_MAX_K) {      // a k_max <= EB_MAX_K rules out wide instances: skip the scan
    int kk = 0;
    for (int64_t i = 0; i < n; ++i) {
      int64_t sz = b->offsets[i + 1] - b->offsets[i];
      if (sz < 0) return EB_ERR_INVALID_ARG;
      if (sz > kk) kk = (int)(sz > EB_MAX_K_DFTSP ? EB_MAX_K_DFTSP + 1 : sz);
      n_wide += (sz > EB_MAX_K && sz <= EB_MAX_K_DFTSP);
    }
    if (K <= 0 || kk < K) K = kk;
  }
  if (K > EB_MAX_K_DFTSP) K = EB_MAX_K_DFTSP;
  if (K < 1) K = 1;
  return dftsp_host_pipeline(h, ctxs, n_ctx, *prm, n, b->offsets, b->ctx_index, K, n_wide, *out,
                             WideUp{&b->req});
}

int32_t eb_dftsp_batch_packed(eb_handle* h, const eb_context* ctxs, int32_t n_ctx, const eb_search_params* prm,
                              const eb_batch_packed* b, eb_dftsp_result* out, int32_t mem) {
  if (!h || !ctxs || n_ctx < 1 || !prm || !b || !out || !out->status || !out->z_found ||
      !out->nodes_visited || !out->nodes_pruned || b->n_inst < 0)
    return EB_ERR_INVALID_ARG;
  if (prm->ladder_len < 0 || prm->ladder_len > EB_MAX_CLASSES) return EB_ERR_INVALID_ARG;
  const eb_requests_packed& r = b->req;
  if ((!r.token_codes && (!r.prompt_tokens || !r.output_tokens)) || !r.deadline_s || !r.waiting_s ||
      !r.channel_gain || !r.uplink_power_w)
    return EB_ERR_INVALID_ARG;
  if (r.token_codes && (r.n_dict < 1 || r.n_dict > 16)) return EB_ERR_INVALID_ARG;
  if (prm->collect_trajectory && (!out->traj || !out->traj_offsets)) return EB_ERR_INVALID_ARG;
  if (mem != EB_MEM_HOST) return EB_ERR_INVALID_ARG;
  if (b->k_max < 1 || b->k_max > EB_MAX_K) return EB_ERR_INVALID_ARG;
  if (!b->offsets && b->n_req != b->n_inst * (int64_t)b->k_max) return EB_ERR_INVALID_ARG;
  EB_CUDA(cudaSetDevice(h->device));
  if (b->n_inst == 0) return EB_OK;
  return dftsp_host_pipeline(h, ctxs, n_ctx, *prm, b->n_inst, b->offsets, b->ctx_index, b->k_max, 0, *out,
                             WireUp{&r});
}

int32_t eb_dfs_single(eb_handle* h, int32_t z, int32_t n_cls, const int32_t* sizes, const int32_t* lengths,
                      const int32_t* prompt, const double* k_up, const double* k_down, const double* deadline_s,
                      const double* waiting_s, const double coeff[8], int64_t padded_len, int32_t has_tau_min,
                      double tau_min, const eb_search_params* prm, int32_t* out_found, int32_t* out_counts,
                      int64_t* out_visited, int64_t* out_pruned) {
  if (!h || !prm || n_cls < 0 || n_cls > EB_MAX_CLASSES || (n_cls > 0 && (!sizes || !lengths)) || !coeff ||
      !out_found || !out_visited || !out_pruned)
    return EB_ERR_INVALID_ARG;
  EB_CUDA(cudaSetDevice(h->device));
  int total = 0;
  for (int k = 0; k < n_cls; ++k) {
    if (sizes[k] < 0) return EB_ERR_INVALID_ARG;
    total += sizes[k];
  }
  if (total > EB_MAX_K) return EB_ERR_K_TOO_LARGE;
  if (total > 0 && (!prompt || !k_up || !k_down || !deadline_s || !waiting_s)) return EB_ERR_INVALID_ARG;
  const size_t nm = (size_t)(total > 0 ? total : 1), nc = (size_t)(n_cls > 0 ? n_cls : 1);
  Stage S(h, h->stream);
  int32_t* d_sizes = n_cls ? S.up(sizes, nc) : S.alloc<int32_t>(1);
  int32_t* d_len = n_cls ? S.up(lengths, nc) : S.alloc<int32_t>(1);
  int32_t* d_pr = total ? S.up(prompt, nm) : S.alloc<int32_t>(1);
  double* d_ku = total ? S.up(k_up, nm) : S.alloc<double>(1);
  double* d_kd = total ? S.up(k_down, nm) : S.alloc<double>(1);
  double* d_dl = total ? S.up(deadline_s, nm) : S.alloc<double>(1);
  double* d_wt = total ? S.up(waiting_s, nm) : S.alloc<double>(1);
  double* d_co = S.up(coeff, 8);
  int32_t* d_res = S.alloc<int32_t>(2 + EB_MAX_CLASSES + 4);
  if (S.err) return S.err;
  int rc = launch_dfs_single(h, h->stream, z, n_cls, d_sizes, d_len, d_pr, d_ku, d_kd, d_dl, d_wt, d_co,
                             padded_len, has_tau_min, tau_min, *prm, d_res);
  if (rc) return rc;
  int32_t res[2 + EB_MAX_CLASSES + 4];
  S.down(res, d_res, 2 + EB_MAX_CLASSES + 4);
  rc = S.sync();
  if (rc) return rc;
  *out_found = res[0];
  if (out_counts)
    for (int k = 0; k < n_cls; ++k) out_counts[k] = res[2 + k];
  int64_t v, p;
  memcpy(&v, &res[2 + EB_MAX_CLASSES], 8);
  memcpy(&p, &res[2 + EB_MAX_CLASSES + 2], 8);
  *out_visited = v;
  *out_pruned = p;
  return EB_OK;
}

int32_t eb_exhaustive_batch(eb_handle* h, const eb_context* ctxs, int32_t n_ctx, const eb_batch* b, int32_t cap,
                            int32_t* status, int32_t* z_found, int64_t* lexrank, int64_t* nodes_visited,
                            uint64_t* subset_mask, int32_t mem) {
  if (!h || !ctxs || n_ctx < 1 || !b || !b->offsets || !status || !z_found || !lexrank || !nodes_visited ||
      b->n_inst < 0 || !req_complete(b->req, false))
    return EB_ERR_INVALID_ARG;
  EB_CUDA(cudaSetDevice(h->device));
  if (b->n_inst == 0) return EB_OK;
  if (mem == EB_MEM_DEVICE)
    return launch_exh_batch(h, h->stream, ctxs, n_ctx, b->n_inst, b->offsets, b->ctx_index, 0, b->req, cap,
                            status, z_found, lexrank, nodes_visited, subset_mask);
  const int64_t n = b->n_inst, R0 = b->offsets[0], nr = b->offsets[n] - R0;
  Stage S(h, h->stream);
  const eb_context* d_ctx = S.up(ctxs, (size_t)n_ctx);
  const int64_t* d_off = S.up(b->offsets, (size_t)n + 1);
  const int32_t* d_ci = b->ctx_index ? S.up(b->ctx_index, (size_t)n) : nullptr;
  eb_requests d_req = upload_req(S, b->req, R0, nr);
  int32_t* d_st = S.alloc<int32_t>(n);
  int32_t* d_z = S.alloc<int32_t>(n);
  int64_t* d_rk = S.alloc<int64_t>(n);
  int64_t* d_nd = S.alloc<int64_t>(n);
  uint64_t* d_mk = S.out(subset_mask, n);
  if (S.err) return S.err;
  int rc = launch_exh_batch(h, h->stream, d_ctx, n_ctx, n, d_off, d_ci, R0, d_req, cap, d_st, d_z, d_rk, d_nd,
                            d_mk);
  if (rc) return rc;
  S.down(status, d_st, n);
  S.down(z_found, d_z, n);
  S.down(lexrank, d_rk, n);
  S.down(nodes_visited, d_nd, n);
  S.down(subset_mask, d_mk, n);
  return S.sync();
}

int32_t eb_exhaustive_level_range(eb_handle* h, const eb_context* ctx, int32_t k, const eb_requests* req,
                                  int32_t z, int64_t rank_lo, int64_t rank_hi, int64_t* first_rank) {
  if (!h || !ctx || !req || !first_rank || k < 1 || k > EB_MAX_K || z < 1 || z > k || rank_lo < 0 ||
      rank_hi < rank_lo || !req_complete(*req, false))
    return EB_ERR_INVALID_ARG;
  EB_CUDA(cudaSetDevice(h->device));
  *first_rank = -1;
  if (rank_hi == rank_lo) return EB_OK;
  Stage S(h, h->stream);
  eb_requests d_req = upload_req(S, *req, 0, k);
  unsigned long long* d_best = S.alloc<unsigned long long>(2);   // best rank, work counter
  int* d_status = S.alloc<int>(1);
  if (S.err) return S.err;
  int status = 0;
  int rc = exh_range(h, h->stream, *ctx, d_req, k, z, rank_lo, rank_hi, d_best, d_status, first_rank, &status);
  if (rc) return rc;
  rc = S.sync();
  if (rc) return rc;
  return status ? status : EB_OK;
}

int32_t eb_exhaustive_live_levels(eb_handle* h, const eb_context* ctx, int32_t k, const eb_requests* req,
                                  uint64_t* live_mask) {
  if (!h || !ctx || !req || !live_mask || k < 1 || k > EB_MAX_K || !req_complete(*req, false))
    return EB_ERR_INVALID_ARG;
  EB_CUDA(cudaSetDevice(h->device));
  *live_mask = 0;
  Stage S(h, h->stream);
  eb_requests d_req = upload_req(S, *req, 0, k);
  unsigned long long* d_mask = S.alloc<unsigned long long>(1);
  int* d_status = S.alloc<int>(1);
  if (S.err) return S.err;
  int status = 0;
  int rc = exh_levels(h, h->stream, *ctx, d_req, k, d_mask, d_status, live_mask, &status);
  if (rc) return rc;
  rc = S.sync();
  if (rc) return rc;
  return status ? status : EB_OK;
}

int32_t eb_check_direct_batch(eb_handle* h, const eb_context* ctxs, int32_t n_ctx, const eb_requests* req,
                              int64_t n_rows, int64_t n_sub, const int64_t* sub_off, const int32_t* members,
                              const int32_t* sub_ctx, const int64_t* padded_len, int32_t* status,
                              uint8_t* out_ok, double* out_metrics, int32_t mem) {
  if (!h || !ctxs || n_ctx < 1 || !req || n_sub < 0 || !sub_off || !padded_len || !status || !out_ok ||
      !req_complete(*req, false))
    return EB_ERR_INVALID_ARG;
  EB_CUDA(cudaSetDevice(h->device));
  if (n_sub == 0) return EB_OK;
  if (mem == EB_MEM_DEVICE)
    return launch_check_direct(h, h->stream, ctxs, n_ctx, *req, n_sub, sub_off, members, sub_ctx, padded_len,
                               status, out_ok, out_metrics);
  int64_t nm = sub_off[n_sub] - sub_off[0];
  if (sub_off[0] != 0 || nm < 0) return EB_ERR_INVALID_ARG;
  Stage S(h, h->stream);
  const eb_context* d_ctx = S.up(ctxs, (size_t)n_ctx);
  eb_requests d_req = upload_req(S, *req, 0, n_rows);
  const int64_t* d_off = S.up(sub_off, (size_t)n_sub + 1);
  const int32_t* d_mem = S.up(members, (size_t)nm);
  const int32_t* d_sc = sub_ctx ? S.up(sub_ctx, (size_t)n_sub) : nullptr;
  const int64_t* d_pad = S.up(padded_len, (size_t)n_sub);
  int32_t* d_st = S.alloc<int32_t>(n_sub);
  uint8_t* d_ok = S.alloc<uint8_t>(n_sub);
  double* d_met = S.out(out_metrics, (size_t)n_sub * 4);
  if (S.err) return S.err;
  int rc = launch_check_direct(h, h->stream, d_ctx, n_ctx, d_req, n_sub, d_off, d_mem, d_sc, d_pad, d_st, d_ok,
                               d_met);
  if (rc) return rc;
  S.down(status, d_st, n_sub);
  S.down(out_ok, d_ok, n_sub);
  S.down(out_metrics, d_met, (size_t)n_sub * 4);
  return S.sync();
}

int32_t eb_check_knapsack_batch(eb_handle* h, int64_t n_sub, const int64_t* sub_off, const int32_t* prompt,
                                const int32_t* output, const double* k_up, const double* k_down,
                                const double* coeff, const int32_t* z, const double* tau_min, uint8_t* out_ok,
                                int32_t mem) {
  if (!h || n_sub < 0 || !sub_off || !coeff || !z || !tau_min || !out_ok) return EB_ERR_INVALID_ARG;
  EB_CUDA(cudaSetDevice(h->device));
  if (n_sub == 0) return EB_OK;
  if (mem == EB_MEM_DEVICE)
    return launch_check_knapsack(h, h->stream, n_sub, sub_off, prompt, output, k_up, k_down, coeff, z, tau_min,
                                 out_ok);
  int64_t nm = sub_off[n_sub];
  if (sub_off[0] != 0 || nm < 0) return EB_ERR_INVALID_ARG;
  Stage S(h, h->stream);
  const int64_t* d_off = S.up(sub_off, (size_t)n_sub + 1);
  const int32_t* d_p = S.up(prompt, (size_t)nm);
  const int32_t* d_o = S.up(output, (size_t)nm);
  const double* d_ku = S.up(k_up, (size_t)nm);
  const double* d_kd = S.up(k_down, (size_t)nm);
  const double* d_co = S.up(coeff, (size_t)n_sub * 6);
  const int32_t* d_z = S.up(z, (size_t)n_sub);
  const double* d_tm = S.up(tau_min, (size_t)n_sub);
  uint8_t* d_ok = S.alloc<uint8_t>(n_sub);
  if (S.err) return S.err;
  int rc = launch_check_knapsack(h, h->stream, n_sub, d_off, d_p, d_o, d_ku, d_kd, d_co, d_z, d_tm, d_ok);
  if (rc) return rc;
  S.down(out_ok, d_ok, n_sub);
  return S.sync();
}

int32_t eb_coefficients_batch(eb_handle* h, const eb_context* ctxs, int32_t n_ctx, const eb_batch* b,
                              const int64_t* padded_len, int32_t* status, int32_t* error_index,
                              double* out_scalar, double* out_req, int32_t mem) {
  if (!h || !ctxs || n_ctx < 1 || !b || !b->offsets || !status || !out_scalar || !out_req ||
      !req_complete(b->req, false))
    return EB_ERR_INVALID_ARG;
  EB_CUDA(cudaSetDevice(h->device));
  if (b->n_inst == 0) return EB_OK;
  if (mem == EB_MEM_DEVICE)
    return launch_coeff(h, h->stream, ctxs, n_ctx, b->n_inst, b->offsets, b->ctx_index, 0, b->req, padded_len,
                        status, error_index, out_scalar, out_req);
  const int64_t n = b->n_inst, R0 = b->offsets[0], nr = b->offsets[n] - R0;
  Stage S(h, h->stream);
  const eb_context* d_ctx = S.up(ctxs, (size_t)n_ctx);
  const int64_t* d_off = S.up(b->offsets, (size_t)n + 1);
  const int32_t* d_ci = b->ctx_index ? S.up(b->ctx_index, (size_t)n) : nullptr;
  eb_requests d_req = upload_req(S, b->req, R0, nr);
  const int64_t* d_pad = padded_len ? S.up(padded_len, (size_t)n) : nullptr;
  int32_t* d_st = S.alloc<int32_t>(n);
  int32_t* d_err = S.out(error_index, n);
  double* d_sc = S.alloc<double>((size_t)n * 6);
  double* d_rq = S.alloc<double>((size_t)nr * 4);
  if (S.err) return S.err;
  int rc = launch_coeff(h, h->stream, d_ctx, n_ctx, n, d_off, d_ci, R0, d_req, d_pad, d_st, d_err, d_sc, d_rq);
  if (rc) return rc;
  S.down(status, d_st, n);
  S.down(error_index, d_err, n);
  S.down(out_scalar, d_sc, (size_t)n * 6);
  S.down(out_req + 4 * R0, d_rq, (size_t)nr * 4);
  return S.sync();
}

int32_t eb_link_batch(eb_handle* h, const eb_context* ctxs, int32_t n_ctx, const eb_requests* req, int64_t n,
                      const int32_t* req_ctx, int32_t* status, double* out, int32_t mem) {
  if (!h || !ctxs || n_ctx < 1 || !req || n < 0 || !status || !out || !req->channel_gain ||
      !req->uplink_power_w || !req->prompt_tokens || !req->output_tokens)
    return EB_ERR_INVALID_ARG;
  EB_CUDA(cudaSetDevice(h->device));
  if (n == 0) return EB_OK;
  if (mem == EB_MEM_DEVICE) return launch_link(h, h->stream, ctxs, n_ctx, *req, n, req_ctx, status, out);
  Stage S(h, h->stream);
  const eb_context* d_ctx = S.up(ctxs, (size_t)n_ctx);
  eb_requests d_req;
  memset(&d_req, 0, sizeof(d_req));
  d_req.prompt_tokens = S.up(req->prompt_tokens, n);
  d_req.output_tokens = S.up(req->output_tokens, n);
  d_req.channel_gain = S.up(req->channel_gain, n);
  d_req.uplink_power_w = S.up(req->uplink_power_w, n);
  const int32_t* d_rc = req_ctx ? S.up(req_ctx, (size_t)n) : nullptr;
  int32_t* d_st = S.alloc<int32_t>(n);
  double* d_out = S.alloc<double>((size_t)n * 6);
  if (S.err) return S.err;
  int rc = launch_link(h, h->stream, d_ctx, n_ctx, d_req, n, d_rc, d_st, d_out);
  if (rc) return rc;
  S.down(status, d_st, n);
  S.down(out, d_out, (size_t)n * 6);
  return S.sync();
}

int32_t eb_admission_batch(eb_handle* h, const eb_context* ctxs, int32_t n_ctx, const eb_batch* b,
                           int32_t accuracy_check, int32_t prefilter, int32_t* status, uint8_t* out_keep,
                           int32_t mem) {
  if (!h || !ctxs || n_ctx < 1 || !b || !b->offsets || !status || !out_keep ||
      (accuracy_check && !b->req.tolerance) || (prefilter && !req_complete(b->req, false)))
    return EB_ERR_INVALID_ARG;
  EB_CUDA(cudaSetDevice(h->device));
  if (b->n_inst == 0) return EB_OK;
  if (mem == EB_MEM_DEVICE)
    return launch_admission(h, h->stream, ctxs, n_ctx, b->n_inst, b->n_req, b->offsets, b->ctx_index, 0,
                            b->req, accuracy_check, prefilter, status, out_keep);
  const int64_t n = b->n_inst, R0 = b->offsets[0], nr = b->offsets[n] - R0;
  Stage S(h, h->stream);
  const eb_context* d_ctx = S.up(ctxs, (size_t)n_ctx);
  const int64_t* d_off = S.up(b->offsets, (size_t)n + 1);
  const int32_t* d_ci = b->ctx_index ? S.up(b->ctx_index, (size_t)n) : nullptr;
  eb_requests d_req = upload_req(S, b->req, R0, nr);
  int32_t* d_st = S.alloc<int32_t>(nr);
  uint8_t* d_k = S.alloc<uint8_t>(nr);
  if (S.err) return S.err;
  int rc = launch_admission(h, h->stream, d_ctx, n_ctx, n, nr, d_off, d_ci, R0, d_req, accuracy_check, prefilter,
                            d_st, d_k);
  if (rc) return rc;
  S.down(status + R0, d_st, nr);
  S.down(out_keep + R0, d_k, nr);
  return S.sync();
}

int32_t eb_batch_cost_batch(eb_handle* h, const eb_context* ctxs, int32_t n_ctx, int64_t n_plans,
                            const int64_t* plan_off, const int32_t* prompt, const int32_t* output,
                            const int64_t* padded_len, const int64_t* weight_copies, const int32_t* plan_ctx,
                            double* out, int32_t mem) {
  if (!h || !ctxs || n_ctx < 1 || n_plans < 0 || !plan_off || !padded_len || !out) return EB_ERR_INVALID_ARG;
  EB_CUDA(cudaSetDevice(h->device));
  if (n_plans == 0) return EB_OK;
  if (mem == EB_MEM_DEVICE)
    return launch_batch_cost(h, h->stream, ctxs, n_ctx, n_plans, plan_off, prompt, output, padded_len,
                             weight_copies, plan_ctx, out);
  int64_t ne = plan_off[n_plans];
  if (plan_off[0] != 0 || ne < 0) return EB_ERR_INVALID_ARG;
  Stage S(h, h->stream);
  const eb_context* d_ctx = S.up(ctxs, (size_t)n_ctx);
  const int64_t* d_off = S.up(plan_off, (size_t)n_plans + 1);
  const int32_t* d_p = S.up(prompt, (size_t)ne);
  const int32_t* d_o = S.up(output, (size_t)ne);
  const int64_t* d_pad = S.up(padded_len, (size_t)n_plans);
  const int64_t* d_cp = weight_copies ? S.up(weight_copies, (size_t)n_plans) : nullptr;
  const int32_t* d_pc = plan_ctx ? S.up(plan_ctx, (size_t)n_plans) : nullptr;
  double* d_out = S.alloc<double>((size_t)n_plans * 2);
  if (S.err) return S.err;
  int rc = launch_batch_cost(h, h->stream, d_ctx, n_ctx, n_plans, d_off, d_p, d_o, d_pad, d_cp, d_pc, d_out);
  if (rc) return rc;
  S.down(out, d_out, (size_t)n_plans * 2);
  return S.sync();
}

int32_t eb_static_batch_size_batch(eb_handle* h, const eb_context* ctxs, int32_t n, const double* slot_s,
                                   const int64_t* s_max, const int64_t* n_max, int64_t* out_b, int32_t mem) {
  if (!h || !ctxs || n < 0 || !slot_s || !s_max || !n_max || !out_b) return EB_ERR_INVALID_ARG;
  EB_CUDA(cudaSetDevice(h->device));
  if (n == 0) return EB_OK;
  if (mem == EB_MEM_DEVICE) return launch_static_b(h, h->stream, ctxs, n, slot_s, s_max, n_max, out_b);
  Stage S(h, h->stream);
  const eb_context* d_ctx = S.up(ctxs, (size_t)n);
  const double* d_sl = S.up(slot_s, (size_t)n);
  const int64_t* d_s = S.up(s_max, (size_t)n);
  const int64_t* d_n = S.up(n_max, (size_t)n);
  int64_t* d_out = S.alloc<int64_t>(n);
  if (S.err) return S.err;
  int rc = launch_static_b(h, h->stream, d_ctx, n, d_sl, d_s, d_n, d_out);
  if (rc) return rc;
  S.down(out_b, d_out, (size_t)n);
  return S.sync();
}

int32_t eb_stb_batch(eb_handle* h, const eb_context* ctxs, int32_t n_ctx, const eb_batch* b, const int64_t* bsz,
                     int32_t accuracy_check, int32_t* status, uint8_t* out_sel, int32_t mem) {
  if (!h || !ctxs || n_ctx < 1 || !b || !b->offsets || !bsz || !status || !out_sel) return EB_ERR_INVALID_ARG;
  EB_CUDA(cudaSetDevice(h->device));
  if (b->n_inst == 0) return EB_OK;
  if (mem == EB_MEM_DEVICE)
    return launch_stb(h, h->stream, ctxs, n_ctx, b->n_inst, b->offsets, b->ctx_index, 0, b->req, bsz,
                      accuracy_check, status, out_sel);
  const int64_t n = b->n_inst, R0 = b->offsets[0], nr = b->offsets[n] - R0;
  Stage S(h, h->stream);
  const eb_context* d_ctx = S.up(ctxs, (size_t)n_ctx);
  const int64_t* d_off = S.up(b->offsets, (size_t)n + 1);
  const int32_t* d_ci = b->ctx_index ? S.up(b->ctx_index, (size_t)n) : nullptr;
  eb_requests d_req = upload_req(S, b->req, R0, nr);
  const int64_t* d_b = S.up(bsz, (size_t)n);
  int32_t* d_st = S.alloc<int32_t>(n);
  uint8_t* d_sel = S.alloc<uint8_t>(nr);
  if (S.err) return S.err;
  int rc = launch_stb(h, h->stream, d_ctx, n_ctx, n, d_off, d_ci, R0, d_req, d_b, accuracy_check, d_st, d_sel);
  if (rc) return rc;
  S.down(status, d_st, n);
  S.down(out_sel + R0, d_sel, nr);
  return S.sync();
}

int32_t eb_nob_batch(eb_handle* h, const eb_context* ctxs, int32_t n_ctx, const eb_batch* b, const double* now,
                     int32_t accuracy_check, const int32_t* n_dev, int32_t max_dev, double* busy_until, int32_t* status,
                     int8_t* out_action, double* out_completion, int32_t* out_order, int32_t mem) {
  if (!h || !ctxs || n_ctx < 1 || !b || !b->offsets || !now || max_dev < 1 || !busy_until || !status ||
      !out_action || !out_completion || !out_order)
    return EB_ERR_INVALID_ARG;
  EB_CUDA(cudaSetDevice(h->device));
  if (b->n_inst == 0) return EB_OK;
  if (mem == EB_MEM_DEVICE)
    return launch_nob(h, h->stream, ctxs, n_ctx, b->n_inst, b->offsets, b->ctx_index, 0, b->req, now,
                      accuracy_check, n_dev, max_dev, busy_until, status, out_action, out_completion, out_order);
  const int64_t n = b->n_inst, R0 = b->offsets[0], nr = b->offsets[n] - R0;
  Stage S(h, h->stream);
  const eb_context* d_ctx = S.up(ctxs, (size_t)n_ctx);
  const int64_t* d_off = S.up(b->offsets, (size_t)n + 1);
  const int32_t* d_ci = b->ctx_index ? S.up(b->ctx_index, (size_t)n) : nullptr;
  eb_requests d_req = upload_req(S, b->req, R0, nr);
  const double* d_now = S.up(now, (size_t)n);
  const int32_t* d_nd = n_dev ? S.up(n_dev, (size_t)n) : nullptr;
  double* d_busy = S.up(busy_until, (size_t)n * max_dev);
  int32_t* d_st = S.alloc<int32_t>(n);
  int8_t* d_act = S.alloc<int8_t>(nr);
  double* d_cmp = S.alloc<double>(nr);
  int32_t* d_ord = S.alloc<int32_t>(nr);
  if (S.err) return S.err;
  int rc = launch_nob(h, h->stream, d_ctx, n_ctx, n, d_off, d_ci, R0, d_req, d_now, accuracy_check, d_nd, max_dev,
                      d_busy, d_st, d_act, d_cmp, d_ord);
  if (rc) return rc;
  S.down(busy_until, d_busy, (size_t)n * max_dev);
  S.down(status, d_st, n);
  S.down(out_action + R0, d_act, nr);
  S.down(out_completion + R0, d_cmp, nr);
  S.down(out_order + R0, d_ord, nr);
  return S.sync();
}

}  // extern "C"
