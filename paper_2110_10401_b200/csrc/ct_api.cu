// C ABI (include/commtrace_b200.h): context, path dispatch, finalisation.
//
// ct_analyze runs the fast kernel on the trace as given; if its layout preconditions
// fail it canonicalises the trace with the exact sort-based join (ct_exact.cu) and runs
// the fast kernel on the canonical stream.  There is no host fallback: every record is
// classified, joined, expanded and accumulated on the device; the host only reads back
// a few kilobytes of counters and maps flags to the reference's exception classes.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "ct_canon.cuh"
#include "ct_exact.cuh"
#include "ct_fast.cuh"

namespace ct {
template <bool SH>
__global__ void fast_kernel(FastParams P);
__global__ void range_check_kernel(const ct_record* recs, const WarpSlot* slots, const Chans chans,
                                   uint32_t total_warps, GlobalState* st);
int generate(int kind, uint64_t seed, uint64_t first, uint64_t n, ct_record* out, cudaStream_t st);
uint64_t generate_boundary(int kind, uint64_t at);
void launch_emit(const ct_record* recs, uint64_t n, const ExpandParams& ex, uint32_t* counts,
                 const uint64_t* offsets, int64_t* rows, int pass, unsigned int* flags, cudaStream_t st);
}  // namespace ct

using namespace ct;

struct ct_context {
  int device = 0;
  cudaStream_t stream = nullptr;
  int num_sms = 148;
  std::string err;
  ct_record* in_buf = nullptr;
  uint64_t in_cap = 0;
  GlobalState* st = nullptr;
  unsigned long long* cells = nullptr;  // bytes then freq
  size_t cells_cap = 0;                 // entries per array
  unsigned long long* tcf = nullptr;    // [5][n_comms] type_comm_first, then [n_comms] comm_first
  size_t tcf_cap = 0;
  WarpSlot* slots = nullptr;   // per (warp range, comm slot) order summaries
  size_t slots_cap = 0;
  uint64_t* chans = nullptr;   // per (warp range, p2p channel) order summaries (Chans layout)
  size_t chans_cap = 0;
  uint32_t last_total_warps = 0;
  uint16_t* ring = nullptr;  // order then inverse
  int ring_cap = 0;
  cudaEvent_t ev[4];
  // last result
  ct_summary last{};
  int last_g2 = 0;
  GlobalState last_state{};
  const ct_record* last_input = nullptr;  // device pointer of last analysed array
  uint64_t last_n = 0;
  uint32_t last_comms = 0;
  bool mat_valid = false;
  ExactResult mat;
  ct_record* canon_keep = nullptr;  // exact-path canonical stream of the last call
  bool last_explicit = false;
  uint64_t canon_n = 0;
  ShardState shard;  // multi-GPU canonicalise-then-shard state (ct_shard_*)
  unsigned char* exp_tab = nullptr;  // ct_partial_export: global comm / channel hash tables
  size_t exp_tab_cap = 0;
  // pinned host copies of the last fast run's state / cells / first-occurrence keys:
  // read back with one synchronisation, then used by summarize_state
  GlobalState* h_state = nullptr;  // [0] initial state uploaded, [1] result
  unsigned long long* h_cells = nullptr;
  size_t h_cells_cap = 0;
  unsigned long long* h_tcf = nullptr;
  size_t h_tcf_cap = 0;
  int h_g2 = 0;             // layout the host copies hold (0: none)
  uint32_t h_comms = 0;
};

namespace {

int fail(ct_context* c, int code, const std::string& msg) {
  if (c) c->err = msg;
  return code;
}

int cuda_fail(ct_context* c, cudaError_t e, const char* where) {
  return fail(c, CT_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define CTX_TRY(c, x)                                        \
  do {                                                       \
    cudaError_t e_ = (x);                                    \
    if (e_ != cudaSuccess) return cuda_fail(c, e_, #x);      \
  } while (0)

template <typename T>
int ensure(ct_context* c, T*& p, size_t& cap, size_t need) {
  if (need <= cap && p) return 0;
  if (p) cudaFree(p);
  p = nullptr;
  size_t n = std::max(need, (size_t)1);
  cudaError_t e = cudaMalloc(&p, n * sizeof(T));
  if (e != cudaSuccess) { cap = 0; return cuda_fail(c, e, "cudaMalloc"); }
  cap = n;
  return 0;
}

template <typename T>
int ensure_host(ct_context* c, T*& p, size_t& cap, size_t need) {
  if (need <= cap && p) return 0;
  if (p) cudaFreeHost(p);
  p = nullptr;
  size_t n = std::max(need, (size_t)1);
  cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&p), n * sizeof(T), cudaHostAllocDefault);
  if (e != cudaSuccess) { cap = 0; p = nullptr; return cuda_fail(c, e, "cudaHostAlloc"); }
  cap = n;
  return 0;
}

struct RunOut {
  GlobalState gs;
  float ms_kernel;
  uint32_t launches;
};

// One pass of the fast kernel + the cross-range order check over ``recs``.
int run_fast(ct_context* c, const ct_record* recs, uint64_t n, int gcap, bool explicit_d,
                  const ExpandParams& ex, uint32_t n_comms, cudaStream_t st, RunOut* out) {
  const int g2 = gcap + 2;
  const size_t ncell = (size_t)kTypes * g2 * g2;
  if (ensure(c, c->cells, c->cells_cap, 2 * ncell)) return CT_ERR_CUDA;
  size_t tcf_need = 6 * (size_t)std::max<uint32_t>(n_comms, 1);
  if (ensure(c, c->tcf, c->tcf_cap, tcf_need)) return CT_ERR_CUDA;
  const uint64_t n_chunks = (n + 31) / 32;
  // one CTA (16 warps) per SM; small traces use fewer CTAs (>= 4 chunks per warp)
  uint32_t grid = (uint32_t)std::min<uint64_t>((uint64_t)c->num_sms, (n_chunks + 4 * kWarps - 1) / (4 * kWarps));
  if (grid == 0) grid = 1;
  const uint32_t total_warps = grid * kWarps;
  size_t sc = c->slots_cap;
  if (ensure(c, c->slots, sc, (size_t)total_warps * kCS)) return CT_ERR_CUDA;
  c->slots_cap = sc;
  size_t pc = c->chans_cap;
  if (ensure(c, c->chans, pc, (size_t)total_warps * kPC * kChanWords)) return CT_ERR_CUDA;
  c->chans_cap = pc;
  c->last_total_warps = total_warps;

  CTX_TRY(c, cudaMemsetAsync(c->cells, 0, 2 * ncell * sizeof(unsigned long long), st));
  CTX_TRY(c, cudaMemsetAsync(c->tcf, 0xFF, tcf_need * sizeof(unsigned long long), st));
  {
    size_t hs_cap = c->h_state ? 2 : 0;
    if (ensure_host(c, c->h_state, hs_cap, 2)) return CT_ERR_CUDA;
    if (ensure_host(c, c->h_cells, c->h_cells_cap, 2 * ncell)) return CT_ERR_CUDA;
    if (ensure_host(c, c->h_tcf, c->h_tcf_cap, tcf_need)) return CT_ERR_CUDA;
    c->h_g2 = 0;  // invalid until this run's read-back
    GlobalState& init = c->h_state[0];
    init = GlobalState{};
    init.max_dev = -1;
    for (int k = 0; k < 3; k++) init.copy_first[k] = ~0ull;
    init.oor_key = ~0ull;
    init.of_cell = ~0ull;
    CTX_TRY(c, cudaMemcpyAsync(c->st, &init, sizeof init, cudaMemcpyHostToDevice, st));
  }
  FastParams P{};
  P.recs = recs;
  P.n = n;
  P.gcap = gcap;
  P.g2 = g2;
  P.explicit_d = explicit_d;
  P.ex = ex;
  P.n_comms = n_comms;
  const size_t smem_full = fast_smem_bytes(g2, 1);
  P.smem_hist = smem_full <= 227 * 1024 ? 1 : 0;
  const size_t smem = fast_smem_bytes(g2, P.smem_hist);
  P.st = c->st;
  P.cells = c->cells;
  P.freq = c->cells + ncell;
  P.type_comm_first = c->tcf;
  P.comm_first = c->tcf + 5 * (size_t)std::max<uint32_t>(n_comms, 1);
  P.slots = c->slots;
  P.chans = Chans{c->chans, (uint64_t)total_warps * kPC};
  P.total_warps = total_warps;
  P.n_chunks = n_chunks;
  P.dbg = getenv("CT_DEBUG_MODE") ? atoi(getenv("CT_DEBUG_MODE")) : 0;
  P.sa_flush = 1u << 14;  // CT_SA_FLUSH (tests): write slot accumulators out more often
  if (getenv("CT_SA_FLUSH")) P.sa_flush = (uint32_t)std::min(std::max(atoi(getenv("CT_SA_FLUSH")), 1), 1 << 14);
  uint32_t launches = 0;  // kernels launched (cudaMemset/Memcpy are copy-engine work)
  out->ms_kernel = 0;
  if (n) {
    auto kern = P.smem_hist ? fast_kernel<true> : fast_kernel<false>;
    CTX_TRY(c, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CTX_TRY(c, cudaEventRecord(c->ev[0], st));
    kern<<<grid, kThreads, smem, st>>>(P);
    CTX_TRY(c, cudaGetLastError());
    CTX_TRY(c, cudaEventRecord(c->ev[1], st));
    const uint64_t threads = (uint64_t)total_warps * (kCS + kPC);
    range_check_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(recs, c->slots, P.chans, total_warps,
                                                                          c->st);
    CTX_TRY(c, cudaGetLastError());
    launches += 2;
  }
  // state, cells and first-occurrence keys in one round trip (summarize_state reuses them)
  CTX_TRY(c, cudaMemcpyAsync(&c->h_state[1], c->st, sizeof(GlobalState), cudaMemcpyDeviceToHost, st));
  CTX_TRY(c, cudaMemcpyAsync(c->h_cells, c->cells, 2 * ncell * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
  CTX_TRY(c, cudaMemcpyAsync(c->h_tcf, c->tcf, tcf_need * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
  CTX_TRY(c, cudaStreamSynchronize(st));
  out->gs = c->h_state[1];
  c->h_g2 = g2;
  c->h_comms = n_comms;
  if (n) CTX_TRY(c, cudaEventElapsedTime(&out->ms_kernel, c->ev[0], c->ev[1]));
  out->launches = launches;
  return 0;
}

__global__ void k_max_dev(const ct_record* recs, uint64_t n, int* out) {
  int m = -1;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const ct_record& r = recs[i];
    m = max(m, (int)r.dev);
    if ((r.kc & 7) >= CT_KIND_MEMCPY) {
      const int ck = (r.ad >> 6) & 3;
      if (ck != CT_CKIND_H2D) m = max(m, (int)r.aux);
      if (ck != CT_CKIND_D2H) m = max(m, (int)r.aux2);
    }
  }
  atomicMax(out, m);
}

int host_dev_of(ct_context* c, const ct_record* recs, uint64_t i, cudaStream_t st, ct_record* out) {
  CTX_TRY(c, cudaMemcpyAsync(out, recs + i, sizeof(ct_record), cudaMemcpyDeviceToHost, st));
  CTX_TRY(c, cudaStreamSynchronize(st));
  return 0;
}

// Summary from a (possibly merged) GlobalState plus the cells / first-index tables in
// the context: dict order, net flags, the combined 63-bit bound and the reference's
// status precedence (decomposition errors before accumulation errors).
int summarize_state(ct_context* c, const GlobalState& gs, int gcap, int64_t d, int path,
                    const uint64_t extra_diag[3], const ct_record* arr, uint32_t n_comms,
                    cudaStream_t st, ct_summary* out, const unsigned long long* pre_tcf = nullptr,
                    const unsigned long long* pre_cells = nullptr) {
  const int g2 = gcap + 2;
  const size_t ncell = (size_t)kTypes * g2 * g2;
  c->last_state = gs;
  c->last_g2 = g2;
  out->path = path;
  out->d = d;
  out->g_cap = gcap;
  for (int t = 0; t < kTypes; t++) {
    out->calls[t] = gs.calls[t];
    out->payload_lo[t] = gs.pay_lo[t];
    out->payload_hi[t] = gs.pay_hi[t];
  }
  for (int k = 0; k < CT_NDIAG; k++) out->diag[k] = gs.diag[k];
  out->diag[CT_DIAG_INCOMPLETE] += extra_diag[0];
  out->diag[CT_DIAG_UNMATCHED_SEND] += extra_diag[1];
  out->diag[CT_DIAG_UNMATCHED_RECV] += extra_diag[2];
  std::vector<unsigned long long> h(2 * ncell);  // cells (bytes, then frequencies)
  // per_primitive dict order (matrix.py:334-335): collectives by (comm first-seen,
  // first valid instance), then sendrecv, then copies by first event
  {
    std::vector<unsigned long long> tcf(6 * (size_t)n_comms);
    if (pre_tcf && pre_cells) {  // already on the host (one sync with the caller's own reads)
      std::copy(pre_tcf, pre_tcf + tcf.size(), tcf.begin());
      std::copy(pre_cells, pre_cells + h.size(), h.begin());
    } else {
      CTX_TRY(c, cudaMemcpyAsync(tcf.data(), c->tcf, tcf.size() * 8, cudaMemcpyDeviceToHost, st));
      CTX_TRY(c, cudaMemcpyAsync(h.data(), c->cells, 2 * ncell * 8, cudaMemcpyDeviceToHost, st));  // one sync for both
      CTX_TRY(c, cudaStreamSynchronize(st));
    }
    const unsigned long long* cf = tcf.data() + 5 * (size_t)n_comms;
    std::vector<std::pair<std::pair<uint64_t, uint64_t>, int>> order;
    for (int t = 0; t < 5; t++) {
      uint64_t best_c = ~0ull, best_i = ~0ull;
      for (uint32_t cm = 0; cm < n_comms; cm++) {
        const uint64_t v = tcf[(size_t)t * n_comms + cm];
        if (v == ~0ull) continue;
        if (cf[cm] < best_c || (cf[cm] == best_c && v < best_i)) { best_c = cf[cm]; best_i = v; }
      }
      order.push_back({{best_c, best_i}, t});
    }
    std::sort(order.begin(), order.end());
    for (int k = 0; k < 5; k++)
      out->type_first[order[k].second] = order[k].first.first == ~0ull ? ~0ull : (uint64_t)k;
    out->type_first[CT_T_SENDRECV] = gs.calls[CT_T_SENDRECV] ? 5 : ~0ull;
    std::vector<std::pair<uint64_t, int>> copies;
    for (int k = 0; k < 3; k++) copies.push_back({gs.copy_first[k], k});
    std::sort(copies.begin(), copies.end());
    for (int k = 0; k < 3; k++)
      out->type_first[CT_T_EXPLICIT + copies[k].second] = copies[k].first == ~0ull ? ~0ull : (uint64_t)(6 + k);
  }
  // cells, net flags, combined 63-bit bound (matrix.py:110-113)
  // copy statistics: every copy adds exactly one transfer of its byte count to its type
  // (decompose.py:397-406), so calls / payload are the plane's frequency / byte sums
  // (the fast kernel does not count them separately)
  for (int t = CT_T_EXPLICIT; t < kTypes; t++) {
    unsigned __int128 pay = 0;
    uint64_t calls = 0;
    for (size_t k = (size_t)t * g2 * g2; k < (size_t)(t + 1) * g2 * g2; k++) {
      pay += h[k];
      calls += h[ncell + k];
    }
    out->calls[t] = calls;
    out->payload_lo[t] = (uint64_t)pay;
    out->payload_hi[t] = (uint64_t)(pay >> 64);
  }
  bool overflow = (gs.flags & F_OVERFLOW) != 0;
  uint64_t of_cell = ~0ull;
  int net_used = 0;
  for (int t = 0; t < kTypes; t++)
    for (int a = 0; a < g2; a++)
      if (h[ncell + ((size_t)t * g2 + a) * g2 + kNet] || h[ncell + ((size_t)t * g2 + kNet) * g2 + a])
        net_used |= 1 << t;
  for (int a = 0; a < g2; a++)
    for (int b = 0; b < g2; b++) {
      unsigned __int128 sum = 0;
      for (int t = 0; t < kTypes; t++) sum += h[((size_t)t * g2 + a) * g2 + b];
      if (sum > (unsigned __int128)INT64_MAX) {
        overflow = true;
        if (of_cell == ~0ull) of_cell = ((uint64_t)a << 32) | (uint64_t)b;
      }
    }
  if (overflow && of_cell == ~0ull && gs.of_cell != ~0ull) {  // a per-type sum wrapped past 2^64
    const uint64_t a = (gs.of_cell / g2) % g2, b = gs.of_cell % g2;
    of_cell = (a << 32) | b;
  }
  out->net_used = net_used;
  if (gs.flags & F_COMM_RANGE) return fail(c, CT_ERR_ARGUMENT, "record comm id >= n_comms");
  if (gs.flags & F_BAD_RING) out->status = CT_ERR_INVALID_CONFIG;
  else if (gs.flags & F_WRONG_ALGO) out->status = CT_ERR_WRONG_ALGORITHM;
  else if (gs.flags & F_MISSING_ROOT) out->status = CT_ERR_MISSING_ROOT;
  else if (gs.flags & F_OOR) {
    out->status = CT_ERR_ENDPOINT_RANGE;
    const uint64_t k = gs.oor_key;
    const uint64_t cls = k >> 62, elem = (k >> 21) & ((1ull << 41) - 1);
    const uint64_t a = (k >> 11) & 1023, sub = (k >> 1) & 1023, which = k & 1;
    ct_record r{};
    uint64_t gpu = 0;
    if (!arr) {
      gpu = gs.err_index;  // merged partials carry the offending GPU id
    } else if (cls == 0) {
      ct_record head{};
      if (host_dev_of(c, arr, elem, st, &head)) return CT_ERR_CUDA;
      const bool collnet = (head.ad & 3) == CT_ALGO_COLLNET && ((head.kc >> 3) & 7) == CT_COLL_ALLREDUCE;
      const uint64_t rank = which == 0 || collnet ? a : sub;
      if (host_dev_of(c, arr, elem + rank, st, &r)) return CT_ERR_CUDA;
      gpu = r.dev;
    } else if (cls == 1) {
      if (host_dev_of(c, arr, elem + which, st, &r)) return CT_ERR_CUDA;
      gpu = r.dev;
    } else {
      if (host_dev_of(c, arr, elem, st, &r)) return CT_ERR_CUDA;
      gpu = which ? r.aux2 : r.aux;
    }
    out->err_aux[0] = gpu;
    out->err_aux[1] = (uint64_t)d;
  } else if (overflow) {
    out->status = CT_ERR_OVERFLOW;
    out->err_aux[0] = of_cell;
  }
  return 0;
}

}  // namespace

extern "C" {

int ct_context_create(int device, ct_context** out) {
  if (!out) return CT_ERR_ARGUMENT;
  ct_context* c = new ct_context();
  c->device = device;
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
  for (int k = 0; k < 4 && e == cudaSuccess; k++) e = cudaEventCreate(&c->ev[k]);
  if (e == cudaSuccess) e = cudaMalloc(&c->st, sizeof(GlobalState));
  if (e == cudaSuccess) {  // keep freed stream-ordered memory in the pool (exact-path scratch is large)
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t keep = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
  }
  if (e != cudaSuccess) {
    delete c;
    return CT_ERR_CUDA;
  }
  *out = c;
  return CT_OK;
}

int ct_context_destroy(ct_context* c) {
  if (!c) return CT_ERR_ARGUMENT;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  cudaFree(c->in_buf);
  cudaFree(c->st);
  cudaFree(c->cells);
  cudaFree(c->tcf);
  cudaFree(c->slots);
  cudaFree(c->chans);
  cudaFree(c->exp_tab);
  cudaFreeHost(c->h_state);
  cudaFreeHost(c->h_cells);
  cudaFreeHost(c->h_tcf);
  cudaFree(c->ring);
  if (c->canon_keep) cudaFree(c->canon_keep);
  for (int k = 0; k < 4; k++) cudaEventDestroy(c->ev[k]);
  cudaStreamDestroy(c->stream);
  delete c;
  return CT_OK;
}

const char* ct_last_error(ct_context* c) { return c ? c->err.c_str() : "null context"; }

int ct_analyze(ct_context* c, const ct_record* recs, uint64_t n, int on_device, const ct_config* cfg,
               ct_summary* out, void* stream) {
  if (!c || !cfg || !out || (n && !recs)) return fail(c, CT_ERR_ARGUMENT, "null argument");
  CTX_TRY(c, cudaSetDevice(c->device));
  cudaStream_t st = stream ? (cudaStream_t)stream : c->stream;
  memset(out, 0, sizeof *out);
  out->n_records = n;
  c->mat_valid = false;
  if (c->canon_keep) { cudaFree(c->canon_keep); c->canon_keep = nullptr; c->canon_n = 0; }
  CTX_TRY(c, cudaEventRecord(c->ev[2], st));
  const ct_record* d_recs = recs;
  if (!on_device && n) {
    size_t cap = c->in_cap;
    if (ensure(c, c->in_buf, cap, n)) return CT_ERR_CUDA;
    c->in_cap = cap;
    CTX_TRY(c, cudaMemcpyAsync(c->in_buf, recs, n * sizeof(ct_record), cudaMemcpyHostToDevice, st));
    d_recs = c->in_buf;
  }
  c->last_input = d_recs;
  c->last_n = n;
  const uint32_t n_comms = (uint32_t)std::max(cfg->n_comms, 1);
  c->last_comms = n_comms;
  if (n_comms >= (1u << 31)) return fail(c, CT_ERR_ARGUMENT, "more than 2^31 communicators");

  // ring order: validity is decided here, raising happens only when a ring instance uses it
  ExpandParams ex{};
  ex.tree_threshold = cfg->tree_threshold;
  ex.ring_len = cfg->ring_len > 0 ? cfg->ring_len : -1;
  ex.ring_valid = 1;
  if (cfg->ring_len > 0) {
    const int L = cfg->ring_len;
    std::vector<uint16_t> h(2 * (size_t)L, 0);
    std::vector<int> seen(L, 0);
    for (int k = 0; k < L; k++) {
      uint16_t v = cfg->ring_order[k];
      h[k] = v;
      if (v >= L || seen[v]) ex.ring_valid = 0;
      else { seen[v] = 1; h[L + v] = (uint16_t)k; }
    }
    size_t cap = (size_t)c->ring_cap;
    if (ensure(c, c->ring, cap, 2 * (size_t)L)) return CT_ERR_CUDA;
    c->ring_cap = (int)cap;
    CTX_TRY(c, cudaMemcpyAsync(c->ring, h.data(), 2 * (size_t)L * 2, cudaMemcpyHostToDevice, st));
    ex.ring_order = c->ring;
    ex.ring_inv = c->ring + L;
  }

  const bool explicit_d = cfg->d >= 0;
  c->last_explicit = explicit_d;
  if (explicit_d && cfg->d > 65536) return fail(c, CT_ERR_ARGUMENT, "d exceeds the 16-bit device range");
  int gcap = explicit_d ? (int)cfg->d : (cfg->dev_hint > 0 ? cfg->dev_hint : 16);

  RunOut ro{};
  uint32_t launches = 0;
  int path = 1;
  bool counted = false;  // the counting canonicaliser produced the stream (already analysed)
  int max_dev = -1;
  const ct_record* arr = d_recs;
  uint64_t arr_n = n;
  ExactResult ex_res;
  bool ran_exact = false;
  auto do_exact = [&]() -> int {
    int e = exact_canonicalize(d_recs, n, n_comms, st, false, &ex_res);
    if (e == kExactCapacity) return fail(c, CT_ERR_CAPACITY, "exact path: 2^32 or more collective records");
    if (e) return cuda_fail(c, (cudaError_t)e, "exact path");
    launches += ex_res.launches;
    ran_exact = true;
    path = 2;
    return 0;
  };

  // capture layout (ranks interleaved): counting canonicaliser; its stream must pass the
  // fast kernel's order checks, else the exact path runs on the original records
  auto do_counting = [&]() -> int {  // 1: canonical stream ready, 0: not applicable
    ExactResult cr;
    int md = -1;
    const int e = count_canonicalize(d_recs, n, n_comms, c->num_sms, st, &cr, &md);
    if (e == kCanonUnsupported) return 0;
    if (e) return -cuda_fail(c, (cudaError_t)e, "counting canonicaliser");
    launches += cr.launches;
    RunOut probe{};
    const int gprobe = explicit_d ? gcap : std::max(gcap, md + 1);
    if (int e2 = run_fast(c, cr.canon, cr.m, gprobe, explicit_d, ex, n_comms, st, &probe)) {
      cudaFreeAsync(cr.canon, st);
      return -e2;
    }
    launches += probe.launches;
    if (probe.gs.flags & F_NONCANON) {  // file order is not seq order somewhere: sort instead
      cudaFreeAsync(cr.canon, st);
      return 0;
    }
    ex_res = cr;
    ro = probe;
    gcap = gprobe;
    max_dev = md;
    ran_exact = true;
    counted = true;
    path = 3;
    return 1;
  };

  if (cfg->force_path == 2) {
    if (int e = do_exact()) return e;
  } else if (cfg->force_path == 3) {
    const int r = do_counting();
    if (r < 0) return -r;
    if (r == 0) return fail(c, CT_ERR_NOT_CANONICAL, "trace is outside the counting canonicaliser's scope");
  } else {
    if (int e = run_fast(c, d_recs, n, gcap, explicit_d, ex, n_comms, st, &ro)) return e;
    launches += ro.launches;
    max_dev = ro.gs.max_dev;
    if (ro.gs.flags & F_NONCANON) {
      if (cfg->force_path == 1) return fail(c, CT_ERR_NOT_CANONICAL, "trace is not in the canonical layout");
      max_dev = -1;  // the aborted pass may not have visited every record: re-infer d below
      const int r = do_counting();
      if (r < 0) return -r;
      if (r == 0)
        if (int e = do_exact()) return e;
    }
  }
  if (ran_exact) {
    if (ex_res.fatal) {
      out->status = ex_res.fatal;
      out->path = 2;
      out->err_index = ex_res.err_index;
      memcpy(out->err_aux, ex_res.err_aux, sizeof out->err_aux);
      out->err_aux[3] = (uint64_t)ex_res.fatal_kind;
      if (ex_res.canon) cudaFreeAsync(ex_res.canon, st);
      c->last = *out;
      return out->status;
    }
    if (max_dev < 0 && n) {  // the fast pass did not run: infer d over all records
      int* d_m;
      CTX_TRY(c, cudaMallocAsync(&d_m, 4, st));
      int init = -1;
      CTX_TRY(c, cudaMemcpyAsync(d_m, &init, 4, cudaMemcpyHostToDevice, st));
      k_max_dev<<<std::min<uint64_t>((n + 255) / 256, 4096), 256, 0, st>>>(d_recs, n, d_m);
      CTX_TRY(c, cudaMemcpyAsync(&max_dev, d_m, 4, cudaMemcpyDeviceToHost, st));
      CTX_TRY(c, cudaStreamSynchronize(st));
      cudaFreeAsync(d_m, st);
      launches++;
    }
    arr = ex_res.canon;
    arr_n = ex_res.m;
    c->canon_keep = ex_res.canon;
    c->canon_n = ex_res.m;
    if (!counted) {
      if (int e = run_fast(c, arr, arr_n, gcap, explicit_d, ex, n_comms, st, &ro)) return e;
      launches += ro.launches;
      if (ro.gs.flags & F_NONCANON) return fail(c, CT_ERR_CUDA, "internal: canonical stream rejected");
    }
  }
  const int64_t d = explicit_d ? cfg->d : (int64_t)max_dev + 1;
  if (!explicit_d && d > gcap) {
    // histogram too small for the inferred device count: rerun with the exact size
    gcap = (int)d;
    if (int e = run_fast(c, arr, arr_n, gcap, false, ex, n_comms, st, &ro)) return e;
    launches += ro.launches;
  }
  {
    const uint64_t extra[3] = {ran_exact ? ex_res.n_incomplete : 0, ran_exact ? ex_res.n_unmatched_send : 0,
                               ran_exact ? ex_res.n_unmatched_recv : 0};
    const bool pre = c->h_g2 == gcap + 2 && c->h_comms == n_comms;  // the final run's read-back
    if (int e = summarize_state(c, ro.gs, gcap, d, path, extra, arr, n_comms, st, out, pre ? c->h_tcf : nullptr,
                                pre ? c->h_cells : nullptr))
      return e;
  }
  CTX_TRY(c, cudaEventRecord(c->ev[3], st));
  CTX_TRY(c, cudaEventSynchronize(c->ev[3]));
  CTX_TRY(c, cudaEventElapsedTime(&out->ms_total, c->ev[2], c->ev[3]));
  out->ms_kernel = ro.ms_kernel;
  out->n_launches = launches;
  c->last = *out;
  return out->status;
}

int ct_result_cells(ct_context* c, uint64_t* bytes, uint64_t* freq, uint64_t n_cells) {
  if (!c || !bytes || !freq) return fail(c, CT_ERR_ARGUMENT, "null argument");
  const size_t ncell = (size_t)kTypes * c->last_g2 * c->last_g2;
  if (n_cells < ncell) return fail(c, CT_ERR_ARGUMENT, "cell buffer too small");
  CTX_TRY(c, cudaMemcpyAsync(bytes, c->cells, ncell * 8, cudaMemcpyDeviceToHost, c->stream));
  CTX_TRY(c, cudaMemcpyAsync(freq, c->cells + ncell, ncell * 8, cudaMemcpyDeviceToHost, c->stream));
  CTX_TRY(c, cudaStreamSynchronize(c->stream));
  return CT_OK;
}

static int ensure_materialized(ct_context* c) {
  if (c->mat_valid) return 0;
  c->mat = ExactResult();
  int e = exact_canonicalize(c->last_input, c->last_n, c->last_comms, c->stream, true, &c->mat);
  if (e == kExactCapacity) return fail(c, CT_ERR_CAPACITY, "materialize: 2^32 or more collective records");
  if (e) return cuda_fail(c, (cudaError_t)e, "materialize");
  if (c->mat.canon) cudaFreeAsync(c->mat.canon, c->stream);
  c->mat.canon = nullptr;
  cudaStreamSynchronize(c->stream);
  c->mat_valid = true;
  return 0;
}

int ct_materialize(ct_context* c, const ct_record* recs, uint64_t n, int on_device, int32_t n_comms,
                   ct_summary* out) {
  if (!c || !out || (n && !recs)) return fail(c, CT_ERR_ARGUMENT, "null argument");
  memset(out, 0, sizeof *out);
  CTX_TRY(c, cudaSetDevice(c->device));
  const ct_record* d_recs = recs;
  if (!on_device && n) {
    size_t cap = c->in_cap;
    if (ensure(c, c->in_buf, cap, n)) return CT_ERR_CUDA;
    c->in_cap = cap;
    CTX_TRY(c, cudaMemcpyAsync(c->in_buf, recs, n * sizeof(ct_record), cudaMemcpyHostToDevice, c->stream));
    d_recs = c->in_buf;
  }
  c->last_input = d_recs;
  c->last_n = n;
  c->last_comms = (uint32_t)std::max(n_comms, 1);
  c->mat_valid = false;
  if (int e = ensure_materialized(c)) return e;
  if (c->mat.fatal) {
    out->status = c->mat.fatal;
    out->path = 2;
    out->err_index = c->mat.err_index;
    memcpy(out->err_aux, c->mat.err_aux, sizeof out->err_aux);
    out->err_aux[3] = (uint64_t)c->mat.fatal_kind;
    c->mat_valid = false;
    return out->status;
  }
  return CT_OK;
}

int ct_infer_device_count(ct_context* c, const ct_record* recs, uint64_t n, int on_device, int64_t* d) {
  if (!c || !d || (n && !recs)) return fail(c, CT_ERR_ARGUMENT, "null argument");
  CTX_TRY(c, cudaSetDevice(c->device));
  cudaStream_t st = c->stream;
  const ct_record* d_recs = recs;
  if (!on_device && n) {
    size_t cap = c->in_cap;
    if (ensure(c, c->in_buf, cap, n)) return CT_ERR_CUDA;
    c->in_cap = cap;
    CTX_TRY(c, cudaMemcpyAsync(c->in_buf, recs, n * sizeof(ct_record), cudaMemcpyHostToDevice, st));
    d_recs = c->in_buf;
  }
  int* d_m;
  int m = -1;
  CTX_TRY(c, cudaMallocAsync(&d_m, 4, st));
  CTX_TRY(c, cudaMemcpyAsync(d_m, &m, 4, cudaMemcpyHostToDevice, st));
  if (n) k_max_dev<<<(unsigned)std::min<uint64_t>((n + 255) / 256, 4096), 256, 0, st>>>(d_recs, n, d_m);
  CTX_TRY(c, cudaMemcpyAsync(&m, d_m, 4, cudaMemcpyDeviceToHost, st));
  CTX_TRY(c, cudaStreamSynchronize(st));
  cudaFreeAsync(d_m, st);
  *d = (int64_t)m + 1;
  return CT_OK;
}

int ct_result_groups(ct_context* c, uint64_t* rows, uint64_t row_cap, uint64_t* members,
                     uint64_t member_cap, uint64_t* n_rows, uint64_t* n_members) {
  if (!c || !n_rows || !n_members) return fail(c, CT_ERR_ARGUMENT, "null argument");
  if (int e = ensure_materialized(c)) return e;
  *n_rows = c->mat.groups.size();
  *n_members = c->mat.members.size();
  if (rows && row_cap >= *n_rows)
    for (size_t k = 0; k < c->mat.groups.size(); k++) {
      const GroupRow& g = c->mat.groups[k];
      uint64_t* o = rows + 5 * k;
      o[0] = g.comm; o[1] = g.ordinal; o[2] = g.status; o[3] = g.n_members; o[4] = g.member_off;
    }
  if (members && member_cap >= *n_members)
    std::copy(c->mat.members.begin(), c->mat.members.end(), members);
  return CT_OK;
}

int ct_result_p2p_diags(ct_context* c, uint64_t* rows, uint64_t row_cap, uint64_t* n_rows) {
  if (!c || !n_rows) return fail(c, CT_ERR_ARGUMENT, "null argument");
  if (int e = ensure_materialized(c)) return e;
  *n_rows = c->mat.p2p_diags.size();
  if (rows && row_cap >= *n_rows)
    for (size_t k = 0; k < c->mat.p2p_diags.size(); k++) {
      const P2PDiagRow& g = c->mat.p2p_diags[k];
      uint64_t* o = rows + 7 * k;
      o[0] = g.reason; o[1] = g.comm; o[2] = g.src; o[3] = g.dst; o[4] = g.k; o[5] = g.send_idx; o[6] = g.recv_idx;
    }
  return CT_OK;
}

int ct_emit_transfers(ct_context* c, const ct_record* recs, uint64_t n, int on_device, const ct_config* cfg,
                      int64_t* rows, uint64_t row_cap, uint64_t* n_rows) {
  if (!c || !cfg || !n_rows || (n && !recs)) return fail(c, CT_ERR_ARGUMENT, "null argument");
  CTX_TRY(c, cudaSetDevice(c->device));
  cudaStream_t st = c->stream;
  const ct_record* d_recs = recs;
  if (!on_device && n) {
    size_t cap = c->in_cap;
    if (ensure(c, c->in_buf, cap, n)) return CT_ERR_CUDA;
    c->in_cap = cap;
    CTX_TRY(c, cudaMemcpyAsync(c->in_buf, recs, n * sizeof(ct_record), cudaMemcpyHostToDevice, st));
    d_recs = c->in_buf;
  }
  ExpandParams ex{};
  ex.tree_threshold = cfg->tree_threshold;
  ex.ring_len = cfg->ring_len > 0 ? cfg->ring_len : -1;
  ex.ring_valid = 1;
  if (cfg->ring_len > 0) {
    const int L = cfg->ring_len;
    std::vector<uint16_t> h(2 * (size_t)L, 0);
    std::vector<int> seen(L, 0);
    for (int k = 0; k < L; k++) {
      uint16_t v = cfg->ring_order[k];
      h[k] = v;
      if (v >= L || seen[v]) ex.ring_valid = 0;
      else { seen[v] = 1; h[L + v] = (uint16_t)k; }
    }
    size_t cap = (size_t)c->ring_cap;
    if (ensure(c, c->ring, cap, 2 * (size_t)L)) return CT_ERR_CUDA;
    c->ring_cap = (int)cap;
    CTX_TRY(c, cudaMemcpyAsync(c->ring, h.data(), 2 * (size_t)L * 2, cudaMemcpyHostToDevice, st));
    ex.ring_order = c->ring;
    ex.ring_inv = c->ring + L;
  }
  uint32_t* counts;
  uint64_t* offs;
  unsigned int* flags;
  CTX_TRY(c, cudaMallocAsync(&counts, (n + 1) * 4, st));
  CTX_TRY(c, cudaMallocAsync(&offs, (n + 1) * 8, st));
  CTX_TRY(c, cudaMallocAsync(&flags, 4, st));
  CTX_TRY(c, cudaMemsetAsync(flags, 0, 4, st));
  CTX_TRY(c, cudaMemsetAsync(counts + n, 0, 4, st));
  launch_emit(d_recs, n, ex, counts, nullptr, nullptr, 0, flags, st);
  size_t tmp = 0;
  void* t = nullptr;
  CTX_TRY(c, cub::DeviceScan::ExclusiveSum(nullptr, tmp, counts, offs, (int64_t)(n + 1), st));
  CTX_TRY(c, cudaMallocAsync(&t, tmp, st));
  CTX_TRY(c, cub::DeviceScan::ExclusiveSum(t, tmp, counts, offs, (int64_t)(n + 1), st));
  uint64_t total = 0;
  unsigned int hflags = 0;
  CTX_TRY(c, cudaMemcpyAsync(&total, offs + n, 8, cudaMemcpyDeviceToHost, st));
  CTX_TRY(c, cudaMemcpyAsync(&hflags, flags, 4, cudaMemcpyDeviceToHost, st));
  CTX_TRY(c, cudaStreamSynchronize(st));
  *n_rows = total;
  int status = CT_OK;
  if (hflags & F_BAD_RING) status = CT_ERR_INVALID_CONFIG;
  else if (hflags & F_WRONG_ALGO) status = CT_ERR_WRONG_ALGORITHM;
  else if (hflags & F_MISSING_ROOT) status = CT_ERR_MISSING_ROOT;
  if (status == CT_OK && rows && row_cap >= total && total) {
    int64_t* d_rows;
    CTX_TRY(c, cudaMallocAsync(&d_rows, total * 7 * 8, st));
    launch_emit(d_recs, n, ex, counts, offs, d_rows, 1, flags, st);
    CTX_TRY(c, cudaMemcpyAsync(rows, d_rows, total * 7 * 8, cudaMemcpyDeviceToHost, st));
    CTX_TRY(c, cudaStreamSynchronize(st));
    cudaFreeAsync(d_rows, st);
  }
  cudaFreeAsync(t, st);
  cudaFreeAsync(counts, st);
  cudaFreeAsync(offs, st);
  cudaFreeAsync(flags, st);
  CTX_TRY(c, cudaStreamSynchronize(st));
  return status;
}

int ct_generate(ct_context* c, int kind, uint64_t seed, uint64_t first, uint64_t n, ct_record* dev_out,
                void* stream) {
  if (!c || (n && !dev_out)) return fail(c, CT_ERR_ARGUMENT, "null argument");
  CTX_TRY(c, cudaSetDevice(c->device));
  cudaStream_t st = stream ? (cudaStream_t)stream : c->stream;
  int e = generate(kind, seed, first, n, dev_out, st);
  if (e) return fail(c, CT_ERR_ARGUMENT, "unknown generator kind");
  CTX_TRY(c, cudaGetLastError());
  CTX_TRY(c, cudaStreamSynchronize(st));
  return CT_OK;
}

uint64_t ct_generate_boundary(int kind, uint64_t at) { return generate_boundary(kind, at); }

}  // extern "C"

// ------------------------------------------------------------------ multi-GPU partials
// Layout (uint64 words): header[16] | calls[9] pay_lo[9] pay_hi[9] diag[6] |
// tcf[6 * n_comms] | cells[ncell] | freq[ncell] | kExport comm summaries | 1 flag word.
// Header: magic, g2, n_comms, n, flags, max_dev + 1, oor_key, oor_gpu, copy_first[3],
// path, 4 reserved.  A comm summary: comm, n, first / last block head, the records of
// the shard's first and last block of the comm (<= 32 each), p2p first / last seq per
// (rank, send|recv) — what the merge needs to re-check seq order across shards.
namespace {
constexpr uint64_t kPartialMagic = 0x4354503250415254ull;
constexpr int kExport = 16;
constexpr uint64_t kExpWords = 4 + 2 * 32 * 4;  // comm, n, first / last head, 2 x 32 records
constexpr int kExportCh = 64;                    // p2p channel summaries
constexpr uint64_t kChWords = 5;                 // key, first_s, first_r, last_s, last_r
constexpr uint64_t kHdr = 16, kStats = 33;

uint64_t partial_words(int g2, uint32_t n_comms) {
  return kHdr + kStats + 6ull * n_comms + 2ull * kTypes * g2 * g2 + kExport * kExpWords + kExportCh * kChWords + 1;
}

// The unique communicators (<= kExport) and p2p channels (<= kExportCh) of a shard's warp
// ranges, each with its first and last occurrence (lowest / highest warp range), then
// the boundary summaries the merge checks across shards (first / last block records,
// first / last channel seqs).  k_export_scan: every CTA hashes its slice of the warp
// summaries into shared-memory sets and merges them into global ones (a few atomics per
// CTA); k_export_write (one CTA) compacts the global sets into the partial.
constexpr int kTC = 2 * kExport, kTH = 2 * kExportCh;
struct ExpTab {
  unsigned long long ckey[kTC], hkey[kTH];  // ~0: empty
  uint32_t cmin[kTC], hmin[kTH];            // ~0 initially
  uint32_t cmax[kTC], hmax[kTH];            // 0 initially
  uint32_t overflow;
};
constexpr size_t kExpTabFF = offsetof(ExpTab, cmax);  // bytes set to 0xFF, the rest to 0

__device__ int exp_insert(unsigned long long* tab, int cap, unsigned long long key) {
  uint32_t h = (uint32_t)((key * 0x9E3779B97F4A7C15ull) >> 40) % (uint32_t)cap;
  for (int probe = 0; probe < cap; probe++, h = (h + 1) % (uint32_t)cap) {
    const unsigned long long old = atomicCAS(&tab[h], ~0ull, key);
    if (old == ~0ull || old == key) return (int)h;
  }
  return -1;
}

__global__ void __launch_bounds__(256) k_export_scan(const WarpSlot* slots, const Chans chans, uint32_t total_warps,
                                                     ExpTab* g) {
  __shared__ unsigned long long ckey[kTC], hkey[kTH];
  __shared__ uint32_t cmin[kTC], cmax[kTC], hmin[kTH], hmax[kTH];
  __shared__ int ovf;
  const int tid = threadIdx.x;
  for (int i = tid; i < kTC; i += blockDim.x) { ckey[i] = ~0ull; cmin[i] = ~0u; cmax[i] = 0; }
  for (int i = tid; i < kTH; i += blockDim.x) { hkey[i] = ~0ull; hmin[i] = ~0u; hmax[i] = 0; }
  if (tid == 0) ovf = 0;
  __syncthreads();
  const uint64_t ns = (uint64_t)total_warps * kCS, nq = (uint64_t)total_warps * kPC;
  const uint64_t s0 = ns * blockIdx.x / gridDim.x, s1 = ns * (blockIdx.x + 1) / gridDim.x;
  for (uint64_t i = s0 + tid; i < s1; i += blockDim.x) {
    const WarpSlot& x = slots[i];
    if (x.comm == 0xFFFFFFFFu || x.n == 0) continue;
    const int h = exp_insert(ckey, kTC, x.comm);
    if (h < 0) { ovf = 1; continue; }
    atomicMin(&cmin[h], (uint32_t)i);
    atomicMax(&cmax[h], (uint32_t)i);
  }
  const uint64_t q0 = nq * blockIdx.x / gridDim.x, q1 = nq * (blockIdx.x + 1) / gridDim.x;
  for (uint64_t i = q0 + tid; i < q1; i += blockDim.x) {
    const unsigned long long k = chans.key(i);
    if (k == ~0ull) continue;
    const int h = exp_insert(hkey, kTH, k);
    if (h < 0) { ovf = 1; continue; }
    atomicMin(&hmin[h], (uint32_t)i);
    atomicMax(&hmax[h], (uint32_t)i);
  }
  __syncthreads();
  for (int i = tid; i < kTC; i += blockDim.x)
    if (ckey[i] != ~0ull) {
      const int h = exp_insert(g->ckey, kTC, ckey[i]);
      if (h < 0) { ovf = 1; continue; }
      atomicMin(&g->cmin[h], cmin[i]);
      atomicMax(&g->cmax[h], cmax[i]);
    }
  for (int i = tid; i < kTH; i += blockDim.x)
    if (hkey[i] != ~0ull) {
      const int h = exp_insert(g->hkey, kTH, hkey[i]);
      if (h < 0) { ovf = 1; continue; }
      atomicMin(&g->hmin[h], hmin[i]);
      atomicMax(&g->hmax[h], hmax[i]);
    }
  __syncthreads();
  if (tid == 0 && ovf) g->overflow = 1;
}

__global__ void __launch_bounds__(256) k_export_write(const ExpTab* g, const WarpSlot* slots, const Chans chans,
                                                      const ct_record* recs, uint64_t* exp, uint64_t* chx,
                                                      uint64_t* overflow) {
  __shared__ int nc, nh, ovf;
  const int tid = threadIdx.x;
  if (tid == 0) { nc = 0; nh = 0; ovf = g->overflow ? 1 : 0; }
  __syncthreads();
  // compact into the export lists (any order: the merge matches entries by key)
  for (int i = tid; i < kTC; i += blockDim.x)
    if (g->ckey[i] != ~0ull) {
      const int e = atomicAdd(&nc, 1);
      if (e >= kExport) { ovf = 1; continue; }
      const WarpSlot& f = slots[g->cmin[i]];
      const WarpSlot& l = slots[g->cmax[i]];
      uint64_t* o = exp + e * kExpWords;
      o[0] = g->ckey[i];
      o[1] = f.n;
      o[2] = f.coll_first;
      o[3] = l.coll_last;
      if (f.n <= 32) {
        ct_record* fr = reinterpret_cast<ct_record*>(o + 4);
        ct_record* lr = reinterpret_cast<ct_record*>(o + 4 + 32 * 4);
        for (uint32_t r = 0; r < f.n; r++) { fr[r] = recs[f.coll_first + r]; lr[r] = recs[l.coll_last + r]; }
      }
    }
  for (int i = tid; i < kTH; i += blockDim.x)
    if (g->hkey[i] != ~0ull) {
      const int e = atomicAdd(&nh, 1);
      if (e >= kExportCh) { ovf = 1; continue; }
      uint64_t* o = chx + e * kChWords;
      o[0] = g->hkey[i];
      o[1] = chans.first_s(g->hmin[i]);
      o[2] = chans.first_r(g->hmin[i]);
      o[3] = chans.last_s(g->hmax[i]);
      o[4] = chans.last_r(g->hmax[i]);
    }
  __syncthreads();
  if (tid == 0 && ovf) *overflow = 1;
}

__global__ void k_merge_partials(const uint64_t* parts, int world, uint64_t words, int g2, uint32_t n_comms,
                                 unsigned long long* cells, unsigned long long* tcf, GlobalState* gs,
                                 unsigned long long* info) {
  const uint64_t o_tcf = kHdr + kStats;
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x, stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j = tid; j < 6ull * n_comms; j += stride) {
    uint64_t best = ~0ull, base = 0;
    for (int w = 0; w < world; w++) {
      const uint64_t v = parts[w * words + o_tcf + j];
      if (v != ~0ull && v + base < best) best = v + base;
      base += parts[w * words + 3];
    }
    tcf[j] = best;
  }
  if (tid == 0) {
    // every partial: a ct partial of this layout (info[1]: 1 not a partial, 2 layouts
    // differ); info[0]: records over all shards
    unsigned long long n_all = 0, bad = 0;
    for (int w = 0; w < world; w++) {
      const uint64_t* p = parts + w * words;
      if (p[0] != kPartialMagic) bad |= 1;
      else if (p[1] != (uint64_t)g2 || p[2] != n_comms) bad |= 2;
      n_all += p[3];
    }
    info[0] = n_all;
    info[1] = bad;
    GlobalState g{};
    g.max_dev = -1;
    g.oor_key = ~0ull;
    g.of_cell = ~0ull;
    for (int k = 0; k < 3; k++) g.copy_first[k] = ~0ull;
    uint64_t base = 0;
    for (int w = 0; w < world; w++) {
      const uint64_t* p = parts + w * words;
      g.flags |= (uint32_t)p[4];
      if (p[11] != 1) g.flags |= F_NONCANON;  // every shard must have taken the fast path
      if (p[words - 1]) g.flags |= F_NONCANON;  // comm summary overflow
      g.max_dev = max(g.max_dev, (int)p[5] - 1);
      if (p[6] != ~0ull) {
        const uint64_t k = p[6] + (base << 21);
        if (k < g.oor_key) { g.oor_key = k; g.err_index = p[7]; }
      }
      for (int k = 0; k < 3; k++)
        if (p[8 + k] != ~0ull && p[8 + k] + base < g.copy_first[k]) g.copy_first[k] = p[8 + k] + base;
      for (int t = 0; t < kTypes; t++) {
        g.calls[t] += p[kHdr + t];
        const unsigned long long old = g.pay_lo[t];
        g.pay_lo[t] = old + p[kHdr + 9 + t];
        g.pay_hi[t] += p[kHdr + 18 + t] + (g.pay_lo[t] < old ? 1 : 0);
      }
      for (int k = 0; k < CT_NDIAG; k++) g.diag[k] += p[kHdr + 27 + k];
      base += p[3];
    }
    g.flags |= gs->flags;  // k_merge_order ran before this kernel
    *gs = g;
  }
}

__global__ void k_merge_cells(const uint64_t* parts, int world, uint64_t words, int g2, uint32_t n_comms,
                              unsigned long long* cells, GlobalState* gs) {
  const uint64_t ncell = (uint64_t)kTypes * g2 * g2;
  const uint64_t o_cells = kHdr + kStats + 6ull * n_comms;
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < 2 * ncell; j += (uint64_t)gridDim.x * blockDim.x) {
    unsigned __int128 s = 0;
    for (int w = 0; w < world; w++) s += parts[w * words + o_cells + j];
    if (s >> 64) { atomicOr(&gs->flags, F_OVERFLOW); s = ~0ull; }
    cells[j] = (unsigned long long)s;
  }
}

// shard-boundary order: for every (shard v, summary) with a first element, the nearest
// earlier shard holding the same chain must end before it
__global__ void k_merge_order(const uint64_t* parts, int world, uint64_t words, uint64_t o_exp, GlobalState* gs) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int per = kExport + kExportCh;
  if (t >= world * per) return;
  const int v = t / per, e = t % per;
  if (v == 0) return;
  const uint64_t o_ch = o_exp + kExport * kExpWords;
  if (e < kExport) {
    const uint64_t* me = parts + v * words + o_exp + e * kExpWords;
    if (me[0] == ~0ull || !me[1]) return;
    for (int w = v - 1; w >= 0; w--)
      for (int q = 0; q < kExport; q++) {
        const uint64_t* o = parts + w * words + o_exp + q * kExpWords;
        if (o[0] != me[0] || !o[1]) continue;
        bool ok = o[1] == me[1] && me[1] <= 32;
        const ct_record* lr = reinterpret_cast<const ct_record*>(o + 4 + 32 * 4);
        const ct_record* fr = reinterpret_cast<const ct_record*>(me + 4);
        for (uint64_t r = 0; ok && r < me[1]; r++) ok = lr[r].seq < fr[r].seq;
        if (!ok) atomicOr(&gs->flags, F_NONCANON);
        return;
      }
    return;
  }
  const uint64_t* me = parts + v * words + o_ch + (e - kExport) * kChWords;
  if (me[0] == ~0ull) return;
  for (int w = v - 1; w >= 0; w--)
    for (int q = 0; q < kExportCh; q++) {
      const uint64_t* o = parts + w * words + o_ch + q * kChWords;
      if (o[0] != me[0]) continue;
      if (me[1] < o[3] || me[2] < o[4]) atomicOr(&gs->flags, F_NONCANON);
      return;
    }
}
}  // namespace

extern "C" {

int ct_partial_size(ct_context* c, uint64_t* words) {
  if (!c || !words) return fail(c, CT_ERR_ARGUMENT, "null argument");
  *words = partial_words(c->last_g2, c->last_comms);
  return CT_OK;
}

int ct_partial_export(ct_context* c, uint64_t* dev_out, uint64_t words, void* stream) {
  if (!c || !dev_out) return fail(c, CT_ERR_ARGUMENT, "null argument");
  const int g2 = c->last_g2;
  const uint32_t nc = c->last_comms;
  if (words != partial_words(g2, nc)) return fail(c, CT_ERR_ARGUMENT, "partial size mismatch");
  CTX_TRY(c, cudaSetDevice(c->device));
  cudaStream_t st = stream ? (cudaStream_t)stream : c->stream;
  const GlobalState& gs = c->last_state;
  const uint64_t ncell = (uint64_t)kTypes * g2 * g2;
  std::vector<uint64_t> hdr(kHdr + kStats, 0);
  hdr[0] = kPartialMagic;
  hdr[1] = (uint64_t)g2;
  hdr[2] = nc;
  hdr[3] = c->last_n;
  hdr[4] = gs.flags;
  hdr[5] = (uint64_t)(gs.max_dev + 1);
  hdr[6] = gs.oor_key;
  hdr[7] = (c->last.status == CT_ERR_ENDPOINT_RANGE) ? c->last.err_aux[0] : 0;
  for (int k = 0; k < 3; k++) hdr[8 + k] = gs.copy_first[k];
  hdr[11] = (uint64_t)c->last.path;
  for (int t = 0; t < kTypes; t++) {
    hdr[kHdr + t] = gs.calls[t];
    hdr[kHdr + 9 + t] = gs.pay_lo[t];
    hdr[kHdr + 18 + t] = gs.pay_hi[t];
  }
  for (int k = 0; k < CT_NDIAG; k++) hdr[kHdr + 27 + k] = c->last.diag[k];
  if (c->shard.valid && c->last_input == c->shard.part) {
    // a routed part (ct_shard_*): the diagnostics of records that never reach a part
    // (incomplete groups, unmatched p2p: counted once, on rank 0) and d over ALL records
    hdr[kHdr + 27 + CT_DIAG_INCOMPLETE] += c->shard.extra_diag[0];
    hdr[kHdr + 27 + CT_DIAG_UNMATCHED_SEND] += c->shard.extra_diag[1];
    hdr[kHdr + 27 + CT_DIAG_UNMATCHED_RECV] += c->shard.extra_diag[2];
    hdr[5] = std::max<uint64_t>(hdr[5], (uint64_t)(c->shard.global_max_dev + 1));
  }
  const uint64_t o_tcf = kHdr + kStats, o_cells = o_tcf + 6ull * nc, o_exp = o_cells + 2 * ncell;
  CTX_TRY(c, cudaMemcpyAsync(dev_out, hdr.data(), hdr.size() * 8, cudaMemcpyHostToDevice, st));
  CTX_TRY(c, cudaMemcpyAsync(dev_out + o_tcf, c->tcf, 6ull * nc * 8, cudaMemcpyDeviceToDevice, st));
  CTX_TRY(c, cudaMemcpyAsync(dev_out + o_cells, c->cells, 2 * ncell * 8, cudaMemcpyDeviceToDevice, st));
  CTX_TRY(c, cudaMemsetAsync(dev_out + o_exp, 0xFF, (kExport * kExpWords + kExportCh * kChWords) * 8, st));
  CTX_TRY(c, cudaMemsetAsync(dev_out + words - 1, 0, 8, st));
  if (c->last.path == 1 && c->last_total_warps) {
    uint64_t* chx = dev_out + o_exp + kExport * kExpWords;
    if (ensure(c, c->exp_tab, c->exp_tab_cap, sizeof(ExpTab))) return CT_ERR_CUDA;
    ExpTab* g = reinterpret_cast<ExpTab*>(c->exp_tab);
    CTX_TRY(c, cudaMemsetAsync(c->exp_tab, 0xFF, kExpTabFF, st));
    CTX_TRY(c, cudaMemsetAsync(c->exp_tab + kExpTabFF, 0, sizeof(ExpTab) - kExpTabFF, st));
    const Chans ch{c->chans, (uint64_t)c->last_total_warps * kPC};
    const unsigned grid = (unsigned)std::min<uint64_t>((uint64_t)c->num_sms, std::max<uint64_t>(1, c->last_total_warps / 8));
    k_export_scan<<<grid, 256, 0, st>>>(c->slots, ch, c->last_total_warps, g);
    k_export_write<<<1, 256, 0, st>>>(g, c->slots, ch, c->last_input, dev_out + o_exp, chx, dev_out + words - 1);
    CTX_TRY(c, cudaGetLastError());
  }
  return CT_OK;
}

int ct_partial_merge(ct_context* c, const uint64_t* dev_in, int world, uint64_t words, ct_summary* out,
                     void* stream) {
  if (!c || !dev_in || !out || world < 1) return fail(c, CT_ERR_ARGUMENT, "bad argument");
  CTX_TRY(c, cudaSetDevice(c->device));
  cudaStream_t st = stream ? (cudaStream_t)stream : c->stream;
  // the layout is this rank's own (every rank analysed with the same d / dev_hint and
  // comm count); the merge kernel checks every partial against it on the device, so the
  // whole merge costs one host round trip
  const int g2 = c->last_g2;
  const uint32_t nc = c->last_comms;
  if (g2 < 3 || words != partial_words(g2, nc)) return fail(c, CT_ERR_ARGUMENT, "partial size mismatch");
  const uint64_t ncell = (uint64_t)kTypes * g2 * g2;
  size_t cap = c->cells_cap;
  if (ensure(c, c->cells, cap, 2 * ncell)) return CT_ERR_CUDA;
  c->cells_cap = cap;
  cap = c->tcf_cap;
  if (ensure(c, c->tcf, cap, 6ull * nc)) return CT_ERR_CUDA;
  c->tcf_cap = cap;
  if (ensure(c, c->exp_tab, c->exp_tab_cap, sizeof(ExpTab) + 16)) return CT_ERR_CUDA;
  unsigned long long* info = reinterpret_cast<unsigned long long*>(c->exp_tab + ((sizeof(ExpTab) + 7) & ~7ull));
  memset(out, 0, sizeof *out);
  CTX_TRY(c, cudaEventRecord(c->ev[2], st));
  CTX_TRY(c, cudaMemsetAsync(c->st, 0, sizeof(GlobalState), st));
  const uint64_t o_exp = kHdr + kStats + 6ull * nc + 2 * ncell;
  k_merge_order<<<(world * (kExport + kExportCh) + 255) / 256, 256, 0, st>>>(dev_in, world, words, o_exp, c->st);
  k_merge_partials<<<1, 256, 0, st>>>(dev_in, world, words, g2, nc, c->cells, c->tcf, c->st, info);
  k_merge_cells<<<64, 256, 0, st>>>(dev_in, world, words, g2, nc, c->cells, c->st);
  CTX_TRY(c, cudaGetLastError());
  GlobalState gs;
  unsigned long long hinfo[2];
  std::vector<unsigned long long> h_tcf(6 * (size_t)nc), h_cells(2 * ncell);
  CTX_TRY(c, cudaMemcpyAsync(&gs, c->st, sizeof gs, cudaMemcpyDeviceToHost, st));
  CTX_TRY(c, cudaMemcpyAsync(hinfo, info, sizeof hinfo, cudaMemcpyDeviceToHost, st));
  CTX_TRY(c, cudaMemcpyAsync(h_tcf.data(), c->tcf, h_tcf.size() * 8, cudaMemcpyDeviceToHost, st));
  CTX_TRY(c, cudaMemcpyAsync(h_cells.data(), c->cells, h_cells.size() * 8, cudaMemcpyDeviceToHost, st));
  CTX_TRY(c, cudaEventRecord(c->ev[3], st));
  CTX_TRY(c, cudaStreamSynchronize(st));
  if (hinfo[1] & 1) return fail(c, CT_ERR_ARGUMENT, "not a ct partial");
  if (hinfo[1] & 2)
    return fail(c, CT_ERR_ARGUMENT, "partials disagree on layout (use the same d / dev_hint on every rank)");
  if (gs.flags & F_NONCANON)
    return fail(c, CT_ERR_NOT_CANONICAL, "sharded analysis needs the canonical layout in every shard and across shard boundaries");
  const int gcap = g2 - 2;
  const int64_t d = c->last_explicit ? c->last.d : (int64_t)gs.max_dev + 1;
  const uint64_t extra[3] = {0, 0, 0};
  if (int e = summarize_state(c, gs, gcap, d, 1, extra, nullptr, nc, st, out, h_tcf.data(), h_cells.data())) return e;
  out->n_records = hinfo[0];
  CTX_TRY(c, cudaEventElapsedTime(&out->ms_total, c->ev[2], c->ev[3]));
  out->n_launches = 3;
  c->last = *out;
  return out->status;
}

}  // extern "C"

// ------------------------------------------------------------------ multi-GPU, any layout
extern "C" {

int ct_shard_words(int32_t n_comms, uint64_t* meta_words, uint64_t* count_words) {
  if (!meta_words || !count_words || n_comms < 1) return CT_ERR_ARGUMENT;
  *meta_words = shard_meta_words((uint32_t)n_comms);
  *count_words = shard_count_words();
  return CT_OK;
}

static int shard_status(ct_context* c, int e, const char* where) {
  if (e == 0) return CT_OK;
  if (e == kCanonUnsupported)
    return fail(c, CT_ERR_NOT_CANONICAL, std::string(where) + ": trace outside the sharded canonicaliser's scope");
  return cuda_fail(c, (cudaError_t)e, where);
}

int ct_shard_meta(ct_context* c, const ct_record* recs, uint64_t n, int32_t n_comms, uint64_t* dev_out, void* stream) {
  if (!c || !dev_out || (n && !recs) || n_comms < 1) return fail(c, CT_ERR_ARGUMENT, "bad argument");
  CTX_TRY(c, cudaSetDevice(c->device));
  cudaStream_t st = stream ? (cudaStream_t)stream : c->stream;
  return shard_status(c, shard_meta(recs, n, (uint32_t)n_comms, c->num_sms, st, dev_out), "ct_shard_meta");
}

int ct_shard_count(ct_context* c, const ct_record* recs, uint64_t n, int32_t n_comms, const uint64_t* dev_metas,
                   int world, uint64_t* dev_out, void* stream) {
  if (!c || !dev_out || !dev_metas || world < 1 || (n && !recs) || n_comms < 1)
    return fail(c, CT_ERR_ARGUMENT, "bad argument");
  CTX_TRY(c, cudaSetDevice(c->device));
  cudaStream_t st = stream ? (cudaStream_t)stream : c->stream;
  return shard_status(c, shard_count(&c->shard, recs, n, (uint32_t)n_comms, dev_metas, world, c->num_sms, st, dev_out),
                      "ct_shard_count");
}

int ct_shard_route(ct_context* c, int32_t n_comms, const uint64_t* dev_metas, const uint64_t* dev_counts, int world,
                   int rank, uint64_t* dev_out_pos, ct_record* dev_out_rec, uint64_t* send_counts,
                   uint64_t* recv_counts, uint64_t* part_len, void* stream) {
  if (!c || !dev_metas || !dev_counts || world < 1 || rank < 0 || rank >= world || !send_counts || !recv_counts ||
      !part_len || n_comms < 1)
    return fail(c, CT_ERR_ARGUMENT, "bad argument");
  CTX_TRY(c, cudaSetDevice(c->device));
  cudaStream_t st = stream ? (cudaStream_t)stream : c->stream;
  return shard_status(c, shard_route(&c->shard, (uint32_t)n_comms, dev_metas, dev_counts, world, rank, c->num_sms, st,
                                     dev_out_pos, dev_out_rec, send_counts, recv_counts, part_len),
                      "ct_shard_route");
}

int ct_shard_assemble(ct_context* c, const uint64_t* dev_in_pos, const ct_record* dev_in_rec, uint64_t n_in,
                      ct_record* dev_part, void* stream) {
  if (!c || (n_in && (!dev_in_pos || !dev_in_rec)) || !dev_part) return fail(c, CT_ERR_ARGUMENT, "bad argument");
  CTX_TRY(c, cudaSetDevice(c->device));
  cudaStream_t st = stream ? (cudaStream_t)stream : c->stream;
  return shard_status(c, shard_assemble(&c->shard, dev_in_pos, dev_in_rec, n_in, dev_part, st), "ct_shard_assemble");
}

}  // extern "C"

extern "C" int ct_element_boundary(ct_context* c, const ct_record* recs, uint64_t n, int on_device, uint64_t at,
                                   uint64_t* out) {
  if (!c || !out || (n && !recs)) return fail(c, CT_ERR_ARGUMENT, "null argument");
  if (at >= n) { *out = n; return CT_OK; }
  const uint64_t k = std::min<uint64_t>(64, n - at);
  ct_record buf[64];
  if (on_device) {
    CTX_TRY(c, cudaSetDevice(c->device));
    CTX_TRY(c, cudaMemcpyAsync(buf, recs + at, k * sizeof(ct_record), cudaMemcpyDeviceToHost, c->stream));
    CTX_TRY(c, cudaStreamSynchronize(c->stream));
  } else {
    memcpy(buf, recs + at, k * sizeof(ct_record));
  }
  for (uint64_t i = 0; i < k; i++) {
    const int kind = buf[i].kc & 7;
    if ((kind == CT_KIND_COLLECTIVE && buf[i].rank == 0) || kind == CT_KIND_SEND ||
        (kind >= CT_KIND_MEMCPY && kind <= CT_KIND_ZEROCOPY)) {
      *out = at + i;
      return CT_OK;
    }
  }
  if (at + k == n) { *out = n; return CT_OK; }
  return fail(c, CT_ERR_NOT_CANONICAL, "no element start within 64 records");
}
