// Exact path: device sort-based join (see ct_exact.cuh).
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include "ct_exact.cuh"

namespace ct {

namespace {

constexpr uint64_t kNone = ~0ull;

#define CT_TRY(x)                                  \
  do {                                             \
    cudaError_t e_ = (x);                          \
    if (e_ != cudaSuccess) return (int)e_;         \
  } while (0)

__global__ void k_classify(const ct_record* recs, uint64_t n, uint8_t* fc, uint8_t* fp, uint8_t* fx) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const int kind = recs[i].kc & 7;
    fc[i] = kind == CT_KIND_COLLECTIVE;
    fp[i] = kind == CT_KIND_SEND || kind == CT_KIND_RECV;
    fx[i] = kind >= CT_KIND_MEMCPY;
  }
}

__global__ void k_first_coll(const ct_record* recs, const uint64_t* idx, uint64_t m,
                             unsigned long long* first) {
  // per comm: the smallest record index.  Lanes of one comm combine first (one atomic per
  // comm per warp), and an atomic is skipped when the cell already holds a smaller index.
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t p0 = blockIdx.x * (uint64_t)blockDim.x; p0 < m; p0 += stride) {
    const uint64_t p = p0 + (threadIdx.x & ~31u) + (threadIdx.x & 31u);
    const bool act = p < m;
    const uint64_t i = act ? idx[p] : ~0ull;
    const uint32_t c = act ? recs[i].comm : 0xFFFFFFFFu;
    if (__all_sync(0xFFFFFFFFu, __match_any_sync(0xFFFFFFFFu, c) == 0xFFFFFFFFu)) {  // one comm: warp minimum
      unsigned long long mn = i;
      for (int o = 16; o; o >>= 1) {
        const unsigned long long x = __shfl_xor_sync(0xFFFFFFFFu, mn, o);
        mn = x < mn ? x : mn;
      }
      if ((threadIdx.x & 31u) == 0 && act && mn < first[c]) atomicMin(first + c, mn);
    } else if (act && i < first[c]) {
      atomicMin(first + c, (unsigned long long)i);
    }
  }
}

__global__ void k_nranks_check(const ct_record* recs, const uint64_t* idx, uint64_t m,
                               const unsigned long long* first, unsigned long long* bad) {
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < m;
       p += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i = idx[p];
    const uint64_t f = first[recs[i].comm];
    if (recs[i].nranks != recs[f].nranks) atomicMin(bad, (unsigned long long)i);
  }
}

__global__ void k_keys_seq(const ct_record* recs, const uint64_t* idx, uint64_t m, uint64_t* keys) {
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < m;
       p += (uint64_t)gridDim.x * blockDim.x)
    keys[p] = recs[idx[p]].seq;
}

__global__ void k_keys_comm_rank(const ct_record* recs, const uint64_t* idx, uint64_t m, uint64_t* keys) {
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < m;
       p += (uint64_t)gridDim.x * blockDim.x) {
    const ct_record& r = recs[idx[p]];
    keys[p] = ((uint64_t)r.comm << 16) | r.rank;
  }
}

// p2p channel key: comm | src | dst | is_recv (decompose.py:350-353)
__global__ void k_keys_channel(const ct_record* recs, const uint64_t* idx, uint64_t m, uint64_t* keys) {
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < m;
       p += (uint64_t)gridDim.x * blockDim.x) {
    const ct_record& r = recs[idx[p]];
    const bool recv = (r.kc & 7) == CT_KIND_RECV;
    const uint64_t src = recv ? r.aux : r.rank, dst = recv ? r.rank : r.aux;
    keys[p] = ((uint64_t)r.comm << 33) | (src << 17) | (dst << 1) | (recv ? 1 : 0);
  }
}

// segment heads of (comm, rank) streams in the sorted order, duplicate seq detection
__global__ void k_stream_heads(const ct_record* recs, const uint64_t* idx, uint64_t m,
                               uint64_t* headpos, unsigned long long* n_dup) {
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < m;
       p += (uint64_t)gridDim.x * blockDim.x) {
    const ct_record& r = recs[idx[p]];
    bool head = p == 0;
    if (!head) {
      const ct_record& q = recs[idx[p - 1]];
      head = q.comm != r.comm || q.rank != r.rank;
      if (!head && q.seq == r.seq) atomicAdd(n_dup, 1ull);
    }
    headpos[p] = head ? p : 0;
  }
}

__global__ void k_stream_first(const uint64_t* idx, const uint64_t* seg, uint64_t m,
                               unsigned long long* seg_first) {
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < m;
       p += (uint64_t)gridDim.x * blockDim.x)
    atomicMin(seg_first + seg[p], (unsigned long long)idx[p]);
}

// reference precedence of the duplicate-seq error: comm first-seen order, then the
// rank's first-seen order within the comm, then the smallest duplicated seq
// (grouping.py:114-123).  ``stage`` selects which key is being minimised.
__global__ void k_dup_select(const ct_record* recs, const uint64_t* idx, const uint64_t* seg,
                             uint64_t m, const unsigned long long* first_coll,
                             const unsigned long long* seg_first, unsigned long long* best, int stage) {
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < m;
       p += (uint64_t)gridDim.x * blockDim.x) {
    if (p == 0 || seg[p] == p) continue;
    const ct_record& r = recs[idx[p]];
    const ct_record& q = recs[idx[p - 1]];
    if (q.comm != r.comm || q.rank != r.rank || q.seq != r.seq) continue;
    const uint64_t k1 = first_coll[r.comm], k2 = seg_first[seg[p]], k3 = r.seq;
    if (stage == 0) atomicMin(best, (unsigned long long)k1);
    else if (stage == 1) { if (k1 == best[0]) atomicMin(best + 1, (unsigned long long)k2); }
    else if (k1 == best[0] && k2 == best[1]) atomicMin(best + 2, (unsigned long long)k3);
  }
}

__global__ void k_group_keys(const ct_record* recs, const uint64_t* idx, const uint64_t* seg,
                             uint64_t m, const uint32_t* comm_rank, uint64_t* keys) {
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < m;
       p += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t ordinal = p - seg[p];
    keys[p] = ((uint64_t)comm_rank[recs[idx[p]].comm] << 32) | ordinal;
  }
}

__global__ void k_fill_u64(unsigned long long* a, uint64_t n, unsigned long long v) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    a[i] = v;
}

__global__ void k_iota_u32(uint32_t* a, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    a[i] = (uint32_t)i;
}

__global__ void k_comm_rank(const uint32_t* sorted_comms, uint64_t n, uint32_t* comm_rank) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n;
       j += (uint64_t)gridDim.x * blockDim.x)
    comm_rank[sorted_comms[j]] = (uint32_t)j;
}

// per group run: emitted length (n if complete), status for materialisation
__global__ void k_group_runs(const ct_record* recs, const uint64_t* idx, const uint64_t* run_off,
                             const int64_t* run_len, const uint64_t* n_runs, uint64_t* emit_len,
                             uint64_t* status, unsigned long long* n_incomplete) {
  const uint64_t R = *n_runs;
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < R; k += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t off = run_off[k];
    const uint64_t len = (uint64_t)run_len[k];
    const ct_record& h = recs[idx[off]];
    const bool complete = len == h.nranks;
    emit_len[k] = complete ? len : 0;
    uint64_t st = CT_DIAG_INCOMPLETE + 1;
    if (!complete) {
      atomicAdd(n_incomplete, 1ull);
    } else {
      bool incompat = false, dup = false;
      for (uint64_t a = 0; a < len && !incompat; a++) {
        const ct_record& q = recs[idx[off + a]];
        if ((q.kc & 0x78) != (h.kc & 0x78) || (q.ad & 0x3F) != (h.ad & 0x3F) || q.count != h.count ||
            (((h.kc >> 6) & 1) && q.aux != h.aux))
          incompat = true;
      }
      for (uint64_t a = 0; a < len && !dup && !incompat; a++)
        for (uint64_t b = a + 1; b < len; b++)
          if (recs[idx[off + a]].dev == recs[idx[off + b]].dev) { dup = true; break; }
      st = incompat ? CT_DIAG_INCOMPATIBLE + 1 : dup ? CT_DIAG_DUPLICATE_DEVICE + 1 : 0;
    }
    status[k] = st;
  }
}

__global__ void k_emit_groups(const ct_record* recs, const uint64_t* idx, const uint64_t* run_off,
                              const int64_t* run_len, const uint64_t* n_runs, const uint64_t* emit_off,
                              const uint64_t* emit_len, ct_record* out, uint64_t* src_map) {
  const uint64_t R = *n_runs;
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < R; k += (uint64_t)gridDim.x * blockDim.x) {
    if (!emit_len[k]) continue;
    const uint64_t off = run_off[k], len = (uint64_t)run_len[k], o = emit_off[k];
    for (uint64_t a = 0; a < len; a++) {
      out[o + a] = recs[idx[off + a]];
      if (src_map) src_map[o + a] = idx[off + a];
    }
  }
}

// p2p channel runs: pair the k-th send with the k-th recv of each channel
__global__ void k_p2p_runs(const uint64_t* ukey, const int64_t* run_len, const uint64_t* n_runs,
                           uint64_t* emit_len, unsigned long long* n_us, unsigned long long* n_ur) {
  const uint64_t R = *n_runs;
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < R; k += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t key = ukey[k];
    uint64_t s = 0, r = 0;
    emit_len[k] = 0;
    if ((key & 1) == 0) {
      s = run_len[k];
      if (k + 1 < R && ukey[k + 1] == (key | 1)) r = run_len[k + 1];
    } else {
      if (k > 0 && ukey[k - 1] == (key & ~1ull)) continue;  // counted with its send run
      r = run_len[k];
    }
    const uint64_t pairs = s < r ? s : r;
    if (s > pairs) atomicAdd(n_us, (unsigned long long)(s - pairs));
    if (r > pairs) atomicAdd(n_ur, (unsigned long long)(r - pairs));
    if ((key & 1) == 0) emit_len[k] = 2 * pairs;
  }
}

__global__ void k_emit_pairs(const ct_record* recs, const uint64_t* idx, const uint64_t* run_off,
                             const int64_t* run_len, const uint64_t* n_runs, const uint64_t* emit_off,
                             const uint64_t* emit_len, uint64_t base, uint64_t n_pairs, ct_record* out,
                             uint64_t* src_map) {
  // one thread per emitted pair: its channel run is the last run whose output offset is
  // <= 2j (runs are laid out back to back in emit_off order)
  const uint64_t R = *n_runs;
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n_pairs;
       j += (uint64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = (int64_t)R - 1;
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) / 2;
      if (emit_off[mid] <= 2 * j) lo = mid; else hi = mid - 1;
    }
    const int64_t k = lo;
    const uint64_t local = j - emit_off[k] / 2, soff = run_off[k], roff = run_off[k + 1];
    const uint64_t o = base + 2 * j;
    out[o] = recs[idx[soff + local]];
    out[o + 1] = recs[idx[roff + local]];
    if (src_map) { src_map[o] = idx[soff + local]; src_map[o + 1] = idx[roff + local]; }
  }
}

// materialisation: count/dtype disagreement of every FIFO pair (decompose.py:362)
__global__ void k_pair_mismatch(const ct_record* recs, const uint64_t* idx, const uint64_t* run_off,
                                const uint64_t* emit_len, const uint64_t* n_runs, uint8_t* mis,
                                const uint64_t* emit_off) {
  const uint64_t R = *n_runs;
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < R; k += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t pairs = emit_len[k] / 2, soff = run_off[k], roff = run_off[k + 1];
    for (uint64_t j = 0; j < pairs; j++) {
      const ct_record& a = recs[idx[soff + j]];
      const ct_record& b = recs[idx[roff + j]];
      mis[emit_off[k] / 2 + j] = a.count != b.count || ((a.ad >> 2) & 15) != ((b.ad >> 2) & 15);
    }
  }
}

__global__ void k_gather(const ct_record* recs, const uint64_t* idx, uint64_t m, uint64_t base,
                         ct_record* out, uint64_t* src_map) {
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < m;
       p += (uint64_t)gridDim.x * blockDim.x) {
    out[base + p] = recs[idx[p]];
    if (src_map) src_map[base + p] = idx[p];
  }
}

struct Pool {
  cudaStream_t st;
  std::vector<void*> bufs;
  template <typename T>
  T* get(uint64_t count) {
    void* p = nullptr;
    if (cudaMallocAsync(&p, (count ? count : 1) * sizeof(T), st) != cudaSuccess) return nullptr;
    bufs.push_back(p);
    return static_cast<T*>(p);
  }
  ~Pool() {
    for (void* p : bufs) cudaFreeAsync(p, st);
  }
};

inline int grid_for(uint64_t n) {
  uint64_t g = (n + 255) / 256;
  return (int)(g < 1 ? 1 : (g > 4096 ? 4096 : g));
}

template <typename T>
T read1(const T* d, cudaStream_t st) {
  T h{};
  cudaMemcpyAsync(&h, d, sizeof(T), cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  return h;
}

// stable LSD sort of (keys, vals): CUB radix sort is stable
int sort_pairs(Pool& pool, const uint64_t* kin, uint64_t* kout, const uint64_t* vin, uint64_t* vout,
               uint64_t m, int end_bit) {
  size_t tmp = 0;
  CT_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tmp, kin, kout, vin, vout, m, 0, end_bit, pool.st));
  void* t = pool.get<uint8_t>(tmp);
  if (!t) return (int)cudaErrorMemoryAllocation;
  CT_TRY(cub::DeviceRadixSort::SortPairs(t, tmp, kin, kout, vin, vout, m, 0, end_bit, pool.st));
  return 0;
}

int select_flagged(Pool& pool, const uint8_t* flags, uint64_t n, uint64_t* out, uint64_t* count_host) {
  uint64_t* d_num = pool.get<uint64_t>(1);
  size_t tmp = 0;
  thrust::counting_iterator<uint64_t> it(0);
  CT_TRY(cub::DeviceSelect::Flagged(nullptr, tmp, it, flags, out, d_num, (int64_t)n, pool.st));
  void* t = pool.get<uint8_t>(tmp);
  if (!t) return (int)cudaErrorMemoryAllocation;
  CT_TRY(cub::DeviceSelect::Flagged(t, tmp, it, flags, out, d_num, (int64_t)n, pool.st));
  *count_host = read1(d_num, pool.st);
  return 0;
}

// run-length encoding of sorted keys with 64-bit item and run counts (CUB's
// DeviceRunLengthEncode takes an int item count): run heads are flagged and selected
// (64-bit DeviceSelect), giving the unique keys, run lengths and run offsets at once
__global__ void k_run_heads(const uint64_t* keys, uint64_t m, uint8_t* flag) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x)
    flag[i] = i == 0 || keys[i] != keys[i - 1];
}

__global__ void k_run_fill(const uint64_t* keys, const uint64_t* heads, const uint64_t* n_runs, uint64_t m,
                           uint64_t* uniq, int64_t* lens) {
  const uint64_t R = *n_runs;
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < R; k += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t h = heads[k], nx = k + 1 < R ? heads[k + 1] : m;
    uniq[k] = keys[h];
    lens[k] = (int64_t)(nx - h);
  }
}


int rle(Pool& pool, const uint64_t* keys, uint64_t m, uint64_t* uniq, int64_t* lens, uint64_t* offs,
        uint64_t* d_runs, uint64_t* runs_host) {
  uint8_t* flag = pool.get<uint8_t>(m);
  if (!flag) return (int)cudaErrorMemoryAllocation;
  k_run_heads<<<grid_for(m), 256, 0, pool.st>>>(keys, m, flag);
  size_t tmp = 0;
  thrust::counting_iterator<uint64_t> it(0);
  CT_TRY(cub::DeviceSelect::Flagged(nullptr, tmp, it, flag, offs, d_runs, (int64_t)m, pool.st));
  void* t = pool.get<uint8_t>(tmp);
  if (!t) return (int)cudaErrorMemoryAllocation;
  CT_TRY(cub::DeviceSelect::Flagged(t, tmp, it, flag, offs, d_runs, (int64_t)m, pool.st));
  k_run_fill<<<grid_for(m), 256, 0, pool.st>>>(keys, offs, d_runs, m, uniq, lens);
  CT_TRY(cudaMemcpyAsync(runs_host, d_runs, 8, cudaMemcpyDeviceToHost, pool.st));
  CT_TRY(cudaStreamSynchronize(pool.st));
  return 0;
}

template <typename In, typename Out>
int excl_sum(Pool& pool, In in, Out out, uint64_t m) {
  size_t tmp = 0;
  CT_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, (int64_t)m, pool.st));
  void* t = pool.get<uint8_t>(tmp);
  if (!t) return (int)cudaErrorMemoryAllocation;
  CT_TRY(cub::DeviceScan::ExclusiveSum(t, tmp, in, out, (int64_t)m, pool.st));
  return 0;
}

struct MaxOp {
  __device__ __forceinline__ uint64_t operator()(uint64_t a, uint64_t b) const { return a > b ? a : b; }
};

}  // namespace

int exact_canonicalize(const ct_record* recs, uint64_t n, uint32_t n_comms, cudaStream_t st,
                       bool materialize, ExactResult* res) {
  Pool pool{st, {}};
  uint32_t L = 0;
  uint8_t* fc = pool.get<uint8_t>(n);
  uint8_t* fp = pool.get<uint8_t>(n);
  uint8_t* fx = pool.get<uint8_t>(n);
  if (!fc || !fp || !fx) return (int)cudaErrorMemoryAllocation;
  k_classify<<<grid_for(n), 256, 0, st>>>(recs, n, fc, fp, fx); L++;
  uint64_t nc = 0, np = 0, nx = 0;
  uint64_t* cidx = pool.get<uint64_t>(n);
  uint64_t* pidx = pool.get<uint64_t>(n);
  uint64_t* xidx = pool.get<uint64_t>(n);
  int e;
  if ((e = select_flagged(pool, fc, n, cidx, &nc))) return e;
  if ((e = select_flagged(pool, fp, n, pidx, &np))) return e;
  if ((e = select_flagged(pool, fx, n, xidx, &nx))) return e;
  L += 6;

  // ---- collectives: nranks agreement per comm (grouping.py:97-109)
  unsigned long long* first_coll = pool.get<unsigned long long>(n_comms ? n_comms : 1);
  unsigned long long* bad = pool.get<unsigned long long>(4);
  k_fill_u64<<<grid_for(n_comms), 256, 0, st>>>(first_coll, n_comms, kNone);
  k_fill_u64<<<1, 32, 0, st>>>(bad, 4, kNone);
  L += 2;
  if (nc) {
    k_first_coll<<<grid_for(nc), 256, 0, st>>>(recs, cidx, nc, first_coll);
    k_nranks_check<<<grid_for(nc), 256, 0, st>>>(recs, cidx, nc, first_coll, bad);
    L += 2;
    const uint64_t b = read1(bad, st);
    if (b != kNone) {
      ct_record rb, rf;
      cudaMemcpyAsync(&rb, recs + b, sizeof rb, cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      uint64_t f = 0;
      cudaMemcpyAsync(&f, first_coll + rb.comm, sizeof f, cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      cudaMemcpyAsync(&rf, recs + f, sizeof rf, cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      res->fatal = CT_ERR_INVARIANT;
      res->fatal_kind = 1;
      res->err_index = b;
      res->err_aux[0] = rb.comm;
      res->err_aux[1] = rf.nranks;
      res->err_aux[2] = rb.nranks;
      res->launches = L;
      return 0;
    }
  }

  uint64_t coll_total = 0;
  uint64_t* order = nullptr;  // collectives sorted by (comm, rank, seq)
  uint64_t* seg = nullptr;
  if (nc) {
    uint64_t* k1 = pool.get<uint64_t>(nc);
    uint64_t* k2 = pool.get<uint64_t>(nc);
    uint64_t* v1 = pool.get<uint64_t>(nc);
    order = pool.get<uint64_t>(nc);
    k_keys_seq<<<grid_for(nc), 256, 0, st>>>(recs, cidx, nc, k1);
    if ((e = sort_pairs(pool, k1, k2, cidx, v1, nc, 64))) return e;
    k_keys_comm_rank<<<grid_for(nc), 256, 0, st>>>(recs, v1, nc, k1);
    if ((e = sort_pairs(pool, k1, k2, v1, order, nc, 48))) return e;
    L += 4;
    // ---- ordinals and duplicate seq (grouping.py:115-123)
    uint64_t* headpos = pool.get<uint64_t>(nc);
    seg = pool.get<uint64_t>(nc);
    unsigned long long* ndup = pool.get<unsigned long long>(1);
    cudaMemsetAsync(ndup, 0, 8, st);
    k_stream_heads<<<grid_for(nc), 256, 0, st>>>(recs, order, nc, headpos, ndup);
    {
      size_t tmp = 0;
      CT_TRY(cub::DeviceScan::InclusiveScan(nullptr, tmp, headpos, seg, MaxOp{}, (int64_t)nc, st));
      void* t = pool.get<uint8_t>(tmp);
      CT_TRY(cub::DeviceScan::InclusiveScan(t, tmp, headpos, seg, MaxOp{}, (int64_t)nc, st));
    }
    L += 2;
    if (read1(ndup, st)) {
      unsigned long long* seg_first = pool.get<unsigned long long>(nc);
      k_fill_u64<<<grid_for(nc), 256, 0, st>>>(seg_first, nc, kNone);
      k_stream_first<<<grid_for(nc), 256, 0, st>>>(order, seg, nc, seg_first);
      for (int stage = 0; stage < 3; stage++)
        k_dup_select<<<grid_for(nc), 256, 0, st>>>(recs, order, seg, nc, first_coll, seg_first, bad, stage);
      unsigned long long best[3];
      cudaMemcpyAsync(best, bad, sizeof best, cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      ct_record rr;
      cudaMemcpyAsync(&rr, recs + best[1], sizeof rr, cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      res->fatal = CT_ERR_INVARIANT;
      res->fatal_kind = 2;
      res->err_index = best[1];
      res->err_aux[0] = rr.comm;
      res->err_aux[1] = rr.rank;
      res->err_aux[2] = best[2];
      res->launches = L + 5;
      return 0;
    }
    // ---- groups by (comm first-seen rank, ordinal)
    uint64_t* csort_k = pool.get<uint64_t>(n_comms);
    uint32_t* cids = pool.get<uint32_t>(n_comms);
    uint32_t* cids_sorted = pool.get<uint32_t>(n_comms);
    uint32_t* comm_rank = pool.get<uint32_t>(n_comms);
    k_iota_u32<<<grid_for(n_comms), 256, 0, st>>>(cids, n_comms);
    {
      size_t tmp = 0;
      CT_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tmp, (const uint64_t*)first_coll, csort_k, cids,
                                             cids_sorted, (uint64_t)n_comms, 0, 64, st));
      void* t = pool.get<uint8_t>(tmp);
      CT_TRY(cub::DeviceRadixSort::SortPairs(t, tmp, (const uint64_t*)first_coll, csort_k, cids,
                                             cids_sorted, (uint64_t)n_comms, 0, 64, st));
    }
    k_comm_rank<<<grid_for(n_comms), 256, 0, st>>>(cids_sorted, n_comms, comm_rank);
    if (nc >> 32) return kExactCapacity;  // ordinals are 32-bit in the group key
    k_group_keys<<<grid_for(nc), 256, 0, st>>>(recs, order, seg, nc, comm_rank, k1);
    uint64_t* gorder = pool.get<uint64_t>(nc);
    if ((e = sort_pairs(pool, k1, k2, order, gorder, nc, 64))) return e;
    L += 5;
    uint64_t* ukey = pool.get<uint64_t>(nc);
    int64_t* rlen = pool.get<int64_t>(nc);
    uint64_t* d_runs = pool.get<uint64_t>(1);
    uint64_t* roff = pool.get<uint64_t>(nc + 1);
    uint64_t R = 0;
    if ((e = rle(pool, k2, nc, ukey, rlen, roff, d_runs, &R))) return e;
    uint64_t* elen = pool.get<uint64_t>(R + 1);
    uint64_t* eoff = pool.get<uint64_t>(R + 1);
    uint64_t* gstat = pool.get<uint64_t>(R + 1);
    unsigned long long* ninc = pool.get<unsigned long long>(1);
    cudaMemsetAsync(ninc, 0, 8, st);
    k_group_runs<<<grid_for(R), 256, 0, st>>>(recs, gorder, roff, rlen, d_runs, elen, gstat, ninc);
    cudaMemsetAsync(elen + R, 0, 8, st);
    if ((e = excl_sum(pool, elen, eoff, R + 1))) return e;
    coll_total = read1(eoff + R, st);
    res->n_incomplete = read1(ninc, st);
    L += 4;
    order = gorder;
    // stash for emission below
    res->canon = nullptr;
    // canonical buffer sized after p2p counting; emit groups now into a temp
    ct_record* tmp_out = pool.get<ct_record>(coll_total);
    uint64_t* tmp_map = materialize ? pool.get<uint64_t>(coll_total) : nullptr;
    k_emit_groups<<<grid_for(R), 256, 0, st>>>(recs, gorder, roff, rlen, d_runs, eoff, elen, tmp_out, tmp_map);
    L++;
    if (materialize) {
      std::vector<uint64_t> h_roff(R), h_len(R), h_stat(R), h_ukey(R), h_members(nc);
      std::vector<int64_t> h_rlen(R);
      cudaMemcpyAsync(h_roff.data(), roff, R * 8, cudaMemcpyDeviceToHost, st);
      cudaMemcpyAsync(h_rlen.data(), rlen, R * 8, cudaMemcpyDeviceToHost, st);
      cudaMemcpyAsync(h_stat.data(), gstat, R * 8, cudaMemcpyDeviceToHost, st);
      cudaMemcpyAsync(h_ukey.data(), ukey, R * 8, cudaMemcpyDeviceToHost, st);
      cudaMemcpyAsync(h_members.data(), gorder, nc * 8, cudaMemcpyDeviceToHost, st);
      std::vector<uint32_t> h_sorted(n_comms);
      cudaMemcpyAsync(h_sorted.data(), cids_sorted, (size_t)n_comms * 4, cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      res->members = h_members;
      for (uint64_t k = 0; k < R; k++) {
        GroupRow g;
        g.comm = h_sorted[h_ukey[k] >> 32];
        g.ordinal = h_ukey[k] & 0xFFFFFFFFull;
        g.status = h_stat[k];
        g.n_members = (uint64_t)h_rlen[k];
        g.member_off = h_roff[k];
        res->groups.push_back(g);
      }
    }
    // keep tmp_out alive by moving it into a persistent allocation below
    res->m = coll_total;
    res->canon = tmp_out;  // provisional; replaced below
    res->canon_src.clear();
    if (tmp_map) {
      res->canon_src.resize(coll_total);
      cudaMemcpyAsync(res->canon_src.data(), tmp_map, coll_total * 8, cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
    }
  }
  ct_record* coll_out = res->canon;
  res->canon = nullptr;

  // ---- p2p: FIFO pairing per channel (decompose.py:342-394)
  uint64_t pair_total = 0;
  ct_record* pair_out = nullptr;
  std::vector<uint64_t> pair_map;
  if (np) {
    uint64_t* k1 = pool.get<uint64_t>(np);
    uint64_t* k2 = pool.get<uint64_t>(np);
    uint64_t* v1 = pool.get<uint64_t>(np);
    uint64_t* v2 = pool.get<uint64_t>(np);
    k_keys_seq<<<grid_for(np), 256, 0, st>>>(recs, pidx, np, k1);
    if ((e = sort_pairs(pool, k1, k2, pidx, v1, np, 64))) return e;
    k_keys_channel<<<grid_for(np), 256, 0, st>>>(recs, v1, np, k1);
    if ((e = sort_pairs(pool, k1, k2, v1, v2, np, 64))) return e;
    uint64_t* ukey = pool.get<uint64_t>(np);
    int64_t* rlen = pool.get<int64_t>(np);
    uint64_t* d_runs = pool.get<uint64_t>(1);
    uint64_t* roff = pool.get<uint64_t>(np + 1);
    uint64_t R = 0;
    if ((e = rle(pool, k2, np, ukey, rlen, roff, d_runs, &R))) return e;
    uint64_t* elen = pool.get<uint64_t>(R + 1);
    uint64_t* eoff = pool.get<uint64_t>(R + 1);
    unsigned long long* nus = pool.get<unsigned long long>(2);
    cudaMemsetAsync(nus, 0, 16, st);
    k_p2p_runs<<<grid_for(R), 256, 0, st>>>(ukey, rlen, d_runs, elen, nus, nus + 1);
    cudaMemsetAsync(elen + R, 0, 8, st);
    if ((e = excl_sum(pool, elen, eoff, R + 1))) return e;
    pair_total = read1(eoff + R, st);
    unsigned long long hu[2];
    cudaMemcpyAsync(hu, nus, 16, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    res->n_unmatched_send = hu[0];
    res->n_unmatched_recv = hu[1];
    pair_out = pool.get<ct_record>(pair_total);
    uint64_t* pmap = materialize ? pool.get<uint64_t>(pair_total) : nullptr;
    k_emit_pairs<<<grid_for(pair_total / 2), 256, 0, st>>>(recs, v2, roff, rlen, d_runs, eoff, elen, 0, pair_total / 2,
                                                          pair_out, pmap);
    L += 9;
    if (materialize) {
      // every p2p diagnostic, reference order is restored on the host
      uint8_t* d_mis = pool.get<uint8_t>(pair_total / 2 + 1);
      k_pair_mismatch<<<grid_for(R), 256, 0, st>>>(recs, v2, roff, elen, d_runs, d_mis, eoff);
      std::vector<uint8_t> h_mis(pair_total / 2 + 1);
      std::vector<uint64_t> h_eoff(R);
      cudaMemcpyAsync(h_mis.data(), d_mis, pair_total / 2 + 1, cudaMemcpyDeviceToHost, st);
      cudaMemcpyAsync(h_eoff.data(), eoff, R * 8, cudaMemcpyDeviceToHost, st);
      std::vector<uint64_t> h_ukey(R), h_roff(R), h_v(np);
      std::vector<int64_t> h_rlen(R);
      cudaMemcpyAsync(h_ukey.data(), ukey, R * 8, cudaMemcpyDeviceToHost, st);
      cudaMemcpyAsync(h_roff.data(), roff, R * 8, cudaMemcpyDeviceToHost, st);
      cudaMemcpyAsync(h_rlen.data(), rlen, R * 8, cudaMemcpyDeviceToHost, st);
      cudaMemcpyAsync(h_v.data(), v2, np * 8, cudaMemcpyDeviceToHost, st);
      if (pmap) {
        pair_map.resize(pair_total);
        cudaMemcpyAsync(pair_map.data(), pmap, pair_total * 8, cudaMemcpyDeviceToHost, st);
      }
      cudaStreamSynchronize(st);
      for (uint64_t k = 0; k < R; k++) {
        const uint64_t key = h_ukey[k];
        uint64_t s = 0, r = 0, so = 0, ro = 0;
        if ((key & 1) == 0) {
          s = h_rlen[k]; so = h_roff[k];
          if (k + 1 < R && h_ukey[k + 1] == (key | 1)) { r = h_rlen[k + 1]; ro = h_roff[k + 1]; }
        } else {
          if (k > 0 && h_ukey[k - 1] == (key & ~1ull)) continue;
          r = h_rlen[k]; ro = h_roff[k];
        }
        const uint64_t comm = key >> 33, src = (key >> 17) & 0xFFFF, dst = (key >> 1) & 0xFFFF;
        const uint64_t pairs = s < r ? s : r;
        for (uint64_t j = 0; j < pairs; j++)  // matched pairs are rows too (reason CT_NDIAG)
          res->p2p_diags.push_back({h_mis[h_eoff[k] / 2 + j] ? (uint64_t)CT_DIAG_MISMATCHED_P2P : (uint64_t)CT_NDIAG,
                                    comm, src, dst, j, h_v[so + j], h_v[ro + j]});
        for (uint64_t j = pairs; j < s; j++)
          res->p2p_diags.push_back({(uint64_t)CT_DIAG_UNMATCHED_SEND, comm, src, dst, j, h_v[so + j], kNone});
        for (uint64_t j = pairs; j < r; j++)
          res->p2p_diags.push_back({(uint64_t)CT_DIAG_UNMATCHED_RECV, comm, src, dst, j, kNone, h_v[ro + j]});
      }
    }
  }

  // ---- assemble canonical stream
  const uint64_t m = coll_total + pair_total + nx;
  ct_record* canon = nullptr;
  CT_TRY(cudaMallocAsync(&canon, (m ? m : 1) * sizeof(ct_record), st));
  if (coll_total) CT_TRY(cudaMemcpyAsync(canon, coll_out, coll_total * sizeof(ct_record), cudaMemcpyDeviceToDevice, st));
  if (pair_total) CT_TRY(cudaMemcpyAsync(canon + coll_total, pair_out, pair_total * sizeof(ct_record), cudaMemcpyDeviceToDevice, st));
  uint64_t* xmap = (materialize && nx) ? pool.get<uint64_t>(nx) : nullptr;
  if (nx) { k_gather<<<grid_for(nx), 256, 0, st>>>(recs, xidx, nx, coll_total + pair_total, canon, nullptr); L++; }
  if (materialize) {
    res->canon_src.resize(m);
    if (pair_total)
      std::copy(pair_map.begin(), pair_map.end(), res->canon_src.begin() + coll_total);
    if (nx) {
      std::vector<uint64_t> hx(nx);
      cudaMemcpyAsync(hx.data(), xidx, nx * 8, cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      std::copy(hx.begin(), hx.end(), res->canon_src.begin() + coll_total + pair_total);
    }
  }
  (void)xmap;
  res->canon = canon;
  res->m = m;
  res->launches = L;
  CT_TRY(cudaGetLastError());
  return 0;
}

}  // namespace ct
