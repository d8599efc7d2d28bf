// Counting canonicaliser: capture-layout traces (ranks interleaved, as an LD_PRELOAD
// interposer writes them, one O_APPEND line per call per process) -> the canonical
// stream the fast kernel takes, in three streaming passes instead of the exact path's
// radix sorts.
//
// The reference groups collectives by (comm, ordinal), the ordinal being a record's
// position in its (comm, rank) stream sorted by seq (grouping.py:82-183), and pairs
// sends with recvs FIFO per (comm, src, dst) channel in seq order (decompose.py:342-394).
// In a capture every process appends its own calls in call order, so per (comm, rank)
// file order IS seq order: the ordinal is a running count.  This path assumes exactly
// that and never checks it itself -- the fast kernel re-checks per (comm, rank) strictly
// increasing seq (and per channel non-decreasing seq) on the canonical stream it writes,
// so a trace breaking the assumption is rejected there and takes the exact path.
//
//   k_meta    one read: max nranks, comm first-seen index, nranks per comm, max device
//   k_count   per tile (a warp's contiguous chunk) a histogram of keys: (comm, rank) for
//             collectives, (comm, src, dst) channel for sends and for recvs, one key for
//             copies; one exclusive scan over [key][tile] gives every tile's starting
//             ordinal per key
//   k_scatter per record: ordinal = tile start + rank among equal keys in the batch
//             (__match_any_sync); destination = key base + ordinal * stride, written as
//             [complete groups (comm first-seen, ordinal), ranks consecutive]
//             [matched pairs per channel (comm, src, dst), FIFO][copies in file order]
// Incomplete groups and unmatched sends / recvs are counted (the same diagnostics the
// exact path reports) and dropped.  Traces whose key space does not fit (many comms or
// ranks), whose nranks disagree within a comm (a fatal error the exact path reports
// with the reference's message) or with malformed records fall back to the exact path.
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "ct_canon.cuh"

namespace ct {

namespace {

constexpr int kMetaThreads = 256;
constexpr uint32_t kMaxKeys = 4096;     // per-warp shared counters (16 KB)
constexpr int kCanonWarps = 4;          // warps per CTA in the count / scatter passes
constexpr uint32_t kMaxMetaComms = 1024;

struct Meta {
  unsigned int nmax;  // max nranks over collective / p2p records
  unsigned int bad;   // a record the canonical layout cannot express
  int max_dev;        // max device id (dev, copy GPU endpoints)
  unsigned int pad;
};

__device__ __forceinline__ uint32_t key_of(const uint4& b, uint32_t nmax, uint32_t kc, uint32_t kh) {
  const uint32_t kind = (b.w >> 16) & 7u, comm = b.x, rank = b.y >> 16, peer = b.z >> 16;
  if (kind == CT_KIND_COLLECTIVE) return comm * nmax + rank;
  if (kind == CT_KIND_SEND) return kc + (comm * nmax + rank) * nmax + peer;
  if (kind == CT_KIND_RECV) return kc + kh + (comm * nmax + peer) * nmax + rank;
  return kc + 2 * kh;  // copies
}

// Blocked ranges (CTA b owns [b*span, (b+1)*span)) so first-seen indices fit 32 bits per
// CTA; per-comm minima / maxima in shared memory, flushed once per CTA.
__global__ void __launch_bounds__(kMetaThreads) k_meta(const ct_record* recs, uint64_t n, uint64_t span,
                                                       uint32_t n_comms, Meta* meta, unsigned int* nr_min,
                                                       unsigned int* nr_max, unsigned long long* cfirst) {
  __shared__ unsigned int s_min[kMaxMetaComms], s_max[kMaxMetaComms], s_first[kMaxMetaComms];
  for (uint32_t c = threadIdx.x; c < n_comms; c += blockDim.x) {
    s_min[c] = 0xFFFFFFFFu; s_max[c] = 0; s_first[c] = 0xFFFFFFFFu;
  }
  __syncthreads();
  const uint64_t lo = blockIdx.x * span, hi = min(n, lo + span);
  unsigned int nmax = 0, bad = 0;
  int max_dev = -1;
  uint32_t last_comm = 0xFFFFFFFFu;  // this thread's last collective comm (skip repeated shared atomics)
  uint32_t last_nr = 0;
  for (uint64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    const uint4 b = __ldg(reinterpret_cast<const uint4*>(recs + i) + 1);
    const uint32_t kind = (b.w >> 16) & 7u, comm = b.x, nr = b.y & 0xFFFFu, rank = b.y >> 16;
    const uint32_t dev = b.z & 0xFFFFu, aux = b.z >> 16, aux2 = b.w & 0xFFFFu;
    max_dev = max(max_dev, (int)dev);
    if (kind <= CT_KIND_RECV) {
      if (comm >= n_comms || nr == 0 || rank >= nr || (kind != CT_KIND_COLLECTIVE && (aux >= nr || aux == rank))) bad = 1;
      nmax = max(nmax, nr);
      if (kind == CT_KIND_COLLECTIVE && comm < n_comms) {
        if (comm != last_comm || nr != last_nr) {
          atomicMin(&s_min[comm], nr);
          atomicMax(&s_max[comm], nr);
          last_comm = comm;
          last_nr = nr;
        }
        const uint32_t off = (uint32_t)(i - lo);
        if (off < s_first[comm]) atomicMin(&s_first[comm], off);
      }
    } else if (kind <= CT_KIND_ZEROCOPY) {
      const uint32_t ck = b.w >> 30;
      if (ck != CT_CKIND_H2D) max_dev = max(max_dev, (int)aux);
      if (ck != CT_CKIND_D2H) max_dev = max(max_dev, (int)aux2);
    } else {
      bad = 1;
    }
  }
  __syncthreads();
  for (uint32_t c = threadIdx.x; c < n_comms; c += blockDim.x) {
    if (s_max[c]) {
      atomicMin(&nr_min[c], s_min[c]);
      atomicMax(&nr_max[c], s_max[c]);
    }
    if (s_first[c] != 0xFFFFFFFFu) atomicMin(&cfirst[c], (unsigned long long)(lo + s_first[c]));
  }
  nmax = __reduce_max_sync(0xFFFFFFFFu, nmax);
  bad = __reduce_or_sync(0xFFFFFFFFu, bad);
  for (int o = 16; o; o >>= 1) max_dev = max(max_dev, __shfl_xor_sync(0xFFFFFFFFu, max_dev, o));
  if ((threadIdx.x & 31) == 0) {
    if (nmax) atomicMax(&meta->nmax, nmax);
    if (bad) atomicOr(&meta->bad, bad);
    atomicMax(&meta->max_dev, max_dev);
  }
}

// per tile: key histogram -> counts[key * T + tile]
__global__ void __launch_bounds__(32 * kCanonWarps) k_count(const ct_record* recs, uint64_t n, uint64_t chunk,
                                                           uint64_t T, uint32_t K, uint32_t nmax, uint32_t kc,
                                                           uint32_t kh, uint32_t* counts) {
  extern __shared__ unsigned int smem_cnt[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned int* cnt = smem_cnt + (size_t)warp * K;
  const uint64_t W = (uint64_t)gridDim.x * kCanonWarps;
  for (uint64_t t = (uint64_t)blockIdx.x * kCanonWarps + warp; t < T; t += W) {
    for (uint32_t k = lane; k < K; k += 32) cnt[k] = 0;
    __syncwarp();
    const uint64_t lo = t * chunk, hi = min(n, lo + chunk);
    for (uint64_t i = lo + lane; i < hi; i += 32) {
      const uint4 b = __ldg(reinterpret_cast<const uint4*>(recs + i) + 1);
      atomicAdd(&cnt[key_of(b, nmax, kc, kh)], 1u);
    }
    __syncwarp();
    for (uint32_t k = lane; k < K; k += 32) counts[(uint64_t)k * T + t] = cnt[k];
    __syncwarp();
  }
}

__global__ void k_key_totals(const uint32_t* counts, const uint64_t* offs, uint64_t T, uint32_t K, uint64_t* base,
                             uint64_t* total) {
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < K; k += gridDim.x * blockDim.x) {
    const uint64_t b = offs[(uint64_t)k * T];
    base[k] = b;
    total[k] = offs[(uint64_t)k * T + T - 1] + counts[(uint64_t)k * T + T - 1] - b;
  }
}

struct Dest {  // key -> canonical position of ordinal o: pos + o * stride when o < limit
  unsigned long long pos;
  unsigned long long limit;
  unsigned long long stride;
};

__global__ void __launch_bounds__(32 * kCanonWarps) k_scatter(const ct_record* recs, uint64_t n, uint64_t chunk,
                                                             uint64_t T, uint32_t K, uint32_t nmax, uint32_t kc,
                                                             uint32_t kh, const uint64_t* offs, const uint64_t* base,
                                                             const Dest* dest, ct_record* out) {
  extern __shared__ unsigned int smem_run[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1;
  unsigned int* run = smem_run + (size_t)warp * K;
  const uint64_t W = (uint64_t)gridDim.x * kCanonWarps;
  for (uint64_t t = (uint64_t)blockIdx.x * kCanonWarps + warp; t < T; t += W) {
    for (uint32_t k = lane; k < K; k += 32) run[k] = (unsigned int)(offs[(uint64_t)k * T + t] - base[k]);
    __syncwarp();
    const uint64_t lo = t * chunk, hi = min(n, lo + chunk);
    for (uint64_t i0 = lo; i0 < hi; i0 += 32) {
      const uint64_t i = i0 + lane;
      const bool act = i < hi;
      uint4 a = make_uint4(0, 0, 0, 0), b = a;
      if (act) {
        const uint4* p = reinterpret_cast<const uint4*>(recs + i);
        a = __ldg(p);
        b = __ldg(p + 1);
      }
      const uint32_t key = act ? key_of(b, nmax, kc, kh) : 0x80000000u | (uint32_t)lane;
      const unsigned m = __match_any_sync(0xFFFFFFFFu, key);
      const uint32_t ord = act ? run[key] + __popc(m & lt) : 0u;
      __syncwarp();
      if (act && (m >> lane) == 1u) run[key] += __popc(m);
      __syncwarp();
      if (act) {
        const Dest d = dest[key];
        if (ord < d.limit) {
          uint4* o = reinterpret_cast<uint4*>(out + d.pos + (uint64_t)ord * d.stride);
          o[0] = a;
          o[1] = b;
        }
      }
    }
    __syncwarp();
  }
}

template <typename T>
T* dalloc(uint64_t count, cudaStream_t st) {
  T* p = nullptr;
  if (cudaMallocAsync(&p, (count ? count : 1) * sizeof(T), st) != cudaSuccess) return nullptr;
  return p;
}

}  // namespace

int count_canonicalize(const ct_record* recs, uint64_t n, uint32_t n_comms, int num_sms, cudaStream_t st,
                       ExactResult* res, int* max_dev) {
  if (n == 0 || n >= (1ull << 32) || n_comms > kMaxMetaComms) return kCanonUnsupported;
  uint32_t L = 0;
  std::vector<void*> scratch;
  auto cleanup = [&]() {
    for (void* p : scratch) cudaFreeAsync(p, st);
  };
  // ---- pass 1: meta
  Meta* meta = dalloc<Meta>(1, st);
  unsigned int* nr_min = dalloc<unsigned int>(n_comms, st);
  unsigned int* nr_max = dalloc<unsigned int>(n_comms, st);
  unsigned long long* cfirst = dalloc<unsigned long long>(n_comms, st);
  scratch.insert(scratch.end(), {meta, nr_min, nr_max, cfirst});
  if (!meta || !nr_min || !nr_max || !cfirst) { cleanup(); return (int)cudaErrorMemoryAllocation; }
  Meta m0{0, 0, -1, 0};
  cudaMemcpyAsync(meta, &m0, sizeof m0, cudaMemcpyHostToDevice, st);
  cudaMemsetAsync(nr_min, 0xFF, n_comms * 4, st);
  cudaMemsetAsync(nr_max, 0, n_comms * 4, st);
  cudaMemsetAsync(cfirst, 0xFF, n_comms * 8, st);
  const uint64_t blocks = std::min<uint64_t>((uint64_t)num_sms * 8, (n + 4095) / 4096);
  const uint64_t span = (n + blocks - 1) / blocks;
  k_meta<<<(unsigned)blocks, kMetaThreads, 0, st>>>(recs, n, span, n_comms, meta, nr_min, nr_max, cfirst);
  L++;
  Meta hm;
  std::vector<unsigned int> h_min(n_comms), h_max(n_comms);
  std::vector<unsigned long long> h_first(n_comms);
  cudaMemcpyAsync(&hm, meta, sizeof hm, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(h_min.data(), nr_min, n_comms * 4, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(h_max.data(), nr_max, n_comms * 4, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(h_first.data(), cfirst, n_comms * 8, cudaMemcpyDeviceToHost, st);
  if (cudaError_t e = cudaStreamSynchronize(st)) { cleanup(); return (int)e; }
  if (hm.bad) { cleanup(); return kCanonUnsupported; }
  for (uint32_t c = 0; c < n_comms; c++)
    if (h_max[c] && h_min[c] != h_max[c]) { cleanup(); return kCanonUnsupported; }  // nranks disagreement
  const uint32_t nmax = std::max(hm.nmax, 1u);
  const uint64_t kc = (uint64_t)n_comms * nmax, kh = (uint64_t)n_comms * nmax * nmax;
  const uint64_t K64 = kc + 2 * kh + 1;
  if (K64 > kMaxKeys) { cleanup(); return kCanonUnsupported; }
  const uint32_t K = (uint32_t)K64;
  // ---- pass 2: per-tile key counts, one exclusive scan over [key][tile]
  uint64_t chunk = 1024;
  while ((n + chunk - 1) / chunk * (uint64_t)K > (64ull << 20)) chunk *= 2;  // <= 64M counters
  const uint64_t T = (n + chunk - 1) / chunk;
  uint32_t* counts = dalloc<uint32_t>(T * K, st);
  uint64_t* offs = dalloc<uint64_t>(T * K, st);
  uint64_t* kbase = dalloc<uint64_t>(K, st);
  uint64_t* ktot = dalloc<uint64_t>(K, st);
  scratch.insert(scratch.end(), {counts, offs, kbase, ktot});
  if (!counts || !offs || !kbase || !ktot) { cleanup(); return (int)cudaErrorMemoryAllocation; }
  const size_t smem = (size_t)kCanonWarps * K * 4;
  const uint64_t ctas = std::min<uint64_t>((uint64_t)num_sms * 8, (T + kCanonWarps - 1) / kCanonWarps);
  cudaFuncSetAttribute(k_count, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_count<<<(unsigned)ctas, 32 * kCanonWarps, smem, st>>>(recs, n, chunk, T, K, nmax, (uint32_t)kc, (uint32_t)kh,
                                                          counts);
  L++;
  {
    size_t tmp = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp, counts, offs, (int64_t)(T * K), st);
    void* t = dalloc<uint8_t>(tmp, st);
    scratch.push_back(t);
    if (!t) { cleanup(); return (int)cudaErrorMemoryAllocation; }
    if (cudaError_t e = cub::DeviceScan::ExclusiveSum(t, tmp, counts, offs, (int64_t)(T * K), st)) { cleanup(); return (int)e; }
    L++;
  }
  k_key_totals<<<(K + 255) / 256, 256, 0, st>>>(counts, offs, T, K, kbase, ktot);
  L++;
  std::vector<uint64_t> tot(K);
  cudaMemcpyAsync(tot.data(), ktot, K * 8, cudaMemcpyDeviceToHost, st);
  if (cudaError_t e = cudaStreamSynchronize(st)) { cleanup(); return (int)e; }
  // ---- host: layout of the canonical stream (group_collectives / match_p2p order)
  std::vector<Dest> dest(K, Dest{0, 0, 1});
  uint64_t pos = 0, n_incomplete = 0, n_us = 0, n_ur = 0;
  std::vector<uint32_t> corder;
  for (uint32_t c = 0; c < n_comms; c++)
    if (h_first[c] != ~0ull) corder.push_back(c);
  std::sort(corder.begin(), corder.end(), [&](uint32_t a, uint32_t b) { return h_first[a] < h_first[b]; });
  for (uint32_t c : corder) {
    const uint32_t nc = h_max[c];
    uint64_t lo = ~0ull, hi = 0;
    for (uint32_t r = 0; r < nc; r++) {
      lo = std::min(lo, tot[(uint64_t)c * nmax + r]);
      hi = std::max(hi, tot[(uint64_t)c * nmax + r]);
    }
    n_incomplete += hi - lo;  // groups k in [lo, hi) miss at least one rank
    for (uint32_t r = 0; r < nc; r++) dest[(uint64_t)c * nmax + r] = Dest{pos + r, lo, nc};
    pos += lo * nc;
  }
  for (uint64_t ch = 0; ch < kh; ch++) {  // channels in (comm id, src, dst) order
    const uint64_t s = tot[kc + ch], r = tot[kc + kh + ch], p = std::min(s, r);
    n_us += s - p;
    n_ur += r - p;
    dest[kc + ch] = Dest{pos, p, 2};
    dest[kc + kh + ch] = Dest{pos + 1, p, 2};
    pos += 2 * p;
  }
  const uint64_t n_copies = tot[K - 1];
  dest[K - 1] = Dest{pos, n_copies, 1};
  pos += n_copies;
  const uint64_t m = pos;
  // ---- pass 3: scatter
  Dest* d_dest = dalloc<Dest>(K, st);
  ct_record* canon = dalloc<ct_record>(m, st);
  scratch.push_back(d_dest);
  if (!d_dest || !canon) {
    if (canon) cudaFreeAsync(canon, st);
    cleanup();
    return (int)cudaErrorMemoryAllocation;
  }
  cudaMemcpyAsync(d_dest, dest.data(), K * sizeof(Dest), cudaMemcpyHostToDevice, st);
  k_scatter<<<(unsigned)ctas, 32 * kCanonWarps, smem, st>>>(recs, n, chunk, T, K, nmax, (uint32_t)kc, (uint32_t)kh,
                                                            offs, kbase, d_dest, canon);
  L++;
  cleanup();
  if (cudaError_t e = cudaGetLastError()) { cudaFreeAsync(canon, st); return (int)e; }
  res->canon = canon;
  res->m = m;
  res->n_incomplete = n_incomplete;
  res->n_unmatched_send = n_us;
  res->n_unmatched_recv = n_ur;
  res->launches = L;
  *max_dev = hm.max_dev;
  return 0;
}

}  // namespace ct
