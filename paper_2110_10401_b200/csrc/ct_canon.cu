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
constexpr uint32_t kMaxKeys = 4096;     // per-warp shared counters (16 KB; 32 KB of running ordinals)
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

// k_meta and k_count in one read: the key histograms use a guessed key stride ``nmax``
// (the largest nranks of a sample); a record with more ranks sets meta->bad bit 1 and
// the host reruns k_count with the true stride.  Per-comm nranks / first-seen minima
// live in shared memory and are flushed once per CTA.
__global__ void __launch_bounds__(32 * kCanonWarps) k_count_meta(const ct_record* recs, uint64_t n, uint64_t chunk,
                                                                uint64_t T, uint32_t K, uint32_t nmax, uint32_t kc,
                                                                uint32_t kh, uint32_t* counts, uint32_t n_comms,
                                                                Meta* meta, unsigned int* nr_min, unsigned int* nr_max,
                                                                unsigned long long* cfirst) {
  extern __shared__ unsigned long long smem_cm[];
  unsigned long long* s_first = smem_cm;                                  // [n_comms]
  unsigned int* s_min = reinterpret_cast<unsigned int*>(s_first + n_comms);  // [n_comms]
  unsigned int* s_max = s_min + n_comms;                                  // [n_comms]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned int* cnt = s_max + n_comms + (size_t)warp * K;
  for (uint32_t c = threadIdx.x; c < n_comms; c += blockDim.x) {
    s_min[c] = 0xFFFFFFFFu; s_max[c] = 0; s_first[c] = ~0ull;
  }
  __syncthreads();
  unsigned int nm = 0, bad = 0;
  int max_dev = -1;
  uint32_t last_comm = 0xFFFFFFFFu, last_nr = 0;
  const uint64_t W = (uint64_t)gridDim.x * kCanonWarps;
  for (uint64_t t = (uint64_t)blockIdx.x * kCanonWarps + warp; t < T; t += W) {
    for (uint32_t k = lane; k < K; k += 32) cnt[k] = 0;
    __syncwarp();
    const uint64_t lo = t * chunk, hi = min(n, lo + chunk);
    for (uint64_t i = lo + lane; i < hi; i += 32) {
      const uint4 b = __ldg(reinterpret_cast<const uint4*>(recs + i) + 1);
      const uint32_t kind = (b.w >> 16) & 7u, comm = b.x, nr = b.y & 0xFFFFu, rank = b.y >> 16;
      const uint32_t dev = b.z & 0xFFFFu, aux = b.z >> 16, aux2 = b.w & 0xFFFFu;
      max_dev = max(max_dev, (int)dev);
      bool ok = true;
      if (kind <= CT_KIND_RECV) {
        if (comm >= n_comms || nr == 0 || rank >= nr || (kind != CT_KIND_COLLECTIVE && (aux >= nr || aux == rank))) {
          bad |= 1u;
          ok = false;
        }
        nm = max(nm, nr);
        if (nr > nmax) { bad |= 2u; ok = false; }  // the guessed key stride is too small
        if (kind == CT_KIND_COLLECTIVE && comm < n_comms) {
          if (comm != last_comm || nr != last_nr) {
            atomicMin(&s_min[comm], nr);
            atomicMax(&s_max[comm], nr);
            last_comm = comm;
            last_nr = nr;
          }
          if (i < s_first[comm]) atomicMin(&s_first[comm], (unsigned long long)i);
        }
      } else if (kind <= CT_KIND_ZEROCOPY) {
        const uint32_t ck = b.w >> 30;
        if (ck != CT_CKIND_H2D) max_dev = max(max_dev, (int)aux);
        if (ck != CT_CKIND_D2H) max_dev = max(max_dev, (int)aux2);
      } else {
        bad |= 1u;
        ok = false;
      }
      if (ok) atomicAdd(&cnt[key_of(b, nmax, kc, kh)], 1u);
    }
    __syncwarp();
    for (uint32_t k = lane; k < K; k += 32) counts[(uint64_t)k * T + t] = cnt[k];
    __syncwarp();
  }
  __syncthreads();
  for (uint32_t c = threadIdx.x; c < n_comms; c += blockDim.x) {
    if (s_max[c]) {
      atomicMin(&nr_min[c], s_min[c]);
      atomicMax(&nr_max[c], s_max[c]);
    }
    if (s_first[c] != ~0ull) atomicMin(&cfirst[c], s_first[c]);
  }
  nm = __reduce_max_sync(0xFFFFFFFFu, nm);
  bad = __reduce_or_sync(0xFFFFFFFFu, bad);
  for (int o = 16; o; o >>= 1) max_dev = max(max_dev, __shfl_xor_sync(0xFFFFFFFFu, max_dev, o));
  if (lane == 0) {
    if (nm) atomicMax(&meta->nmax, nm);
    if (bad) atomicOr(&meta->bad, bad);
    atomicMax(&meta->max_dev, max_dev);
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

// MODE 0: write each record to its canonical position; MODE 1: write the position itself
// (gpos[i], ~0 when the record is dropped) for the multi-GPU router.  ``shard_off``
// (MODE 1) adds the ordinals of the same keys held by earlier shards.
template <int MODE>
__global__ void __launch_bounds__(32 * kCanonWarps) k_scatter(const ct_record* recs, uint64_t n, uint64_t chunk,
                                                             uint64_t T, uint32_t K, uint32_t nmax, uint32_t kc,
                                                             uint32_t kh, const uint64_t* offs, const uint64_t* base,
                                                             const uint64_t* shard_off, const Dest* dest,
                                                             ct_record* out, uint64_t* gpos) {
  extern __shared__ unsigned long long smem_run[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1;
  unsigned long long* run = smem_run + (size_t)warp * K;
  const uint64_t W = (uint64_t)gridDim.x * kCanonWarps;
  for (uint64_t t = (uint64_t)blockIdx.x * kCanonWarps + warp; t < T; t += W) {
    for (uint32_t k = lane; k < K; k += 32)
      run[k] = offs[(uint64_t)k * T + t] - base[k] + (MODE == 1 ? shard_off[k] : 0ull);
    __syncwarp();
    const uint64_t lo = t * chunk, hi = min(n, lo + chunk);
    for (uint64_t i0 = lo; i0 < hi; i0 += 32) {
      const uint64_t i = i0 + lane;
      const bool act = i < hi;
      uint4 a = make_uint4(0, 0, 0, 0), b = a;
      if (act) {
        const uint4* p = reinterpret_cast<const uint4*>(recs + i);
        if (MODE == 0) a = __ldg(p);
        b = __ldg(p + 1);
      }
      const uint32_t key = act ? key_of(b, nmax, kc, kh) : 0x80000000u | (uint32_t)lane;
      const unsigned m = __match_any_sync(0xFFFFFFFFu, key);
      const unsigned long long ord = act ? run[key] + __popc(m & lt) : 0ull;
      __syncwarp();
      if (act && (m >> lane) == 1u) run[key] += __popc(m);
      __syncwarp();
      if (act) {
        const Dest d = dest[key];
        const bool keep = ord < d.limit;
        const unsigned long long g = d.pos + ord * d.stride;
        if (MODE == 0) {
          if (keep) {
            uint4* o = reinterpret_cast<uint4*>(out + g);
            o[0] = a;
            o[1] = b;
          }
        } else {
          gpos[i] = keep ? g : ~0ull;
        }
      }
    }
    __syncwarp();
  }
}

struct Layout {
  std::vector<Dest> dest;
  uint64_t m = 0, n_incomplete = 0, n_us = 0, n_ur = 0;
  std::vector<uint64_t> rstart, rsize;  // regions of equal-size elements (for shard cuts)
};

// Canonical stream layout from the per-key totals: complete groups in (comm first-seen,
// ordinal) order, matched pairs per channel (comm id, src, dst), copies in file order.
Layout make_layout(uint32_t n_comms, uint32_t nmax, uint32_t K, uint64_t kc, uint64_t kh,
                   const std::vector<unsigned int>& nr_max, const std::vector<unsigned long long>& first,
                   const std::vector<uint64_t>& tot) {
  Layout L;
  L.dest.assign(K, Dest{0, 0, 1});
  uint64_t pos = 0;
  std::vector<uint32_t> corder;
  for (uint32_t c = 0; c < n_comms; c++)
    if (first[c] != ~0ull) corder.push_back(c);
  std::sort(corder.begin(), corder.end(), [&](uint32_t a, uint32_t b) { return first[a] < first[b]; });
  for (uint32_t c : corder) {
    const uint32_t nc = nr_max[c];
    uint64_t lo = ~0ull, hi = 0;
    for (uint32_t r = 0; r < nc; r++) {
      lo = std::min(lo, tot[(uint64_t)c * nmax + r]);
      hi = std::max(hi, tot[(uint64_t)c * nmax + r]);
    }
    L.n_incomplete += hi - lo;  // groups k in [lo, hi) miss at least one rank
    for (uint32_t r = 0; r < nc; r++) L.dest[(uint64_t)c * nmax + r] = Dest{pos + r, lo, nc};
    if (lo) { L.rstart.push_back(pos); L.rsize.push_back(nc); }
    pos += lo * nc;
  }
  for (uint64_t ch = 0; ch < kh; ch++) {  // channels in (comm id, src, dst) order
    const uint64_t sn = tot[kc + ch], rn = tot[kc + kh + ch], p = std::min(sn, rn);
    L.n_us += sn - p;
    L.n_ur += rn - p;
    L.dest[kc + ch] = Dest{pos, p, 2};
    L.dest[kc + kh + ch] = Dest{pos + 1, p, 2};
    if (p) { L.rstart.push_back(pos); L.rsize.push_back(2); }
    pos += 2 * p;
  }
  const uint64_t n_copies = tot[K - 1];
  L.dest[K - 1] = Dest{pos, n_copies, 1};
  if (n_copies) { L.rstart.push_back(pos); L.rsize.push_back(1); }
  pos += n_copies;
  L.m = pos;
  return L;
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
  // ---- pass 1: meta and per-tile key counts in one read (key stride guessed from the
  // first records; a larger nranks later reruns the count with the true stride)
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
  uint32_t nguess = 1;
  {
    const uint64_t ns = std::min<uint64_t>(n, 1024);
    std::vector<ct_record> sample(ns);
    cudaMemcpyAsync(sample.data(), recs, ns * sizeof(ct_record), cudaMemcpyDeviceToHost, st);
    if (cudaError_t e = cudaStreamSynchronize(st)) { cleanup(); return (int)e; }
    for (const ct_record& r : sample)
      if ((r.kc & 7) <= CT_KIND_RECV) nguess = std::max<uint32_t>(nguess, r.nranks);
  }
  uint32_t nmax = nguess, K = 0;
  uint64_t kc = 0, kh = 0, chunk = 1024, T = 0;
  uint32_t* counts = nullptr;
  uint64_t* offs = nullptr;
  auto keyspace = [&](uint32_t nm) -> bool {  // key stride nm -> K, tiles, count buffers
    nmax = nm;
    kc = (uint64_t)n_comms * nmax;
    kh = (uint64_t)n_comms * nmax * nmax;
    const uint64_t K64 = kc + 2 * kh + 1;
    if (K64 > kMaxKeys) return false;
    K = (uint32_t)K64;
    chunk = 1024;
    while ((n + chunk - 1) / chunk * (uint64_t)K > (64ull << 20)) chunk *= 2;  // <= 64M counters
    T = (n + chunk - 1) / chunk;
    counts = dalloc<uint32_t>(T * K, st);
    offs = dalloc<uint64_t>(T * K, st);
    scratch.insert(scratch.end(), {counts, offs});
    return counts && offs;
  };
  if (!keyspace(nguess)) { cleanup(); return kCanonUnsupported; }
  uint64_t* kbase = dalloc<uint64_t>(kMaxKeys, st);
  uint64_t* ktot = dalloc<uint64_t>(kMaxKeys, st);
  scratch.insert(scratch.end(), {kbase, ktot});
  if (!kbase || !ktot) { cleanup(); return (int)cudaErrorMemoryAllocation; }
  uint64_t ctas = std::min<uint64_t>((uint64_t)num_sms * 8, (T + kCanonWarps - 1) / kCanonWarps);
  {
    const size_t smem_cm = (size_t)n_comms * 16 + (size_t)kCanonWarps * K * 4;
    cudaFuncSetAttribute(k_count_meta, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_cm);
    k_count_meta<<<(unsigned)ctas, 32 * kCanonWarps, smem_cm, st>>>(recs, n, chunk, T, K, nmax, (uint32_t)kc,
                                                                     (uint32_t)kh, counts, n_comms, meta, nr_min,
                                                                     nr_max, cfirst);
    L++;
  }
  Meta hm;
  std::vector<unsigned int> h_min(n_comms), h_max(n_comms);
  std::vector<unsigned long long> h_first(n_comms);
  cudaMemcpyAsync(&hm, meta, sizeof hm, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(h_min.data(), nr_min, n_comms * 4, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(h_max.data(), nr_max, n_comms * 4, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(h_first.data(), cfirst, n_comms * 8, cudaMemcpyDeviceToHost, st);
  if (cudaError_t e = cudaStreamSynchronize(st)) { cleanup(); return (int)e; }
  if (hm.bad & 1u) { cleanup(); return kCanonUnsupported; }
  for (uint32_t c = 0; c < n_comms; c++)
    if (h_max[c] && h_min[c] != h_max[c]) { cleanup(); return kCanonUnsupported; }  // nranks disagreement
  if (hm.bad & 2u) {  // the sample under-estimated nranks: count again with the true stride
    if (!keyspace(std::max(hm.nmax, 1u))) { cleanup(); return kCanonUnsupported; }
    ctas = std::min<uint64_t>((uint64_t)num_sms * 8, (T + kCanonWarps - 1) / kCanonWarps);
    const size_t smem_c = (size_t)kCanonWarps * K * 4;
    cudaFuncSetAttribute(k_count, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_c);
    k_count<<<(unsigned)ctas, 32 * kCanonWarps, smem_c, st>>>(recs, n, chunk, T, K, nmax, (uint32_t)kc, (uint32_t)kh,
                                                              counts);
    L++;
  }
  const size_t smem = (size_t)kCanonWarps * K * 4;
  cudaFuncSetAttribute(k_scatter<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(2 * smem));
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
  const Layout lay = make_layout(n_comms, nmax, K, kc, kh, h_max, h_first, tot);
  const std::vector<Dest>& dest = lay.dest;
  const uint64_t m = lay.m, n_incomplete = lay.n_incomplete, n_us = lay.n_us, n_ur = lay.n_ur;
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
  k_scatter<0><<<(unsigned)ctas, 32 * kCanonWarps, 2 * smem, st>>>(recs, n, chunk, T, K, nmax, (uint32_t)kc,
                                                                   (uint32_t)kh, offs, kbase, nullptr, d_dest, canon,
                                                                   nullptr);
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


// ============================================================================
// Multi-GPU: canonicalise globally, then shard (one process per GPU).
//
// Every rank holds a record range of a trace in ANY layout.  Two small all-gathers give
// every rank the per-shard key totals, from which each rank computes the global
// canonical layout (exactly the single-GPU stream above), the global canonical
// position of each of its own records (its ordinal = the same keys' totals in earlier
// shards + its local ordinal) and balanced, element-aligned cuts of that stream into
// one part per rank.  One all-to-all moves every record to the rank owning its
// position; each rank then analyses a slice of the single-GPU canonical stream with the
// fast kernel and the partials merge as for record-range shards.
// ============================================================================
namespace {

constexpr uint64_t kMetaMagic = 0x43545348524d4554ull, kCountMagic = 0x43545348524b4559ull;
constexpr uint64_t kPlanHdr = 16;

__global__ void k_gather_rows(const ct_record* recs, const uint64_t* idx, uint64_t n, ct_record* out) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n; j += (uint64_t)gridDim.x * blockDim.x) {
    const uint4* p = reinterpret_cast<const uint4*>(recs + idx[j]);
    uint4* o = reinterpret_cast<uint4*>(out + j);
    o[0] = p[0];
    o[1] = p[1];
  }
}

__global__ void k_iota64(uint64_t* a, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) a[i] = i;
}

// lower_bound of every cut in the sorted positions
__global__ void k_cut_index(const uint64_t* sorted, uint64_t n, const uint64_t* cuts, int nc, uint64_t* out) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nc) return;
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) / 2;
    if (sorted[mid] < cuts[j]) lo = mid + 1; else hi = mid;
  }
  out[j] = lo;
}

__global__ void k_assemble(const uint64_t* pos, const ct_record* rec, uint64_t n, uint64_t lo, uint64_t len,
                           ct_record* part, unsigned int* bad) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n; j += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t g = pos[j];
    if (g < lo || g - lo >= len) { atomicOr(bad, 1u); continue; }
    const uint4* p = reinterpret_cast<const uint4*>(rec + j);
    uint4* o = reinterpret_cast<uint4*>(part + (g - lo));
    o[0] = p[0];
    o[1] = p[1];
  }
}

int to_host(void* dst, const void* src, size_t bytes, cudaStream_t st) {
  if (cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st)) return (int)e;
  return (int)cudaStreamSynchronize(st);
}

}  // namespace

uint64_t shard_meta_words(uint32_t n_comms) { return kPlanHdr + 3ull * n_comms; }
uint64_t shard_count_words() { return kPlanHdr + kMaxKeys; }

void ShardState::release(cudaStream_t st) {
  if (counts) cudaFreeAsync(counts, st);
  if (offs) cudaFreeAsync(offs, st);
  if (kbase) cudaFreeAsync(kbase, st);
  counts = nullptr; offs = nullptr; kbase = nullptr;
  valid = false;
  part = nullptr;
}

int shard_meta(const ct_record* recs, uint64_t n, uint32_t n_comms, int num_sms, cudaStream_t st, uint64_t* dev_out) {
  if (n_comms > kMaxMetaComms) return kCanonUnsupported;
  std::vector<uint64_t> h(shard_meta_words(n_comms), 0);
  h[0] = kMetaMagic;
  h[1] = n;
  h[5] = n_comms;
  for (uint32_t c = 0; c < n_comms; c++) {
    h[kPlanHdr + c] = 0xFFFFFFFFull;
    h[kPlanHdr + 2ull * n_comms + c] = ~0ull;
  }
  if (n) {
    Meta* meta = dalloc<Meta>(1, st);
    unsigned int* nr_min = dalloc<unsigned int>(n_comms, st);
    unsigned int* nr_max = dalloc<unsigned int>(n_comms, st);
    unsigned long long* cfirst = dalloc<unsigned long long>(n_comms, st);
    if (!meta || !nr_min || !nr_max || !cfirst) return (int)cudaErrorMemoryAllocation;
    Meta m0{0, 0, -1, 0};
    cudaMemcpyAsync(meta, &m0, sizeof m0, cudaMemcpyHostToDevice, st);
    cudaMemsetAsync(nr_min, 0xFF, n_comms * 4, st);
    cudaMemsetAsync(nr_max, 0, n_comms * 4, st);
    cudaMemsetAsync(cfirst, 0xFF, n_comms * 8, st);
    const uint64_t blocks = std::min<uint64_t>((uint64_t)num_sms * 8, (n + 4095) / 4096);
    const uint64_t span = (n + blocks - 1) / blocks;
    k_meta<<<(unsigned)blocks, kMetaThreads, 0, st>>>(recs, n, span, n_comms, meta, nr_min, nr_max, cfirst);
    Meta hm;
    std::vector<unsigned int> h_min(n_comms), h_max(n_comms);
    cudaMemcpyAsync(h_min.data(), nr_min, n_comms * 4, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(h_max.data(), nr_max, n_comms * 4, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(h.data() + kPlanHdr + 2ull * n_comms, cfirst, n_comms * 8, cudaMemcpyDeviceToHost, st);
    if (int e = to_host(&hm, meta, sizeof hm, st)) return e;
    cudaFreeAsync(meta, st); cudaFreeAsync(nr_min, st); cudaFreeAsync(nr_max, st); cudaFreeAsync(cfirst, st);
    h[2] = hm.nmax;
    h[3] = hm.bad;
    h[4] = (uint64_t)(hm.max_dev + 1);
    for (uint32_t c = 0; c < n_comms; c++) {
      h[kPlanHdr + c] = h_min[c];
      h[kPlanHdr + n_comms + c] = h_max[c];
    }
  }
  return (int)cudaMemcpyAsync(dev_out, h.data(), h.size() * 8, cudaMemcpyHostToDevice, st);
}

namespace {
// the global view of the gathered metas: shard sizes, key space, per-comm nranks and
// first-seen positions (global record index)
struct GlobalMeta {
  std::vector<uint64_t> n, base;
  uint32_t nmax = 1, K = 0;
  uint64_t kc = 0, kh = 0;
  int max_dev = -1;
  std::vector<unsigned int> nr_max;
  std::vector<unsigned long long> first;
};

int global_meta(const uint64_t* dev_metas, int world, uint32_t n_comms, cudaStream_t st, GlobalMeta* g) {
  const uint64_t w = shard_meta_words(n_comms);
  std::vector<uint64_t> h(w * world);
  if (int e = to_host(h.data(), dev_metas, h.size() * 8, st)) return e;
  std::vector<unsigned int> nmin(n_comms, 0xFFFFFFFFu);
  g->nr_max.assign(n_comms, 0);
  g->first.assign(n_comms, ~0ull);
  uint64_t base = 0;
  bool bad = false;
  for (int s = 0; s < world; s++) {
    const uint64_t* p = h.data() + w * s;
    if (p[0] != kMetaMagic || p[5] != n_comms) return kCanonUnsupported;
    g->n.push_back(p[1]);
    g->base.push_back(base);
    g->nmax = std::max<uint32_t>(g->nmax, (uint32_t)p[2]);
    bad = bad || p[3];
    g->max_dev = std::max(g->max_dev, (int)p[4] - 1);
    for (uint32_t c = 0; c < n_comms; c++) {
      if (p[kPlanHdr + n_comms + c]) {
        nmin[c] = std::min<unsigned int>(nmin[c], (unsigned int)p[kPlanHdr + c]);
        g->nr_max[c] = std::max<unsigned int>(g->nr_max[c], (unsigned int)p[kPlanHdr + n_comms + c]);
      }
      const uint64_t f = p[kPlanHdr + 2ull * n_comms + c];
      if (f != ~0ull) g->first[c] = std::min<unsigned long long>(g->first[c], base + f);
    }
    base += p[1];
  }
  if (bad || base >= (1ull << 40)) return kCanonUnsupported;
  for (uint32_t c = 0; c < n_comms; c++)
    if (g->nr_max[c] && nmin[c] != g->nr_max[c]) return kCanonUnsupported;  // nranks disagreement
  g->kc = (uint64_t)n_comms * g->nmax;
  g->kh = (uint64_t)n_comms * g->nmax * g->nmax;
  const uint64_t K = g->kc + 2 * g->kh + 1;
  if (K > kMaxKeys) return kCanonUnsupported;
  g->K = (uint32_t)K;
  return 0;
}
}  // namespace

int shard_count(ShardState* S, const ct_record* recs, uint64_t n, uint32_t n_comms, const uint64_t* dev_metas,
                int world, int num_sms, cudaStream_t st, uint64_t* dev_out) {
  S->release(st);
  GlobalMeta g;
  if (int e = global_meta(dev_metas, world, n_comms, st, &g)) return e;
  const uint32_t K = g.K;
  uint64_t chunk = 1024;
  while ((n + chunk - 1) / chunk * (uint64_t)K > (64ull << 20)) chunk *= 2;
  const uint64_t T = std::max<uint64_t>((n + chunk - 1) / chunk, 1);
  S->counts = dalloc<uint32_t>(T * K, st);
  S->offs = dalloc<uint64_t>(T * K, st);
  S->kbase = dalloc<uint64_t>(K, st);
  uint64_t* ktot = dalloc<uint64_t>(K, st);
  if (!S->counts || !S->offs || !S->kbase || !ktot) return (int)cudaErrorMemoryAllocation;
  cudaMemsetAsync(S->counts, 0, T * K * 4, st);
  const size_t smem = (size_t)kCanonWarps * K * 4;
  const uint64_t ctas = std::min<uint64_t>((uint64_t)num_sms * 8, (T + kCanonWarps - 1) / kCanonWarps);
  cudaFuncSetAttribute(k_count, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (n) k_count<<<(unsigned)ctas, 32 * kCanonWarps, smem, st>>>(recs, n, chunk, T, K, g.nmax, (uint32_t)g.kc,
                                                                 (uint32_t)g.kh, S->counts);
  size_t tmp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp, S->counts, S->offs, (int64_t)(T * K), st);
  void* t = dalloc<uint8_t>(tmp, st);
  if (!t) return (int)cudaErrorMemoryAllocation;
  if (cudaError_t e = cub::DeviceScan::ExclusiveSum(t, tmp, S->counts, S->offs, (int64_t)(T * K), st)) return (int)e;
  cudaFreeAsync(t, st);
  k_key_totals<<<(K + 255) / 256, 256, 0, st>>>(S->counts, S->offs, T, K, S->kbase, ktot);
  std::vector<uint64_t> h(shard_count_words(), 0);
  h[0] = kCountMagic;
  h[1] = K;
  h[2] = g.nmax;
  if (int e = to_host(h.data() + kPlanHdr, ktot, K * 8, st)) return e;
  cudaFreeAsync(ktot, st);
  S->recs = recs;
  S->n = n;
  S->chunk = chunk;
  S->T = T;
  S->K = K;
  S->nmax = g.nmax;
  S->kc = g.kc;
  S->kh = g.kh;
  return (int)cudaMemcpyAsync(dev_out, h.data(), h.size() * 8, cudaMemcpyHostToDevice, st);
}

int shard_route(ShardState* S, uint32_t n_comms, const uint64_t* dev_metas, const uint64_t* dev_counts, int world,
                int rank, int num_sms, cudaStream_t st, uint64_t* out_pos, ct_record* out_rec, uint64_t* send_counts,
                uint64_t* recv_counts, uint64_t* part_len) {
  if (!S->counts) return kCanonUnsupported;
  GlobalMeta g;
  if (int e = global_meta(dev_metas, world, n_comms, st, &g)) return e;
  const uint32_t K = S->K;
  if (g.K != K) return kCanonUnsupported;
  const uint64_t cw = shard_count_words();
  std::vector<uint64_t> hc(cw * world);
  if (int e = to_host(hc.data(), dev_counts, hc.size() * 8, st)) return e;
  std::vector<uint64_t> tot(K, 0), shard_off(K, 0);
  for (int s = 0; s < world; s++) {
    const uint64_t* p = hc.data() + cw * s;
    if (p[0] != kCountMagic || p[1] != K) return kCanonUnsupported;
    for (uint32_t k = 0; k < K; k++) {
      if (s < rank) shard_off[k] += p[kPlanHdr + k];
      tot[k] += p[kPlanHdr + k];
    }
  }
  const Layout L = make_layout(n_comms, g.nmax, K, g.kc, g.kh, g.nr_max, g.first, tot);
  // balanced cuts of [0, m) snapped up to element starts
  std::vector<uint64_t> cuts(world + 1, L.m);
  cuts[0] = 0;
  for (int r = 1; r < world; r++) {
    const uint64_t x = L.m * (uint64_t)r / (uint64_t)world;
    uint64_t snap = L.m;
    for (size_t q = 0; q < L.rstart.size(); q++) {
      const uint64_t a = L.rstart[q], b = q + 1 < L.rstart.size() ? L.rstart[q + 1] : L.m;
      if (x < b) { snap = x <= a ? a : a + (x - a + L.rsize[q] - 1) / L.rsize[q] * L.rsize[q]; break; }
    }
    cuts[r] = std::max(cuts[r - 1], std::min(snap, L.m));
  }
  // records arriving from every shard (arithmetic on each key's progression)
  for (int s = 0; s < world; s++) {
    uint64_t cnt = 0;
    const uint64_t* p = hc.data() + cw * s;
    for (uint32_t k = 0; k < K; k++) {
      const Dest& d = L.dest[k];
      uint64_t before = 0;
      for (int q = 0; q < s; q++) before += hc[cw * q + kPlanHdr + k];
      const uint64_t lo = before, hi = std::min<uint64_t>(before + p[kPlanHdr + k], d.limit);
      if (lo >= hi) continue;
      // ordinals K with d.pos + K * stride in [cuts[rank], cuts[rank + 1])
      auto first_at = [&](uint64_t A) -> uint64_t {
        return A <= d.pos ? 0 : (A - d.pos + d.stride - 1) / d.stride;
      };
      const uint64_t a = std::max(lo, first_at(cuts[rank])), b = std::min(hi, first_at(cuts[rank + 1]));
      if (b > a) cnt += b - a;
    }
    recv_counts[s] = cnt;
  }
  // global positions of the local records, sorted (= grouped by destination part)
  const uint64_t n = S->n;
  uint64_t* gpos = dalloc<uint64_t>(n, st);
  uint64_t* gsorted = dalloc<uint64_t>(n, st);
  uint64_t* idx = dalloc<uint64_t>(n, st);
  uint64_t* idx_sorted = dalloc<uint64_t>(n, st);
  Dest* d_dest = dalloc<Dest>(K, st);
  uint64_t* d_off = dalloc<uint64_t>(K, st);
  uint64_t* d_cuts = dalloc<uint64_t>(world + 1, st);
  uint64_t* d_ci = dalloc<uint64_t>(world + 1, st);
  if (!gpos || !gsorted || !idx || !idx_sorted || !d_dest || !d_off || !d_cuts || !d_ci)
    return (int)cudaErrorMemoryAllocation;
  cudaMemcpyAsync(d_dest, L.dest.data(), K * sizeof(Dest), cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(d_off, shard_off.data(), K * 8, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(d_cuts, cuts.data(), (world + 1) * 8, cudaMemcpyHostToDevice, st);
  const size_t smem = (size_t)kCanonWarps * K * 8;
  const uint64_t ctas = std::min<uint64_t>((uint64_t)num_sms * 8, (S->T + kCanonWarps - 1) / kCanonWarps);
  cudaFuncSetAttribute(k_scatter<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  uint64_t kept = 0;
  if (n) {
    k_scatter<1><<<(unsigned)ctas, 32 * kCanonWarps, smem, st>>>(S->recs, n, S->chunk, S->T, K, S->nmax,
                                                                 (uint32_t)S->kc, (uint32_t)S->kh, S->offs, S->kbase,
                                                                 d_off, d_dest, nullptr, gpos);
    k_iota64<<<(unsigned)std::min<uint64_t>((n + 255) / 256, 4096), 256, 0, st>>>(idx, n);
    size_t tmp = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp, gpos, gsorted, idx, idx_sorted, n, 0, 64, st);
    void* t = dalloc<uint8_t>(tmp, st);
    if (!t) return (int)cudaErrorMemoryAllocation;
    if (cudaError_t e = cub::DeviceRadixSort::SortPairs(t, tmp, gpos, gsorted, idx, idx_sorted, n, 0, 64, st))
      return (int)e;
    cudaFreeAsync(t, st);
    k_cut_index<<<1, 64, 0, st>>>(gsorted, n, d_cuts, world + 1, d_ci);
    std::vector<uint64_t> ci(world + 1);
    if (int e = to_host(ci.data(), d_ci, (world + 1) * 8, st)) return e;
    for (int r = 0; r < world; r++) send_counts[r] = ci[r + 1] - ci[r];
    kept = ci[world];  // dropped records (incomplete groups, unmatched p2p) sort to the end
    cudaMemcpyAsync(out_pos, gsorted, kept * 8, cudaMemcpyDeviceToDevice, st);
    if (kept) k_gather_rows<<<(unsigned)std::min<uint64_t>((kept + 255) / 256, 4096), 256, 0, st>>>(S->recs, idx_sorted,
                                                                                                 kept, out_rec);
  } else {
    for (int r = 0; r < world; r++) send_counts[r] = 0;
  }
  for (void* p : {(void*)gpos, (void*)gsorted, (void*)idx, (void*)idx_sorted, (void*)d_dest, (void*)d_off,
                  (void*)d_cuts, (void*)d_ci})
    cudaFreeAsync(p, st);
  S->part_lo = cuts[rank];
  S->part_len = cuts[rank + 1] - cuts[rank];
  *part_len = S->part_len;
  S->extra_diag[0] = rank == 0 ? L.n_incomplete : 0;
  S->extra_diag[1] = rank == 0 ? L.n_us : 0;
  S->extra_diag[2] = rank == 0 ? L.n_ur : 0;
  S->global_max_dev = g.max_dev;
  S->rank = rank;
  if (cudaError_t e = cudaGetLastError()) return (int)e;
  return (int)cudaStreamSynchronize(st);
}

int shard_assemble(ShardState* S, const uint64_t* in_pos, const ct_record* in_rec, uint64_t n_in, ct_record* part,
                   cudaStream_t st) {
  unsigned int* bad = dalloc<unsigned int>(1, st);
  if (!bad) return (int)cudaErrorMemoryAllocation;
  cudaMemsetAsync(bad, 0, 4, st);
  if (n_in)
    k_assemble<<<(unsigned)std::min<uint64_t>((n_in + 255) / 256, 4096), 256, 0, st>>>(in_pos, in_rec, n_in, S->part_lo,
                                                                                     S->part_len, part, bad);
  unsigned int hb = 0;
  if (int e = to_host(&hb, bad, 4, st)) return e;
  cudaFreeAsync(bad, st);
  if (hb || n_in != S->part_len) return kCanonUnsupported;  // records missing / outside the part
  S->part = part;
  S->valid = true;
  return 0;
}

}  // namespace ct
