// Synthetic trace generators, written straight into HBM as packed
// records.  Every record is a pure function of (seed, index), so any range of the
// stream can be produced independently (multi-GPU shards, bounded CPU samples) and
// the layout is the canonical one the reference's own generator emits
// (workload.py:89-159: all ranks of a call consecutive, per-(comm, rank) seq counters).
//
//   C2  n=8 mixed collectives: coll uniform over 5, dtype over 10, count log-uniform
//       [1, 2^28), root uniform, allreduce algo over {ring, tree, collnet, auto}.
//   C3  groups of 40 records: 3 collective blocks (as C2, comm 0), 2 send/recv pairs
//       (comm 1, dev = rank % 6 so some pairs stay on one GPU), 12 copies (comm 2,
//       memcpy/um/zerocopy x h2d/d2h/d2d, bytes log-uniform [1, 2^30)).
//   C4  ResNet-50 data-parallel training, n=8 ring allreduce over reverse-greedy
//       25 MiB gradient buckets (workload.py:69-86, 166-195), one broadcast per
//       parameter tensor at init, 8 x 192 KiB h2d copies per iteration
//       (resnet_like_preset, workload.py:221-235, with the ResNet-50 tensor list).
//   C4i C4 in the capture layout of an LD_PRELOAD interposer (kind 6, see capture_source).
//   C5  ring vs tree allreduce sweep: groups of 35 records holding one block of every
//       n in 2..8 (comm n-2) in a seeded order, algo ring|tree, bytes log-uniform
//       [1 KiB, 1 GiB).
#include <cstring>
#include <vector>

#include "ct_common.cuh"

namespace ct {

namespace {

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__host__ __device__ __forceinline__ uint64_t h2(uint64_t seed, uint64_t a, uint64_t b) {
  return mix64(seed ^ mix64(a * 0xD1B54A32D192ED03ull + b));
}

// log-uniform integer in [2^lo, 2^hi)
__host__ __device__ __forceinline__ uint64_t log_uniform(uint64_t h, int lo, int hi) {
  const int e = lo + (int)((h & 0xFFFF) % (uint64_t)(hi - lo));
  const uint64_t base = 1ull << e;
  return base + ((h >> 16) % base);
}

__device__ __forceinline__ void put(ct_record* out, uint64_t count, uint64_t seq, uint32_t comm,
                                    uint32_t nranks, uint32_t rank, uint32_t dev, uint32_t aux,
                                    uint32_t aux2, uint32_t kc, uint32_t ad) {
  uint4 a, b;
  a.x = (uint32_t)count; a.y = (uint32_t)(count >> 32);
  a.z = (uint32_t)seq;   a.w = (uint32_t)(seq >> 32);
  b.x = comm;
  b.y = (nranks & 0xFFFF) | (rank << 16);
  b.z = (dev & 0xFFFF) | (aux << 16);
  b.w = (aux2 & 0xFFFF) | ((kc & 0xFF) << 16) | ((ad & 0xFF) << 24);
  uint4* o = reinterpret_cast<uint4*>(out);
  o[0] = a;
  o[1] = b;
}

// one C2-style collective record: instance ``inst`` of comm ``comm``, rank r of 8
__device__ __forceinline__ void mixed_collective(ct_record* out, uint64_t seed, uint64_t inst, uint32_t r,
                                                 uint32_t comm, uint64_t seq) {
  const uint64_t h = h2(seed, 2, inst), g = h2(seed, 3, inst);
  const uint32_t coll = (uint32_t)(h % 5);
  const uint32_t dtype = (uint32_t)((h >> 8) % 10);
  const uint64_t count = log_uniform(g, 0, 28);
  const bool rooted = coll == CT_COLL_BROADCAST || coll == CT_COLL_REDUCE;
  const uint32_t root = (uint32_t)((h >> 16) % 8);
  const uint32_t algo = coll == CT_COLL_ALLREDUCE ? (uint32_t)((h >> 24) % 4) : CT_ALGO_RING;
  const uint32_t kc = CT_KIND_COLLECTIVE | (coll << 3) | (rooted ? 1u << 6 : 0u);
  put(out, count, seq, comm, 8, r, r, rooted ? root : 0, 0, kc, algo | (dtype << 2));
}

// ---------------------------------------------------------------- C4 tables
constexpr int kMaxTensors = 256;
constexpr int kMaxBuckets = 64;
__constant__ uint64_t c4_tensor_count[kMaxTensors];  // float32 elements per tensor
__constant__ uint64_t c4_bucket_count[kMaxBuckets];  // float32 elements per bucket
__constant__ uint32_t c4_dims[2];                    // n_tensors, n_buckets

struct C4Tables {
  std::vector<uint64_t> tensor_bytes, bucket_bytes;
};

// ResNet-50 parameter tensors in module order (torchvision layout: conv weights,
// batch-norm weight + bias; 161 tensors, 25,557,032 parameters), float32.
C4Tables c4_tables() {
  std::vector<uint64_t> p;
  auto conv = [&](uint64_t cin, uint64_t cout, uint64_t k) { p.push_back(cout * cin * k * k); };
  auto bn = [&](uint64_t c) { p.push_back(c); p.push_back(c); };
  conv(3, 64, 7); bn(64);
  const int blocks[4] = {3, 4, 6, 3};
  const uint64_t width[4] = {64, 128, 256, 512};
  uint64_t cin = 64;
  for (int s = 0; s < 4; s++) {
    for (int b = 0; b < blocks[s]; b++) {
      const uint64_t w = width[s], cout = 4 * w;
      conv(cin, w, 1); bn(w);
      conv(w, w, 3); bn(w);
      conv(w, cout, 1); bn(cout);
      if (b == 0) { conv(cin, cout, 1); bn(cout); }
      cin = cout;
    }
  }
  p.push_back(2048ull * 1000); p.push_back(1000);
  C4Tables t;
  for (uint64_t x : p) t.tensor_bytes.push_back(4 * x);
  // plan_buckets: reverse walk, close a bucket when the next tensor would overflow it,
  // oversized tensors travel alone (workload.py:69-86)
  const uint64_t cap = 25ull << 20;
  uint64_t cur = 0;
  for (size_t k = t.tensor_bytes.size(); k-- > 0;) {
    const uint64_t s = t.tensor_bytes[k];
    if (s > cap) {
      if (cur) { t.bucket_bytes.push_back(cur); cur = 0; }
      t.bucket_bytes.push_back(s);
      continue;
    }
    if (cur && cur + s > cap) { t.bucket_bytes.push_back(cur); cur = 0; }
    cur += s;
  }
  if (cur) t.bucket_bytes.push_back(cur);
  return t;
}

bool c4_uploaded[64] = {false};

int c4_upload(cudaStream_t st) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64 && c4_uploaded[dev]) return 0;
  C4Tables t = c4_tables();
  uint64_t tc[kMaxTensors] = {0}, bc[kMaxBuckets] = {0};
  for (size_t k = 0; k < t.tensor_bytes.size(); k++) tc[k] = (t.tensor_bytes[k] + 3) / 4;
  for (size_t k = 0; k < t.bucket_bytes.size(); k++) bc[k] = (t.bucket_bytes[k] + 3) / 4;
  uint32_t dims[2] = {(uint32_t)t.tensor_bytes.size(), (uint32_t)t.bucket_bytes.size()};
  if (cudaMemcpyToSymbolAsync(c4_tensor_count, tc, sizeof tc, 0, cudaMemcpyHostToDevice, st) != cudaSuccess) return 1;
  if (cudaMemcpyToSymbolAsync(c4_bucket_count, bc, sizeof bc, 0, cudaMemcpyHostToDevice, st) != cudaSuccess) return 1;
  if (cudaMemcpyToSymbolAsync(c4_dims, dims, sizeof dims, 0, cudaMemcpyHostToDevice, st) != cudaSuccess) return 1;
  cudaStreamSynchronize(st);
  if (dev < 64) c4_uploaded[dev] = true;
  return 0;
}

// ---------------------------------------------------------------- capture layout
// C4 as an LD_PRELOAD interposer records it (kind 6): every process appends its own calls
// in call order, the processes of one job interleave.  The C4 stream is a sequence of
// rounds of 8 records, one per rank (an allreduce block or the 8 per-iteration copies);
// in epochs of kEpochRounds rounds, rank r lags by delta_r(e) in [0, kMaxLag) rounds and
// every round lists its ranks in a seeded order.  Each rank's records keep their order,
// the ranks of one call spread over up to kMaxLag neighbouring calls, and an epoch
// boundary (a multiple of 8 * kEpochRounds records) is a clean cut.
constexpr uint64_t kEpochRounds = 16384;
constexpr uint32_t kMaxLag = 8;

// canonical C4 index of the record at capture position p
__device__ uint64_t capture_source(uint64_t seed, uint64_t p) {
  const uint64_t E = kEpochRounds, e = p / (8 * E), q = p % (8 * E);
  uint32_t lag[8];
#pragma unroll
  for (int r = 0; r < 8; r++) lag[r] = (uint32_t)(h2(seed, 11, e * 8 + r) % kMaxLag);
  auto start = [&](uint64_t t) -> uint64_t {  // records in rounds < t
    uint64_t s = 0;
#pragma unroll
    for (int r = 0; r < 8; r++) s += t > lag[r] ? min(t - lag[r], E) : 0;
    return s;
  };
  uint64_t lo = 0, hi = E + kMaxLag;  // last round t with start(t) <= q
  while (hi - lo > 1) {
    const uint64_t mid = (lo + hi) / 2;
    if (start(mid) <= q) lo = mid; else hi = mid;
  }
  const uint64_t t = lo;
  uint32_t within = (uint32_t)(q - start(t));
  // ranks present in round t, in a seeded order: the within-th smallest hash key
  uint64_t key[8];
  bool here[8];
#pragma unroll
  for (int r = 0; r < 8; r++) {
    here[r] = t >= lag[r] && t - lag[r] < E;
    key[r] = (h2(seed, 12, (e << 24) ^ (t << 3) ^ (uint64_t)r) & ~7ull) | (uint64_t)r;
  }
  int pick = 0;
#pragma unroll
  for (int r = 0; r < 8; r++) {
    if (!here[r]) continue;
    uint32_t below = 0;
#pragma unroll
    for (int s = 0; s < 8; s++) below += here[s] && key[s] < key[r];
    if (below == within) pick = r;
  }
  return e * 8 * E + 8 * (t - lag[pick]) + (uint64_t)pick;
}

// ---------------------------------------------------------------- kernels
__global__ void k_gen(int kind_in, uint64_t seed, uint64_t first, uint64_t n, ct_record* out) {
  const int kind = kind_in == 6 ? 4 : kind_in;  // capture layout of C4: C4 records, permuted
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < n;
       k += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i = kind_in == 6 ? capture_source(seed, first + k) : first + k;
    ct_record* o = out + k;
    if (kind == 2) {
      mixed_collective(o, seed, i / 8, (uint32_t)(i % 8), 0, i / 8);
    } else if (kind == 3) {
      const uint64_t g = i / 40;
      const uint32_t off = (uint32_t)(i % 40);
      // [blk 0..7][cp 8..11][pair 12..13][blk 14..21][cp 22..25][pair 26..27][blk 28..35][cp 36..39]
      int blk = -1, pair = -1, cp = -1;
      uint32_t rel = 0;
      if (off < 8) { blk = 0; rel = off; }
      else if (off < 12) { cp = (int)(off - 8); }
      else if (off < 14) { pair = 0; rel = off - 12; }
      else if (off < 22) { blk = 1; rel = off - 14; }
      else if (off < 26) { cp = 4 + (int)(off - 22); }
      else if (off < 28) { pair = 1; rel = off - 26; }
      else if (off < 36) { blk = 2; rel = off - 28; }
      else { cp = 8 + (int)(off - 36); }
      if (blk >= 0) {
        mixed_collective(o, seed, g * 3 + blk, rel, 0, g * 3 + blk);
      } else if (pair >= 0) {
        const uint64_t pid = g * 2 + pair, h = h2(seed, 5, pid);
        const uint32_t src = (uint32_t)(h % 8), dst = (src + 1 + (uint32_t)((h >> 8) % 7)) % 8;
        const uint32_t dtype = (uint32_t)((h >> 16) % 10);
        const uint64_t count = log_uniform(h2(seed, 6, pid), 0, 20) - 1;
        if (rel == 0) put(o, count, pid, 1, 8, src, src % 6, dst, 0, CT_KIND_SEND, dtype << 2);
        else put(o, count, pid, 1, 8, dst, dst % 6, src, 0, CT_KIND_RECV, dtype << 2);
      } else {
        const uint64_t cid = g * 12 + cp, h = h2(seed, 7, cid);
        const uint32_t kind_c = CT_KIND_MEMCPY + (uint32_t)(h % 3);
        const uint32_t ck = (uint32_t)((h >> 8) % 3);
        const uint32_t a = (uint32_t)((h >> 16) % 8), b = (a + 1 + (uint32_t)((h >> 24) % 7)) % 8;
        const uint64_t bytes = log_uniform(h2(seed, 8, cid), 0, 30) - 1;
        const uint32_t src = ck == CT_CKIND_H2D ? 0 : a, dst = ck == CT_CKIND_D2H ? 0 : (ck == CT_CKIND_H2D ? a : b);
        put(o, bytes, cid, 2, 8, a, a, src, dst, kind_c, ck << 6);
      }
    } else if (kind == 4) {
      const uint64_t T = c4_dims[0], B = c4_dims[1];
      const uint64_t init = 8 * T, iter = 8 + 8 * B;
      if (i < init) {  // one broadcast per tensor from rank 0 (workload.py:178-183)
        const uint64_t t = i / 8;
        const uint32_t r = (uint32_t)(i % 8);
        put(o, c4_tensor_count[t], t, 0, 8, r, r, 0, 0,
            CT_KIND_COLLECTIVE | (CT_COLL_BROADCAST << 3) | (1u << 6), CT_ALGO_RING | (8u << 2));
      } else {
        const uint64_t it = (i - init) / iter, off = (i - init) % iter;
        const uint64_t seq0 = T + it * (B + 1);  // per-rank calls before this iteration
        if (off < 8) {  // h2d copy by rank off to its own GPU (workload.py:186-189)
          const uint32_t r = (uint32_t)off;
          put(o, 192ull << 10, seq0, 0, 8, r, r, 0, r, CT_KIND_MEMCPY, CT_CKIND_H2D << 6);
        } else {
          const uint64_t b = (off - 8) / 8;
          const uint32_t r = (uint32_t)((off - 8) % 8);
          put(o, c4_bucket_count[b], seq0 + 1 + b, 0, 8, r, r, 0, 0,
              CT_KIND_COLLECTIVE | (CT_COLL_ALLREDUCE << 3), CT_ALGO_RING | (8u << 2));
        }
      }
    } else {  // kind 5
      const uint64_t g = i / 35;
      const uint32_t off = (uint32_t)(i % 35);
      // seeded permutation of block sizes 2..8 (Lehmer code of h % 5040)
      uint64_t code = h2(seed, 9, g) % 5040;
      int avail[7] = {2, 3, 4, 5, 6, 7, 8};
      int sizes[7];
      int left = 7;
      uint64_t fact = 720;
      for (int k = 0; k < 7; k++) {
        const int pick = (int)(code / fact);
        code %= fact;
        sizes[k] = avail[pick];
        for (int q = pick; q < left - 1; q++) avail[q] = avail[q + 1];
        left--;
        if (left > 0) fact /= left;
      }
      uint32_t start = 0;
      int nb = 0;
      for (int k = 0; k < 7; k++) {
        if (off < start + (uint32_t)sizes[k]) { nb = sizes[k]; break; }
        start += sizes[k];
      }
      const uint32_t r = off - start;
      const uint64_t h = h2(seed, 10, g * 8 + nb);
      const uint32_t algo = (h & 1) ? CT_ALGO_TREE : CT_ALGO_RING;
      const uint64_t bytes = log_uniform(h >> 1, 10, 30);
      put(o, bytes / 4, g, (uint32_t)(nb - 2), (uint32_t)nb, r, r, 0, 0,
          CT_KIND_COLLECTIVE | (CT_COLL_ALLREDUCE << 3), algo | (8u << 2));
    }
  }
}

}  // namespace

int generate(int kind, uint64_t seed, uint64_t first, uint64_t n, ct_record* out, cudaStream_t st) {
  if (kind < 2 || kind > 6) return 1;
  if ((kind == 4 || kind == 6) && c4_upload(st)) return 1;
  if (!n) return 0;
  uint64_t g = (n + 255) / 256;
  if (g > 148 * 64) g = 148 * 64;
  k_gen<<<(unsigned)g, 256, 0, st>>>(kind, seed, first, n, out);
  return 0;
}

uint64_t generate_boundary(int kind, uint64_t at) {
  if (kind == 3) {  // element starts inside a 40-record group
    static const uint32_t starts[] = {0, 8, 9, 10, 11, 12, 14, 22, 23, 24, 25, 26, 28, 36, 37, 38, 39, 40};
    const uint64_t g = at / 40, off = at % 40;
    for (uint32_t s : starts)
      if (s >= off) return g * 40 + s;
    return (g + 1) * 40;
  }
  const uint64_t q = kind == 5 ? 35 : (kind == 6 ? 8 * kEpochRounds : 8);
  return (at + q - 1) / q * q;
}

// number of records of one C4 training iteration / of the init phase (for configs)
extern "C" void ct_c4_shape(uint64_t* n_tensors, uint64_t* n_buckets, uint64_t* bucket_bytes) {
  C4Tables t = c4_tables();
  *n_tensors = t.tensor_bytes.size();
  *n_buckets = t.bucket_bytes.size();
  for (size_t k = 0; k < t.bucket_bytes.size() && bucket_bytes; k++) bucket_bytes[k] = t.bucket_bytes[k];
}

}  // namespace ct
