// Fast path: fused layout check + expand + accumulate (see ct_fast.cuh for the plan).
#include "ct_fast.cuh"

namespace ct {

namespace {

constexpr uint64_t kEmptyKey = 0x7FFFFFFFFFFFFFFFull;
constexpr uint32_t kEmptyTag = 0xFFFFFFFFu;
constexpr uint64_t kNone = ~0ull;

struct __align__(128) SmemFixed {
  ct_record ring[kStages][kSub];
  unsigned long long mbar[kStages];
  uint64_t ekey[kSub];
  uint16_t elist[kSub];
  uint8_t status[kSub];
  uint8_t iselem[kSub];
  ChainEntry chain[kWarps][kChainW];
  unsigned long long calls[kTypes], pay_lo[kTypes], pay_hi[kTypes];
  unsigned long long tf[5][kCommSm];
  unsigned long long cf[kCommSm];
  unsigned long long copy_first[3];
  uint32_t warp_cnt[kWarps];
  unsigned int diag[CT_NDIAG];
  uint32_t ne;
  uint32_t flags;
  int max_dev;
};

// ------------------------------------------------------------ TMA bulk ring
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(unsigned long long* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes,
                                          unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
  }
}

// ------------------------------------------------------------ record access
struct View {
  const ct_record* g;    // whole analyzed array
  const ct_record* cur;  // current sub-tile in shared memory
  uint64_t base;         // index of cur[0]
  uint32_t len;
  uint64_t n;
  __device__ __forceinline__ Rec get(uint64_t i) const {
    uint64_t off = i - base;
    return off < len ? load_shared(cur + off) : load_global(g + i);
  }
  __device__ __forceinline__ uint32_t dev_of(uint64_t i) const {
    uint64_t off = i - base;
    const uint32_t* w = off < len ? reinterpret_cast<const uint32_t*>(cur + off)
                                  : reinterpret_cast<const uint32_t*>(g + i);
    return (off < len ? w[6] : __ldg(w + 6)) & 0xFFFF;
  }
  __device__ __forceinline__ uint64_t seq_of(uint64_t i) const {
    uint64_t off = i - base;
    if (off < len) return reinterpret_cast<const uint64_t*>(cur + off)[1];
    return __ldg(reinterpret_cast<const unsigned long long*>(g + i) + 1);
  }
};

// Instance validity of the block headed at ``i`` (grouping.py:144-167): signature
// equality first, then pairwise-distinct devices.  Assumes the block lies in [0, n).
__device__ uint8_t head_status(const View& v, uint64_t i, const Rec& head) {
  const uint32_t n = head.nranks;
  if (i + n > v.n) return ST_NONE;
  bool incompat = false, dup = false, wide = false;
  uint64_t seen[4] = {0, 0, 0, 0};
  for (uint32_t m = 0; m < n; m++) {
    Rec q = m == 0 ? head : v.get(i + m);
    if (m && !same_sig(q, head)) incompat = true;
    uint32_t d = q.dev;
    if (d < 256) {
      uint64_t bit = 1ull << (d & 63);
      uint32_t w = d >> 6;
      uint64_t word = w == 0 ? seen[0] : w == 1 ? seen[1] : w == 2 ? seen[2] : seen[3];
      if (word & bit) dup = true;
      word |= bit;
      if (w == 0) seen[0] = word; else if (w == 1) seen[1] = word; else if (w == 2) seen[2] = word; else seen[3] = word;
    } else {
      wide = true;
    }
  }
  if (wide && !dup) {  // devices >= 256: pairwise among the wide ones
    for (uint32_t a = 0; a < n && !dup; a++) {
      uint32_t da = v.dev_of(i + a);
      if (da < 256) continue;
      for (uint32_t b = a + 1; b < n; b++)
        if (v.dev_of(i + b) == da) { dup = true; break; }
    }
  }
  return incompat ? ST_INCOMPAT : dup ? ST_DUPDEV : ST_VALID;
}

// consecutive chain elements (pred before cur): reference seq ordering holds
__device__ bool chain_ok(const View& v, uint64_t pred, uint64_t cur) {
  Rec a = v.get(pred), b = v.get(cur);
  if (b.kind() == CT_KIND_COLLECTIVE) {
    const uint32_t n = b.nranks;
    if (a.nranks != n || pred + n > v.n || cur + n > v.n) return false;
    for (uint32_t r = 0; r < n; r++) {
      uint64_t sa = r ? v.seq_of(pred + r) : a.seq;
      uint64_t sb = r ? v.seq_of(cur + r) : b.seq;
      if (!(sa < sb)) return false;
    }
    return true;
  }
  if (pred + 1 >= v.n || cur + 1 >= v.n) return false;
  return a.seq <= b.seq && v.seq_of(pred + 1) <= v.seq_of(cur + 1);
}

__device__ __forceinline__ uint32_t hash64(uint64_t k) {
  return static_cast<uint32_t>((k * 0x9E3779B97F4A7C15ull) >> 32);
}

// ------------------------------------------------------------ accumulation
struct Acc {
  // register cache: (key, bytes, count); key = cell index or kStatsKeyBit | type
  uint32_t tag[kCacheE];
  unsigned long long sum[kCacheE];
  uint32_t cnt[kCacheE];
  uint32_t flags;
  unsigned long long* hb;  // histogram bytes (shared or global)
  void* hf;                // histogram counts: u32 shared or u64 global
  bool smem;
  SmemFixed* S;
  int g2, gcap;
  bool explicit_d;
  unsigned long long rec_key;  // (class << 62) | (element << 21) | (src rank << 11) for oor ordering
  unsigned long long oor_key;
  unsigned long long of_cell;

  __device__ void init(SmemFixed* s, unsigned long long* b, void* f, bool sm, int g2_, int gcap_, bool ex) {
#pragma unroll
    for (int e = 0; e < kCacheE; e++) { tag[e] = kEmptyTag; sum[e] = 0; cnt[e] = 0; }
    flags = 0; hb = b; hf = f; smem = sm; S = s; g2 = g2_; gcap = gcap_; explicit_d = ex;
    rec_key = 0; oor_key = ~0ull; of_cell = ~0ull;
  }

  __device__ void flush(uint32_t key, unsigned long long v, uint32_t c) {
    if (key & kStatsKeyBit) {
      int t = key & 15;
      unsigned long long old = atomicAdd(&S->pay_lo[t], v);
      if (old + v < old) atomicAdd(&S->pay_hi[t], 1ull);
      atomicAdd(&S->calls[t], (unsigned long long)c);
      return;
    }
    unsigned long long old = atomicAdd(hb + key, v);
    if (old + v < old) { flags |= F_OVERFLOW; if (key < of_cell) of_cell = key; }
    if (smem) atomicAdd(static_cast<unsigned int*>(hf) + key, c);
    else atomicAdd(static_cast<unsigned long long*>(hf) + key, (unsigned long long)c);
  }

  __device__ __forceinline__ void add(uint32_t key, unsigned long long v) {
    bool hit = false;
#pragma unroll
    for (int e = 0; e < kCacheE; e++) {
      if (tag[e] == key) {
        unsigned long long s = sum[e] + v;
        if (s < v) { flags |= F_OVERFLOW; if (key < of_cell) of_cell = key; }
        sum[e] = s;
        cnt[e] += 1;
        hit = true;
      }
    }
    if (!hit) {
      if (tag[kCacheE - 1] != kEmptyTag) flush(tag[kCacheE - 1], sum[kCacheE - 1], cnt[kCacheE - 1]);
#pragma unroll
      for (int e = kCacheE - 1; e > 0; e--) { tag[e] = tag[e - 1]; sum[e] = sum[e - 1]; cnt[e] = cnt[e - 1]; }
      tag[0] = key; sum[0] = v; cnt[0] = 1;
    }
  }

  __device__ void drain() {
#pragma unroll
    for (int e = 0; e < kCacheE; e++) {
      if (tag[e] != kEmptyTag) flush(tag[e], sum[e], cnt[e]);
      tag[e] = kEmptyTag;
    }
  }

  // stats: calls += 1, payload += s (128-bit capable)
  __device__ __forceinline__ void stat(int type, unsigned __int128 s) {
    if ((s >> 63) == 0) { add(kStatsKeyBit | type, (unsigned long long)s); return; }
    unsigned long long lo = (unsigned long long)s, hi = (unsigned long long)(s >> 64);
    unsigned long long old = atomicAdd(&S->pay_lo[type], lo);
    if (old + lo < old) hi += 1;
    atomicAdd(&S->pay_hi[type], hi);
    atomicAdd(&S->calls[type], 1ull);
  }

  // endpoint: gpu g (g >= 0) or -1 host / -2 net
  __device__ __forceinline__ bool index(int ep, int& idx, unsigned long long k) {
    if (ep == -1) { idx = kHost; return true; }
    if (ep == -2) { idx = kNet; return true; }
    if (ep >= gcap) {
      flags |= explicit_d ? F_OOR : F_CAP;
      if (k < oor_key) oor_key = k;
      return false;
    }
    idx = ep + 2;
    return true;
  }

  // ``sub`` orders transfers inside one decomposition: the destination rank for
  // collectives (transfers are sorted by rank pair, decompose.py:92), 0/1 for collnet.
  __device__ __forceinline__ void edge(int type, int src, int dst, unsigned __int128 bytes, int sub = 0) {
    int a, b;
    const unsigned long long k = rec_key | ((unsigned long long)min(sub, 1023) << 1);
    bool ok = index(src, a, k);
    ok = index(dst, b, k | 1) && ok;
    if (!ok) return;
    if ((bytes >> 63) != 0) { flags |= F_OVERFLOW; return; }
    add((uint32_t)((type * g2 + a) * g2 + b), (unsigned long long)bytes);
  }
};

__device__ __forceinline__ void note_min(unsigned long long* slot, unsigned long long v) {
  if (v < *slot) atomicMin(slot, v);
}

}  // namespace

size_t fast_smem_bytes(int g2, int smem_hist) {
  size_t b = sizeof(SmemFixed);
  if (smem_hist) b += (size_t)kTypes * g2 * g2 * (sizeof(unsigned long long) + sizeof(unsigned int));
  return b;
}

__global__ void __launch_bounds__(kThreads, 1) fast_kernel(FastParams P) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  SmemFixed& S = *reinterpret_cast<SmemFixed*>(smem_raw);
  const int ncell = kTypes * P.g2 * P.g2;
  unsigned long long* shb = reinterpret_cast<unsigned long long*>(smem_raw + sizeof(SmemFixed));
  unsigned int* shf = reinterpret_cast<unsigned int*>(shb + ncell);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  const uint32_t s0 = blockIdx.x * P.subs_per_cta;
  const uint32_t s1 = min(s0 + P.subs_per_cta, P.n_subs);
  if (s0 >= s1) return;

  // ---- init shared state
  if (P.smem_hist)
    for (int c = tid; c < ncell; c += kThreads) { shb[c] = 0; shf[c] = 0; }
  for (int c = tid; c < kWarps * kChainW; c += kThreads) {
    S.chain[c / kChainW][c % kChainW].key = kEmptyKey;
  }
  for (int c = tid; c < 5 * kCommSm; c += kThreads) S.tf[c / kCommSm][c % kCommSm] = kNone;
  if (tid < kCommSm) S.cf[tid] = kNone;
  if (tid < kTypes) { S.calls[tid] = 0; S.pay_lo[tid] = 0; S.pay_hi[tid] = 0; }
  if (tid < 3) S.copy_first[tid] = kNone;
  if (tid < CT_NDIAG) S.diag[tid] = 0;
  if (tid == 0) {
    S.flags = 0;
    S.max_dev = -1;
    for (int k = 0; k < kStages; k++) mbar_init(&S.mbar[k], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  auto issue = [&](uint32_t sub, int stage) {
    uint64_t first = (uint64_t)sub * kSub;
    uint32_t cnt = (uint32_t)min((uint64_t)kSub, P.n - first);
    mbar_expect_tx(&S.mbar[stage], cnt * (uint32_t)sizeof(ct_record));
    bulk_load(S.ring[stage], P.recs + first, cnt * (uint32_t)sizeof(ct_record), &S.mbar[stage]);
  };
  if (tid == 0) {
    for (uint32_t k = 0; k < (uint32_t)kStages && s0 + k < s1; k++) issue(s0 + k, k);
  }

  Acc acc;
  acc.init(&S, P.smem_hist ? shb : P.cells, P.smem_hist ? (void*)shf : (void*)P.freq,
           P.smem_hist != 0, P.g2, P.gcap, P.explicit_d != 0);
  int my_max_dev = -1;
  uint32_t n_incompat = 0, n_dupdev = 0, n_mismatch = 0;
  unsigned long long my_copy_first[3] = {kNone, kNone, kNone};

  for (uint32_t s = s0; s < s1; s++) {
    const uint32_t k = s - s0;
    const int stage = k % kStages;
    const uint64_t base = (uint64_t)s * kSub;
    const uint32_t len = (uint32_t)min((uint64_t)kSub, P.n - base);
    mbar_wait(&S.mbar[stage], (k / kStages) & 1);
    View v{P.recs, S.ring[stage], base, len, P.n};

    // ---------------- A1: decode, local layout checks, element status
#pragma unroll
    for (int q = 0; q < kPer; q++) {
      const uint32_t j = tid + q * kThreads;
      uint8_t st = ST_NONE, elem = 0;
      uint64_t key = 0;
      if (j < len) {
        const uint64_t i = base + j;
        const Rec rc = load_shared(v.cur + j);
        const int kind = rc.kind();
        my_max_dev = max(my_max_dev, (int)rc.dev);
        if (rc.comm >= P.n_comms) acc.flags |= F_COMM_RANGE | F_NONCANON;
        if (kind == CT_KIND_COLLECTIVE) {
          const uint32_t n = rc.nranks, r = rc.rank;
          bool ok = r < n;
          if (ok && r > 0) {
            ok = i > 0;
            if (ok) {
              Rec p = v.get(i - 1);
              ok = p.kind() == CT_KIND_COLLECTIVE && p.comm == rc.comm && p.nranks == n && p.rank == r - 1;
            }
          }
          if (ok && r + 1 < n) {
            ok = i + 1 < P.n;
            if (ok) {
              Rec q2 = v.get(i + 1);
              ok = q2.kind() == CT_KIND_COLLECTIVE && q2.comm == rc.comm && q2.nranks == n && q2.rank == r + 1;
            }
          }
          if (!ok) {
            acc.flags |= F_NONCANON;
          } else if (r == 0) {
            st = head_status(v, i, rc);
            if (st == ST_NONE) acc.flags |= F_NONCANON;
            n_incompat += st == ST_INCOMPAT;
            n_dupdev += st == ST_DUPDEV;
            elem = 1;
            key = rc.comm;
            const unsigned long long gi = P.base + i;
            if (rc.comm < kCommSm) note_min(&S.cf[rc.comm], gi);
            else if (rc.comm < P.n_comms) note_min(&P.comm_first[rc.comm], gi);
          }
        } else if (kind == CT_KIND_SEND) {
          bool ok = i + 1 < P.n;
          Rec q2;
          if (ok) {
            q2 = v.get(i + 1);
            ok = q2.kind() == CT_KIND_RECV && q2.comm == rc.comm && q2.rank == rc.aux && q2.aux == rc.rank;
          }
          if (!ok) {
            acc.flags |= F_NONCANON;
          } else {
            const bool mis = q2.count != rc.count || q2.dtype() != rc.dtype();
            st = mis ? ST_MISMATCH : ST_VALID;
            n_mismatch += mis;
            elem = 1;
            key = (1ull << 63) | ((uint64_t)rc.comm << 32) | ((uint64_t)rc.rank << 16) | rc.aux;
          }
        } else if (kind == CT_KIND_RECV) {
          bool ok = i > 0;
          if (ok) {
            Rec p = v.get(i - 1);
            ok = p.kind() == CT_KIND_SEND && p.comm == rc.comm && p.aux == rc.rank && p.rank == rc.aux;
          }
          if (!ok) acc.flags |= F_NONCANON;
        } else {
          const int ck = rc.ckind();
          if (ck != CT_CKIND_H2D) my_max_dev = max(my_max_dev, (int)rc.aux);
          if (ck != CT_CKIND_D2H) my_max_dev = max(my_max_dev, (int)rc.aux2);
        }
      }
      S.status[j] = st;
      S.iselem[j] = elem;
      S.ekey[j] = key;
    }
    __syncthreads();

    // ---------------- A2: compact chain elements in position order
    {
      const uint32_t p0 = warp * 64 + lane, p1 = p0 + 32;
      const unsigned b0 = __ballot_sync(0xFFFFFFFFu, S.iselem[p0]);
      const unsigned b1 = __ballot_sync(0xFFFFFFFFu, S.iselem[p1]);
      if (lane == 0) S.warp_cnt[warp] = __popc(b0) + __popc(b1);
      __syncthreads();
      uint32_t off = 0, tot = 0;
      for (int w = 0; w < kWarps; w++) {
        uint32_t c = S.warp_cnt[w];
        off += w < warp ? c : 0;
        tot += c;
      }
      const unsigned lt = (1u << lane) - 1;
      if (S.iselem[p0]) S.elist[off + __popc(b0 & lt)] = (uint16_t)p0;
      if (S.iselem[p1]) S.elist[off + __popc(b0) + __popc(b1 & lt)] = (uint16_t)p1;
      if (tid == 0) S.ne = tot;
    }
    __syncthreads();

    // ---------------- A3: chain checks, warp-partitioned by key hash
    {
      const uint32_t ne = S.ne;
      ChainEntry* tab = S.chain[warp];
      const unsigned lt = (1u << lane) - 1, gt = ~((2u << lane) - 1);
      for (uint32_t b = 0; b < ne; b += 32) {
        const uint32_t e = b + lane;
        const bool act = e < ne;
        const uint32_t pos = act ? S.elist[e] : 0;
        const uint64_t key = act ? S.ekey[pos] : 0;
        const uint32_t h = hash64(key);
        const bool own = act && (h & (kWarps - 1)) == (uint32_t)warp;
        if (!__any_sync(0xFFFFFFFFu, own)) continue;
        const uint64_t mk = own ? key : (0x7FFFFFFF00000000ull | lane);
        const unsigned m = __match_any_sync(0xFFFFFFFFu, mk);
        const unsigned lower = m & lt, higher = m & gt;
        const int src_lane = lower ? 31 - __clz(lower) : lane;
        const uint32_t ppos = __shfl_sync(0xFFFFFFFFu, pos, src_lane);
        const uint64_t cur = base + pos;
        int slot = -1;
        uint64_t pred = kNone;
        if (own) {
          if (lower) {
            pred = base + ppos;
          } else {
            uint32_t s2 = (h >> 4) % kChainW;
            for (int probe = 0; probe < kChainW; probe++, s2 = (s2 + 1) % kChainW) {
              unsigned long long old = atomicCAS(reinterpret_cast<unsigned long long*>(&tab[s2].key),
                                                 kEmptyKey, key);
              if (old == kEmptyKey) { tab[s2].first = cur; tab[s2].last = cur; slot = s2; break; }
              if (old == key) { pred = tab[s2].last; slot = s2; break; }
            }
            if (slot < 0) acc.flags |= F_CHAIN_CAP | F_NONCANON;
          }
          if (pred != kNone && !chain_ok(v, pred, cur)) acc.flags |= F_NONCANON;
        }
        __syncwarp();
        if (own && !higher) {
          if (slot < 0) {
            uint32_t s2 = (h >> 4) % kChainW;
            for (int probe = 0; probe < kChainW; probe++, s2 = (s2 + 1) % kChainW)
              if (tab[s2].key == key) { slot = s2; break; }
          }
          if (slot >= 0) tab[slot].last = cur;
        }
        __syncwarp();
      }
    }

    // ---------------- B: expansion + accumulation
#pragma unroll
    for (int q = 0; q < kPer; q++) {
      const uint32_t j = tid + q * kThreads;
      if (j >= len) continue;
      const uint64_t i = base + j;
      const Rec rc = load_shared(v.cur + j);
      const int kind = rc.kind();
      if (kind == CT_KIND_COLLECTIVE) {
        const uint32_t r = rc.rank;
        if (r > i || r >= rc.nranks) continue;
        const uint64_t head = i - r;
        uint8_t st;
        if (head >= base) st = S.status[head - base];
        else st = head_status(v, head, v.get(head));
        if (st != ST_VALID) continue;
        if (r == 0) {
          const int t = rc.coll();
          if (t < 5) {
            const unsigned long long gi = P.base + i;
            if (rc.comm < kCommSm) note_min(&S.tf[t][rc.comm], gi);
            else if (rc.comm < P.n_comms) note_min(&P.type_comm_first[(size_t)t * P.n_comms + rc.comm], gi);
          }
        }
        acc.rec_key = (0ull << 62) | (min((unsigned long long)head, (1ull << 41) - 1) << 21) | ((unsigned long long)min(r, 1023u) << 11);
        if ((rc.count >> 40) == 0) expand_collective<uint64_t>(P.ex, v, acc, rc, head);
        else expand_collective<unsigned __int128>(P.ex, v, acc, rc, head);
      } else if (kind == CT_KIND_SEND) {
        if (S.status[j] != ST_VALID) continue;
        const unsigned __int128 nb = (unsigned __int128)rc.count * (unsigned)dtype_width(rc.dtype());
        acc.stat(CT_T_SENDRECV, nb);
        acc.rec_key = (1ull << 62) | (min((unsigned long long)i, (1ull << 41) - 1) << 21);
        const int rdev = (int)v.dev_of(i + 1);
        if (rdev != (int)rc.dev) acc.edge(CT_T_SENDRECV, (int)rc.dev, rdev, nb);
      } else if (kind >= CT_KIND_MEMCPY) {
        const int ck = rc.ckind();
        const int t = CT_T_EXPLICIT + (kind - CT_KIND_MEMCPY);
        acc.stat(t, (unsigned __int128)rc.count);
        acc.rec_key = (2ull << 62) | (min((unsigned long long)i, (1ull << 41) - 1) << 21);
        acc.edge(t, ck == CT_CKIND_H2D ? -1 : (int)rc.aux, ck == CT_CKIND_D2H ? -1 : (int)rc.aux2,
                 (unsigned __int128)rc.count);
        const unsigned long long gi = P.base + i;
        const int c = kind - CT_KIND_MEMCPY;
        if (gi < my_copy_first[c]) my_copy_first[c] = gi;
      }
    }
    __syncthreads();  // everyone done with this stage
    if (tid == 0 && s + kStages < s1) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(s + kStages, stage);
    }
  }

  // ---- CTA epilogue: drain caches, reduce, one global merge
  acc.drain();
  atomicMax(&S.max_dev, my_max_dev);
  if (n_incompat) atomicAdd(&S.diag[CT_DIAG_INCOMPATIBLE], n_incompat);
  if (n_dupdev) atomicAdd(&S.diag[CT_DIAG_DUPLICATE_DEVICE], n_dupdev);
  if (n_mismatch) atomicAdd(&S.diag[CT_DIAG_MISMATCHED_P2P], n_mismatch);
  for (int c = 0; c < 3; c++)
    if (my_copy_first[c] != kNone) atomicMin(&S.copy_first[c], my_copy_first[c]);
  if (acc.flags) atomicOr(&S.flags, acc.flags);
  if (acc.oor_key != ~0ull) atomicMin(&P.st->oor_key, acc.oor_key);
  if (acc.of_cell != ~0ull) atomicMin(&P.st->of_cell, acc.of_cell);
  __syncthreads();

  GlobalState* G = P.st;
  if (P.smem_hist) {
    uint32_t of = 0;
    for (int c = tid; c < ncell; c += kThreads) {
      const unsigned int f = shf[c];
      if (!f) continue;
      const unsigned long long b = shb[c];
      unsigned long long old = atomicAdd(P.cells + c, b);
      if (old + b < old) { of |= F_OVERFLOW; atomicMin(&G->of_cell, (unsigned long long)c); }
      atomicAdd(P.freq + c, (unsigned long long)f);
    }
    if (of) atomicOr(&S.flags, of);
  }
  if (tid < kTypes) {
    const unsigned long long lo = S.pay_lo[tid], hi = S.pay_hi[tid], c = S.calls[tid];
    if (c) {
      unsigned long long old = atomicAdd(&G->pay_lo[tid], lo);
      atomicAdd(&G->pay_hi[tid], hi + (old + lo < old ? 1ull : 0ull));
      atomicAdd(&G->calls[tid], c);
    }
  }
  if (tid < CT_NDIAG && S.diag[tid]) atomicAdd(&G->diag[tid], (unsigned long long)S.diag[tid]);
  if (tid < 3 && S.copy_first[tid] != kNone) atomicMin(&G->copy_first[tid], S.copy_first[tid]);
  for (int c = tid; c < 5 * kCommSm; c += kThreads) {
    const int t = c / kCommSm, cm = c % kCommSm;
    if (S.tf[t][cm] != kNone && (uint32_t)cm < P.n_comms)
      atomicMin(&P.type_comm_first[(size_t)t * P.n_comms + cm], S.tf[t][cm]);
  }
  if (tid < kCommSm && S.cf[tid] != kNone && (uint32_t)tid < P.n_comms)
    atomicMin(&P.comm_first[tid], S.cf[tid]);
  for (int c = tid; c < kWarps * kChainW; c += kThreads) {
    const ChainEntry& e = S.chain[c / kChainW][c % kChainW];
    if (e.key == kEmptyKey) continue;
    uint32_t slot = atomicAdd(&G->n_chain, 1u);
    if (slot < P.chain_cap) P.chain[slot] = e;
    else atomicOr(&S.flags, F_CHAIN_CAP | F_NONCANON);
  }
  __syncthreads();
  if (tid == 0) {
    if (S.flags) atomicOr(&G->flags, S.flags);
    atomicMax(&G->max_dev, S.max_dev);
  }
}

// Cross-CTA chain check: entries sorted by (key, first); consecutive same-key entries
// must satisfy chain_ok(last of earlier, first of later).
__global__ void chain_check_kernel(const ct_record* recs, uint64_t n, const ChainEntry* chain,
                                   const uint32_t* order, uint32_t count, GlobalState* st) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0 || i >= count) return;
  const ChainEntry& a = chain[order[i - 1]];
  const ChainEntry& b = chain[order[i]];
  if (a.key != b.key) return;
  View v{recs, recs, 0, 0, n};
  if (!chain_ok(v, a.last, b.first)) atomicOr(&st->flags, F_NONCANON);
}

}  // namespace ct

namespace ct {

// Cross-CTA chain check in one CTA: bitonic-sort the (key, first) list in shared memory
// and validate consecutive same-key entries.  Lists longer than kChainSortMax set
// F_CHAIN_BIG and the host falls back to CUB radix sorts + chain_check_kernel.
__global__ void __launch_bounds__(1024) chain_sort_check_kernel(const ct_record* recs, uint64_t n,
                                                                const ChainEntry* chain, GlobalState* st) {
  extern __shared__ __align__(16) unsigned char sm[];
  uint64_t* key = reinterpret_cast<uint64_t*>(sm);
  uint64_t* first = key + kChainSortMax;
  uint32_t* idx = reinterpret_cast<uint32_t*>(first + kChainSortMax);
  const uint32_t E = st->n_chain;
  if (E <= 1 || (st->flags & F_NONCANON)) return;
  if (E > kChainSortMax) {
    if (threadIdx.x == 0) atomicOr(&st->flags, F_CHAIN_BIG);
    return;
  }
  uint32_t P = 1;
  while (P < E) P <<= 1;
  for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) {
    key[i] = i < E ? chain[i].key : ~0ull;
    first[i] = i < E ? chain[i].first : ~0ull;
    idx[i] = i;
  }
  __syncthreads();
  for (uint32_t k = 2; k <= P; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) {
        const uint32_t l = i ^ j;
        if (l > i) {
          const bool up = (i & k) == 0;
          const bool gt = key[i] > key[l] || (key[i] == key[l] && first[i] > first[l]);
          if (gt == up) {
            uint64_t tk = key[i]; key[i] = key[l]; key[l] = tk;
            uint64_t tf = first[i]; first[i] = first[l]; first[l] = tf;
            uint32_t ti = idx[i]; idx[i] = idx[l]; idx[l] = ti;
          }
        }
      }
      __syncthreads();
    }
  }
  View v{recs, recs, 0, 0, n};
  for (uint32_t i = threadIdx.x + 1; i < E; i += blockDim.x) {
    if (key[i] != key[i - 1]) continue;
    if (!chain_ok(v, chain[idx[i - 1]].last, chain[idx[i]].first)) atomicOr(&st->flags, F_NONCANON);
  }
}

}  // namespace ct
