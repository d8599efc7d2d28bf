// Fast path: element-parallel streaming layout check + join + expand + accumulate
// (design notes in ct_fast.cuh).
#include "ct_fast.cuh"

#define CT_LIKELY(x) __builtin_expect(!!(x), 1)
#define CT_UNLIKELY(x) __builtin_expect(!!(x), 0)

namespace ct {

namespace {

constexpr uint64_t kNone = ~0ull;
constexpr uint32_t kEmptyTag = 0xFFFFFFFFu;
constexpr unsigned kFull = 0xFFFFFFFFu;
constexpr uint32_t kQM = kQ - 1;
static_assert((kQ & (kQ - 1)) == 0 && kQ >= 96, "queue holds <= 32 carried + 2 chunks of new heads");

// Shared-memory accumulator of repeated instances of one (comm slot, class): class 0 ring
// allreduce (every block but the last full), 1 allgather, 2 reduce-scatter, 3 tree
// allreduce, 4 collnet allreduce, 5 broadcast, 6 reduce (keyed with the root).  Sums are 64-bit as two 32-bit limbs (native atomics) and are written to the
// histogram before they can wrap (FastParams::sa_flush instances, <= 2^14).
struct __align__(16) SAE {
  uint32_t key;               // 1 << 31 | slot | cls << 3 | coll << 6 | n << 9 | root << 13; 0: empty
  uint32_t cnt;               // instances
  uint32_t devs;              // device of rank j in bits [4j, 4j + 4)
  uint32_t pad0;
  uint32_t g[2], d[2], s[2];  // edge sums (ring: gen / dlt; tree: ceil(S/2) / floor(S/2)), payload
  uint32_t cnt2;              // tree: instances with floor(S/2) != 0
  uint32_t pad;
};
constexpr int kSE = 32;             // slot accumulators per warp
constexpr int kCP = 64;             // pooled per-rank seq entries per warp (all comm slots)

struct __align__(16) WarpMem {
  ct_record ring[kRing][32];                 // TMA ring: chunk k lives in slot k % kRing
  SAE sa[kSE];
  unsigned long long cpool[kCP];             // last collective block of each comm: seq per rank,
  uint32_t cbase[kCS];                       //   slot s at cpool[cbase[s] ...] (n entries)
  unsigned long long bar[kRing];
  unsigned long long cfirst[kCS], clast[kCS];
  unsigned long long tfirst[kCS][5];
  uint32_t q[kQ];                            // element queue: ring-relative head positions
  uint32_t tag[kCS];                         // comm id of the slot
  uint32_t sn[kCS];                          // collective nranks of the slot (0: none yet)
  uint32_t uni[kCS];                         // 1: the slot's last block had one seq on every rank,
  unsigned long long useq[kCS];              //    useq (then cpool is not kept up to date)
};

constexpr int kTreeLut = 16;

struct __align__(16) CtaMem {
  // per-type statistics as 32-bit limbs (native shared atomics): [0,4) payload (128-bit),
  // [4,6) calls (64-bit)
  uint32_t st[kTypes][8];
  unsigned long long copy_first[3];
  unsigned long long oor_key;   // min out-of-range ordering key seen by the CTA
  unsigned long long of_cell;   // min cell index whose 64-bit sum wrapped
  // double binary tree peers for n <= kTreeLut (trees.py:57-106): tree_pack() words
  unsigned long long tree_lut[kTreeLut + 1][kTreeLut];
  unsigned int diag[CT_NDIAG];
  uint32_t flags;
  int max_dev;
};
static_assert(sizeof(CtaMem) % 16 == 0, "histogram after CtaMem must stay aligned");
// the shared-memory histogram must fit for d <= 16 (g2 = 18), else the kernel falls back
// to global atomics
static_assert(sizeof(WarpMem) * kWarps + sizeof(CtaMem) + kTypes * 18 * 18 * 12 <= 227 * 1024,
              "shared memory budget: CTA histogram no longer fits for d <= 16");

#ifndef CT_SLACK
#define CT_SLACK 0
#endif
constexpr uint32_t kDrainSlack = CT_SLACK;  // chunks of read-ahead kept free for the TMA ring
constexpr uint32_t kRM = kRing * 32 - 1;  // ring index mask (kRing is a power of two)
static_assert((kRing & (kRing - 1)) == 0, "kRing must be a power of two");

__device__ __forceinline__ CtaMem& cta_mem() {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  return *reinterpret_cast<CtaMem*>(smem_raw + sizeof(WarpMem) * kWarps);
}

// ------------------------------------------------------------ TMA bulk ring
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(unsigned long long* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, unsigned long long* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

// the same on shared-window addresses computed once per warp (no generic->shared
// conversion in the ring loop)
__device__ __forceinline__ void bulk_load_a(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

__device__ __forceinline__ void mbar_wait_a(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
  }
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

// one ring record (two 128-bit words) at a shared-window address; volatile keeps it
// after the mbarrier waits that publish the ring slot
__device__ __forceinline__ void lds256(uint32_t a, uint4& x, uint4& y) {
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(x.x), "=r"(x.y), "=r"(x.z), "=r"(x.w) : "r"(a));
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4+16];" : "=r"(y.x), "=r"(y.y), "=r"(y.z), "=r"(y.w) : "r"(a));
}

__device__ __forceinline__ Rec ring_rec(const ct_record* R, uint32_t pos) { return load_shared(R + (pos & kRM)); }

__device__ __forceinline__ bool is_start(int kind, uint32_t rank) {
  return kind == CT_KIND_COLLECTIVE ? rank == 0
                                    : (kind == CT_KIND_SEND || (kind >= CT_KIND_MEMCPY && kind <= CT_KIND_ZEROCOPY));
}

// first element start at or after x (warp-cooperative, reads global memory)
__device__ uint64_t first_start(const ct_record* g, uint64_t n, uint64_t x, bool& bad) {
  const int lane = threadIdx.x & 31;
  for (int probe = 0; probe < 3; probe++) {
    const uint64_t base = x + 32ull * probe;
    if (base >= n) return n;
    const uint64_t i = base + lane;
    bool st = false;
    if (i < n) {
      const uint4 w = __ldg(reinterpret_cast<const uint4*>(g + i) + 1);
      st = is_start((w.w >> 16) & 7, w.y >> 16);
    }
    const unsigned m = __ballot_sync(kFull, st);
    if (m) return base + (__ffs(m) - 1);
  }
  bad = true;  // no element start within 96 records: not the canonical layout
  return x;
}

// ------------------------------------------------------------ accumulation
// CTA histogram (SH): per cell the byte sum as two 32-bit limbs (lo[ncell], hi[ncell]) and
// a 32-bit frequency, all updated with native shared-memory atomics (a 64-bit shared
// atomic add is a CAS loop).  Without SH the cells are the global 64-bit arrays.
template <bool SH>
__device__ __forceinline__ uint32_t* hist_lo(const FastParams& P) {
  return reinterpret_cast<uint32_t*>(&cta_mem() + 1);
}
__device__ __forceinline__ void note_min_smem(unsigned long long* slot, unsigned long long v) {
  if (v < *slot) atomicMin(slot, v);
}

// an endpoint >= gcap: EndpointOutOfRange with explicit d, else a rerun with a wider table
__device__ __noinline__ uint32_t oor(unsigned long long rec_key, int sub, bool src_bad, int explicit_d) {
  const unsigned long long k = rec_key | ((unsigned long long)min(sub, 1023) << 1);
  note_min_smem(&cta_mem().oor_key, src_bad ? k : (k | 1));
  return explicit_d ? F_OOR : F_CAP;
}

__device__ __noinline__ uint32_t note_overflow(unsigned long long key) {
  note_min_smem(&cta_mem().of_cell, key);
  return F_OVERFLOW;
}

// statistics of type t: payload += (hi:lo), calls += c, carried limb by limb
__device__ __noinline__ void stat_limbs(uint32_t t, unsigned long long lo, unsigned long long hi, uint32_t c) {
  uint32_t* L = cta_mem().st[t];
  unsigned long long carry = 0;
#pragma unroll
  for (int k = 0; k < 4; k++) {
    const unsigned long long add = ((k < 2 ? lo >> (32 * k) : hi >> (32 * (k - 2))) & 0xFFFFFFFFull) + carry;
    carry = add >> 32;
    const uint32_t a32 = (uint32_t)add;
    if (a32) {
      const uint32_t old = atomicAdd(&L[k], a32);
      carry += old + a32 < old ? 1u : 0u;
    }
  }
  const uint32_t old = atomicAdd(&L[4], c);
  if (old + c < old) atomicAdd(&L[5], 1u);
}

// calls += 1, payload += v: the common case inline (two limbs), carries out of line
__device__ __forceinline__ void stat1(uint32_t t, unsigned long long v) {
  uint32_t* L = cta_mem().st[t];
  const uint32_t a = (uint32_t)v, b = (uint32_t)(v >> 32);
  const uint32_t o0 = atomicAdd(&L[0], a);
  const uint32_t c0 = o0 + a < o0 ? 1u : 0u;
  if (b == 0xFFFFFFFFu && c0) {
    stat_limbs(t, 0, 1, 0);  // 2^64
  } else if (b + c0) {
    const uint32_t o1 = atomicAdd(&L[1], b + c0);
    if (o1 + (b + c0) < o1) stat_limbs(t, 0, 1, 0);  // carry into limb 2
  }
  const uint32_t oc = atomicAdd(&L[4], 1u);
  if (oc == 0xFFFFFFFFu) atomicAdd(&L[5], 1u);
}

// Transfers are added straight into the CTA histogram; statistics of the collective
// types and sendrecv (types 0..5) accumulate in registers until the end (or a wrap).
// REGION sink
template <bool SH>
struct Sink {
  const FastParams& P;
  uint32_t flags;
  unsigned long long rec_key;  // (class << 62) | (element << 21) | (src rank << 11) for oor ordering
  uint32_t nc;  // cells per array

  __device__ __forceinline__ explicit Sink(const FastParams& p) : P(p) {
    nc = (uint32_t)(kTypes * p.g2 * p.g2);
    flags = 0;
    rec_key = 0;
  }

  __device__ __forceinline__ void add(uint32_t key, unsigned long long v, uint32_t c = 1) {
    if (SH) {
      uint32_t* lo = hist_lo<SH>(P);
      const uint32_t vlo = (uint32_t)v, vhi = (uint32_t)(v >> 32);  // v < 2^63
      const uint32_t old = atomicAdd(lo + key, vlo);
      const uint32_t inc = vhi + (old + vlo < old ? 1u : 0u);
      if (CT_UNLIKELY(inc)) {
        const uint32_t oh = atomicAdd(lo + nc + key, inc);
        if (oh + inc < oh) flags |= note_overflow(key);  // the 64-bit cell wrapped
      }
      atomicAdd(lo + 2 * nc + key, c);
    } else {
      const unsigned long long old = atomicAdd(P.cells + key, v);
      if (old + v < old) flags |= note_overflow(key);
      atomicAdd(P.freq + key, (unsigned long long)c);
    }
  }

  // endpoint: gpu g (>= 0), -1 host, -2 net.  ``sub`` orders transfers inside one
  // decomposition (destination rank of a collective edge, transfers are sorted by rank
  // pair, decompose.py:92; 0/1 for collnet) for the EndpointOutOfRange message.
  __device__ __forceinline__ void edge(int type, int src, int dst, unsigned __int128 bytes, int sub = 0) {
    if (CT_UNLIKELY(src >= P.gcap || dst >= P.gcap)) {
      flags |= oor(rec_key, sub, src >= P.gcap, P.explicit_d);
      return;
    }
    if ((bytes >> 63) != 0) { flags |= F_OVERFLOW; return; }  // one transfer alone exceeds a cell
    const int a = src == -1 ? kHost : (src == -2 ? kNet : src + 2);
    const int b = dst == -1 ? kHost : (dst == -2 ? kNet : dst + 2);
    add((uint32_t)((type * P.g2 + a) * P.g2 + b), (unsigned long long)bytes);
  }

  // stats: calls += 1, payload += s (128-bit capable)
  __device__ __forceinline__ void stat(int type, unsigned __int128 s) {
    if ((s >> 64) == 0) stat1((uint32_t)type, (unsigned long long)s);
    else stat_limbs((uint32_t)type, (unsigned long long)s, (unsigned long long)(s >> 64), 1u);
  }
};

// Register accumulator for uniform ring-family instances over an identity ring whose
// devices (n <= 8, packed one per byte) are all < gcap.  The edge leaving position q
// carries gen + dlt * ([q == n-2] + [q == n-3]) (mod n): ring allreduce with every block
// but the last full (gen = 2S - 2 chunk, dlt = chunk - last block), allgather /
// reduce-scatter (gen = (n-1) * block, dlt = 0).  Instances with the same (type, n,
// devices) add into 128-bit sums; the n cells are written when the key changes.
// REGION accumulators
__device__ __forceinline__ unsigned long long tree_peers(int n, int j);

// Write accumulated instances of one (type, n, devices) key into the histogram:
// ring classes -- the edge leaving position q carries g + d * ([q == n-2] + [q == n-3]);
// tree -- T1-only peers g, peers in both trees g + d, T2-only peers d (cnt2 transfers).
template <bool SH>
__device__ __noinline__ uint32_t flush_acc(const FastParams& P, int g2, int coll, int n, int mode, int root,
                                           uint32_t devs, unsigned long long g_lo, uint32_t g_hi,
                                           unsigned long long d_lo, uint32_t d_hi, unsigned long long s_lo,
                                           uint32_t s_hi, uint32_t cnt, uint32_t cnt2) {
  Sink<SH> sk(P);
  stat_limbs((uint32_t)coll, s_lo, s_hi, cnt);
  auto emit = [&](int q, int r, uint32_t k_g, uint32_t k_d, uint32_t c) {
    // v = k_g * g + k_d * d as 128 bits (k_* in {0, 1, 2})
    unsigned __int128 v = (unsigned __int128)k_g * (((unsigned __int128)g_hi << 64) | g_lo) +
                          (unsigned __int128)k_d * (((unsigned __int128)d_hi << 64) | d_lo);
    const uint32_t key = (uint32_t)((coll * g2 + (int)((devs >> (4 * q)) & 15u) + 2) * g2 +
                                    (int)((devs >> (4 * r)) & 15u) + 2);
    if ((v >> 63) != 0) sk.flags |= note_overflow(key);  // the cell exceeds 2^63 - 1
    else sk.add(key, (unsigned long long)v, c);
  };
  if (mode == 3) {  // broadcast / reduce pipeline: every position but one sends S (decompose.py:192-224)
    const int skip = coll == CT_COLL_BROADCAST ? (root == 0 ? n - 1 : root - 1) : root;
    for (int q = 0; q < n; q++)
      if (q != skip) emit(q, q + 1 == n ? 0 : q + 1, 1u, 0u, cnt);
  } else if (mode == 0) {
    const int a = n - 2, b = n >= 3 ? n - 3 : n - 1;
    for (int q = 0; q < n; q++) emit(q, q + 1 == n ? 0 : q + 1, 1u, (uint32_t)(q == a) + (uint32_t)(q == b), cnt);
  } else if (mode == 2) {  // collnet: every rank sends S to NET and receives S from it
    const unsigned long long v = g_lo;
    for (int j = 0; j < n; j++) {
      const int dv = (int)((devs >> (4 * j)) & 15u) + 2;
      const uint32_t k_up = (uint32_t)((coll * g2 + dv) * g2 + kNet), k_dn = (uint32_t)((coll * g2 + kNet) * g2 + dv);
      if (g_hi != 0 || (v >> 63) != 0) {
        sk.flags |= note_overflow(k_up);
        sk.flags |= note_overflow(k_dn);
      } else {
        sk.add(k_up, v, cnt);
        sk.add(k_dn, v, cnt);
      }
    }
  } else {
    for (int j = 0; j < n; j++) {
      const unsigned long long w = tree_peers(n, j);
      const int c = (int)(w >> 60);
      for (int x = 0; x < c; x++) {
        const uint32_t code = (uint32_t)(w >> (7 * x));
        const int r = (int)(code & 31);
        if ((code & 0x60) == 0x60) emit(j, r, 1u, 1u, cnt);
        else if (code & 0x20) emit(j, r, 1u, 0u, cnt);
        else if (cnt2) emit(j, r, 0u, 1u, cnt2);
      }
    }
  }
  return sk.flags;
}

// Write out slot accumulator E, then re-key it to ``key`` (with ``devs``) unless key is 0.
template <bool SH>
__device__ __noinline__ uint32_t sa_flush(const FastParams& P, SAE* E, uint32_t key, uint32_t devs) {
  uint32_t f = 0;
  if (E->key && E->cnt)
  {
    const uint32_t cls = E->key >> 3 & 7u;
    f = flush_acc<SH>(P, P.g2, (int)(E->key >> 6 & 7u), (int)(E->key >> 9 & 15u),
                      cls == 3u ? 1 : (cls == 4u ? 2 : (cls >= 5u ? 3 : 0)), (int)(E->key >> 13 & 7u), E->devs,
                      E->g[0] | ((unsigned long long)E->g[1] << 32), 0u, E->d[0] | ((unsigned long long)E->d[1] << 32),
                      0u, E->s[0] | ((unsigned long long)E->s[1] << 32), 0u, E->cnt, E->cnt2);
  }
  if (key) { E->key = key; E->devs = devs; }
  E->g[0] = E->g[1] = E->d[0] = E->d[1] = E->s[0] = E->s[1] = 0;
  E->cnt = E->cnt2 = 0;
  return f;
}

struct RingAcc {
  uint32_t tag;                 // coll | n << 8 (0: empty)
  uint32_t devs;
  unsigned long long g_lo, d_lo, s_lo;  // edge sums, payload sum
  uint32_t g_hi, d_hi, s_hi, cnt;
  uint32_t miss;                // consecutive instances that did not match the key
  uint32_t thr;                 // misses before re-keying: doubles when a key collected few instances

  template <bool SH>
  __device__ __forceinline__ void flush(Sink<SH>& sk, int g2) {
    sk.flags |= flush_acc<SH>(sk.P, g2, (int)(tag & 0xFF), (int)(tag >> 8), 0, 0, devs, g_lo, g_hi, d_lo, d_hi,
                              s_lo, s_hi, cnt, 0u);
  }

  // false: the key differs and is kept (the caller expands the instance itself); after a
  // streak of misses the accumulator is flushed and re-keyed
  template <bool SH>
  __device__ __forceinline__ bool add(Sink<SH>& sk, int g2, uint32_t t, uint32_t dv, unsigned long long g,
                                      unsigned long long d, unsigned long long sz) {
    if (t != tag || dv != devs) {
      if (CT_LIKELY(tag && ++miss < thr)) return false;
      if (tag) {
        thr = cnt < thr ? min(2 * thr, 4096u) : 8u;  // back off when keys do not repeat per lane
        flush(sk, g2);
      }
      tag = t; devs = dv;
      g_lo = d_lo = s_lo = 0; g_hi = d_hi = s_hi = cnt = 0;
    }
    miss = 0;
    const unsigned long long x = g_lo + g, y = d_lo + d, z = s_lo + sz;
    g_hi += x < g ? 1u : 0u;
    d_hi += y < d ? 1u : 0u;
    s_hi += z < sz ? 1u : 0u;
    g_lo = x; d_lo = y; s_lo = z;
    cnt++;
    if (cnt == 0xFFFFFFFFu) { flush(sk, g2); tag = 0; }
    return true;
  }
};

// a copy transfer with an endpoint outside the table or >= 2^63 bytes
template <bool SH>
__device__ __noinline__ uint32_t copy_edge_slow(const FastParams& P, unsigned long long gidx, int type, int src, int dst,
                                                unsigned long long cnt) {
  Sink<SH> sk(P);
  sk.rec_key = (2ull << 62) | (min(gidx, (1ull << 41) - 1) << 21);
  sk.edge(type, src, dst, (unsigned __int128)cnt);
  if (max(src, dst) >= 0) atomicMax(&cta_mem().max_dev, max(src, dst));  // GPU endpoints for d
  return sk.flags;
}

// device of a record held in the warp's ring, by ring-relative position
struct WinDev {
  const ct_record* R;
  __device__ __forceinline__ uint32_t dev_of(uint64_t rel) const { return R[(uint32_t)rel & kRM].dev; }
};

// a collective record with count >= 2^40 (128-bit byte counts): rare, kept out of line
template <bool SH>
__device__ __noinline__ uint32_t expand_wide(const FastParams& P, const ct_record* R, Rec rc, uint32_t head,
                                             unsigned long long rec_key) {
  const WinDev wdv{R};
  Sink<SH> sk(P);
  sk.rec_key = rec_key;
  expand_collective<unsigned __int128>(P.ex, wdv, sk, rc, head);
  return sk.flags;
}

// allocate comm slots for the lanes whose comm is new to this range (warp-collective, one
// comm at a time); -2: more comms than slots in one range
__device__ __noinline__ int alloc_slots(WarpMem& W, bool need, uint32_t comm, int slot, int lane) {
  bool full = false;
  while (true) {
    const unsigned miss = __ballot_sync(kFull, need && slot < 0);
    if (!miss) break;
    const uint32_t cm = __shfl_sync(kFull, comm, __ffs(miss) - 1);
    int free_s = -1;
    for (int s = kCS - 1; s >= 0; s--)
      if (W.tag[s] == kEmptyTag) free_s = s;
    __syncwarp();
    if (free_s < 0) { full = true; break; }
    if (lane == 0) W.tag[free_s] = cm;
    __syncwarp();
    if (need && slot < 0 && comm == cm) slot = free_s;
  }
  return full && need && slot < 0 ? -2 : slot;
}

__device__ __forceinline__ int find_slot(const WarpMem& W, uint32_t comm) {
  int s = -1;
#pragma unroll
  for (int k = 0; k < kCS; k++)
    if (W.tag[k] == comm) s = k;
  return s;
}

// per-rank seq order of the block at ring position p against the comm's previous block:
// the same batch (ring position pp) or the slot table (uniform seq useq, or the pool)
__device__ __noinline__ bool seq_order_ranks(const ct_record* R, uint32_t p, uint32_t n, uint32_t pp, bool in_batch,
                                             bool uni, unsigned long long useq, const unsigned long long* pool,
                                             uint32_t cb) {
  bool ok = true;
  for (uint32_t r = 0; r < n; r++) {
    const unsigned long long ps = in_batch ? R[(pp + r) & kRM].seq : (uni ? useq : pool[(cb + r) & (kCP - 1)]);
    ok = ok && ps < R[(p + r) & kRM].seq;
  }
  return ok;
}

// devices of the block of n records at ring position p when some device is >= 32:
// bit 0 = two records share a device, bit 1 = every device is < gcap
__device__ __noinline__ uint32_t block_devices(const ct_record* R, uint32_t p, uint32_t n, uint32_t gcap) {
  bool dup = false, below = true;
  uint32_t top = 0;
  for (uint32_t m = 0; m < n; m++) {
    const uint32_t d = R[(p + m) & kRM].dev;
    top = max(top, d);
    below = below && d < gcap;
    for (uint32_t m2 = 0; m2 < m; m2++) dup = dup || R[(p + m2) & kRM].dev == d;
  }
  return (dup ? 1u : 0u) | (below ? 2u : 0u) | (top << 16);
}

// p2p order: per (comm, src, dst) channel, send seqs and recv seqs non-decreasing in file
// order (then FIFO-by-position pairing equals the reference's seq-sorted pairing).  Lanes
// hold send/recv pairs in file order (lane = element).
// REGION p2p
__device__ __noinline__ uint32_t p2p_order(const Chans ch, uint64_t off, const Rec ra, uint64_t next_seq, bool sendA,
                                           int lane) {
  uint32_t wflags = 0;
  const unsigned lt = (1u << lane) - 1;
  const unsigned gt = lane == 31 ? 0u : ~((2u << lane) - 1);
  uint64_t key = 0xFFFFFFFF00000000ull | lane, sseq = 0, rseq = 0;
  if (sendA) {
    key = ((uint64_t)ra.comm << 32) | ((uint64_t)ra.rank << 16) | ra.aux;
    sseq = ra.seq;
    rseq = next_seq;
  }
  const unsigned m = __match_any_sync(kFull, key);
  const unsigned lower = m & lt;
  const int pl = lower ? 31 - __clz(lower) : -1;  // previous pair of the channel in this batch
  const uint64_t ps = __shfl_sync(kFull, sseq, pl < 0 ? lane : pl);
  const uint64_t pr = __shfl_sync(kFull, rseq, pl < 0 ? lane : pl);
  // first pair of the channel in this batch: the warp's (private) channel table, looked up
  // with plain loads; channels new to this range are inserted one lane at a time
  const bool first = sendA && !lower;
  int e = -1;
  bool ins = false;
  if (first) {
    uint32_t h = (uint32_t)((key * 0x9E3779B97F4A7C15ull) >> 58) % kPC;
    for (int probe = 0; probe < kPC; probe++, h = (h + 1) % kPC) {
      const uint64_t k = ch.key(off + h);
      if (k == key) {
        if (sseq < ch.last_s(off + h) || rseq < ch.last_r(off + h)) wflags |= F_NONCANON;
        e = (int)h;
        break;
      }
      if (k == kNone) { ins = true; break; }
    }
    if (e < 0 && !ins) wflags |= F_NONCANON;  // more channels than the table holds
  }
  for (unsigned todo = __ballot_sync(kFull, ins); todo; todo &= todo - 1) {
    __syncwarp();
    if (lane == __ffs(todo) - 1) {
      uint32_t h = (uint32_t)((key * 0x9E3779B97F4A7C15ull) >> 58) % kPC;
      for (int probe = 0; probe < kPC; probe++, h = (h + 1) % kPC)
        if (ch.key(off + h) == kNone) {
          ch.key(off + h) = key;
          ch.first_s(off + h) = sseq; ch.first_r(off + h) = rseq;
          ch.last_s(off + h) = sseq; ch.last_r(off + h) = rseq;
          e = (int)h;
          break;
        }
      if (e < 0) wflags |= F_NONCANON;
    }
  }
  if (sendA && pl >= 0 && (sseq < ps || rseq < pr)) wflags |= F_NONCANON;
  const int e_grp = __shfl_sync(kFull, e, sendA ? __ffs(m) - 1 : lane);
  __syncwarp();
  if (sendA && (m & gt) == 0 && e_grp >= 0) { ch.last_s(off + e_grp) = sseq; ch.last_r(off + e_grp) = rseq; }
  __syncwarp();
  return wflags;
}

// REGION tree
// Peers of position j in the double binary tree (trees.py:57-106, decompose.py:227-255)
// packed as 7-bit codes (rank in bits [0,5), bit 5 = T1 edge carrying ceil(S/2), bit 6 =
// T2 edge carrying floor(S/2); an edge in both trees is one transfer of S), the count in
// bits [60,63).  T2 is always included; a T2-only edge is skipped when floor(S/2) == 0.
__device__ __forceinline__ unsigned long long tree_pack(int n, int j) {
  int a0, a1, a2, q0, q1, q2;
  tree_links(n, j, a0, a1, a2);                       // T1: rank == position
  tree_links(n, j == 0 ? n - 1 : j - 1, q0, q1, q2);  // T2: rank at position q is (q + 1) % n
  const int b0 = q0 < 0 ? -1 : (q0 + 1 == n ? 0 : q0 + 1);
  const int b1 = q1 < 0 ? -1 : (q1 + 1 == n ? 0 : q1 + 1);
  const int b2 = q2 < 0 ? -1 : (q2 + 1 == n ? 0 : q2 + 1);
  unsigned long long w = 0;
  int cnt = 0;
  auto put = [&](int r, uint32_t code) {
    w |= (unsigned long long)((uint32_t)r | (code << 5)) << (7 * cnt);
    cnt++;
  };
  if (a0 >= 0) put(a0, 1u | (a0 == b0 || a0 == b1 || a0 == b2 ? 2u : 0u));
  if (a1 >= 0) put(a1, 1u | (a1 == b0 || a1 == b1 || a1 == b2 ? 2u : 0u));
  if (a2 >= 0) put(a2, 1u | (a2 == b0 || a2 == b1 || a2 == b2 ? 2u : 0u));
  if (b0 >= 0 && b0 != a0 && b0 != a1 && b0 != a2) put(b0, 2u);
  if (b1 >= 0 && b1 != a0 && b1 != a1 && b1 != a2) put(b1, 2u);
  if (b2 >= 0 && b2 != a0 && b2 != a1 && b2 != a2) put(b2, 2u);
  return w | ((unsigned long long)cnt << 60);
}

__device__ __noinline__ unsigned long long tree_pack_big(int n, int j) { return tree_pack(n, j); }

__device__ __forceinline__ unsigned long long tree_peers(int n, int j) {
  return n <= kTreeLut ? cta_mem().tree_lut[n][j] : tree_pack_big(n, j);
}

// REGION expand_block
// a lane's follow-up on the warp's slot accumulator after a batch: entry e is full
// (key 0) or held another key (re-key to ``key``)
struct SAReq {
  uint32_t e, key;
  bool act;
};

// Edge-by-edge expansion of one VALID instance (the accumulators did not take it):
// statistics, then every transfer through one emission site.  Out of line to keep the
// accumulator fast path compact in the instruction cache.
template <bool SH>
__device__ __noinline__ uint32_t expand_direct(const FastParams& P, const ct_record* R, const Rec h, uint32_t p,
                                               uint64_t gidx, uint32_t j0, bool fastdev, bool packed,
                                               uint32_t devs, int algo) {
  Sink<SH> sk(P);
  const int n = (int)h.nranks, coll = h.coll();
  const unsigned long long base = min((unsigned long long)gidx, (1ull << 41) - 1) << 21;
  const uint64_t blk = h.count * (uint64_t)dtype_width(h.dtype());
  const bool scatter = coll == CT_COLL_ALLGATHER || coll == CT_COLL_REDUCESCATTER;
  const uint64_t s = scatter ? blk * (uint64_t)n : blk;
  const int g2 = P.g2;
  const bool ring = algo == CT_ALGO_RING, tree = algo == CT_ALGO_TREE;
  const bool rmap = ring && n == P.ex.ring_len;
  const int root_pos = rmap ? (h.has_root() ? (int)P.ex.ring_inv[h.aux] : 0) : (int)h.aux;
  const int skip_pos = coll == CT_COLL_BROADCAST ? (root_pos == 0 ? n - 1 : root_pos - 1)
                                                 : (coll == CT_COLL_REDUCE ? root_pos : -1);
  const uint64_t chunk = ring && coll == CT_COLL_ALLREDUCE ? ceil_div(s, (uint32_t)n) : 0;
  const bool simple = ring && coll == CT_COLL_ALLREDUCE && (uint64_t)(n - 1) * chunk < s;
  const uint64_t gen = 2 * s - 2 * chunk, dlt = chunk - (s - (uint64_t)(n - 1) * chunk);
  const uint64_t fixed = scatter ? s - blk : s;
  sk.stat(coll, (unsigned __int128)s);
  if (algo == CT_ALGO_COLLNET) {
    if (s == 0) return sk.flags;
  } else {
    if ((coll == CT_COLL_BROADCAST || coll == CT_COLL_REDUCE) && !h.has_root()) {
      sk.flags |= F_MISSING_ROOT;
      return sk.flags;
    }
    if (n == 1 || s == 0) return sk.flags;
  }
  if (rmap && !P.ex.ring_valid) { sk.flags |= F_BAD_RING; return sk.flags; }
  // tree shares
  const uint64_t share1 = s - s / 2, share2 = s / 2;
  auto devof = [&](int r) -> int { return packed ? (int)((devs >> (4 * r)) & 15u) : (int)R[(p + r) & kRM].dev; };
  int q = ring ? (int)j0 : 0;
  for (int i = 0; i < n; i++) {
    const int qn = q + 1 == n ? 0 : q + 1;
    const int rs = rmap ? (int)P.ex.ring_order[q] : q;  // sending rank
    int rd = 0, cnt;
    uint64_t rbytes = 0;
    unsigned long long w = 0;
    if (ring) {
      rd = rmap ? (int)P.ex.ring_order[qn] : qn;
      if (coll == CT_COLL_ALLREDUCE) {
        const int q2 = qn + 1 == n ? 0 : qn + 1;
        rbytes = simple ? gen + (qn == n - 1 ? dlt : 0) + (q2 == n - 1 ? dlt : 0)
                        : 2 * s - ring_block(s, chunk, qn) - ring_block(s, chunk, q2);
      } else {
        rbytes = q == skip_pos ? 0 : fixed;
      }
      cnt = rbytes != 0 ? 1 : 0;
    } else if (tree) {
      w = tree_peers(n, q);
      cnt = (int)(w >> 60);
    } else {
      cnt = 2;
    }
    const int me = devof(rs);
    for (int x = 0; x < cnt; x++) {
      int src = me, dst, sub;
      uint64_t bytes;
      if (ring) {
        dst = devof(rd); bytes = rbytes; sub = rd;
      } else if (tree) {
        const uint32_t c = (uint32_t)(w >> (7 * x));
        if ((c & 0x60) == 0x40 && share2 == 0) continue;  // T2-only edge of a 1-byte payload
        sub = (int)(c & 31);
        dst = devof(sub);
        bytes = (c & 0x60) == 0x60 ? s : ((c & 0x20) ? share1 : share2);
      } else {  // collnet: dev -> NET, NET -> dev
        src = x == 0 ? me : -2; dst = x == 0 ? -2 : me; bytes = s; sub = x;
      }
      if (fastdev) {  // every device of the block is < gcap
        sk.add((uint32_t)((coll * g2 + (src < 0 ? kNet : src + 2)) * g2 + (dst < 0 ? kNet : dst + 2)), bytes);
      } else {
        sk.rec_key = base | ((unsigned long long)rs << 11);
        sk.edge(coll, src, dst, (unsigned __int128)bytes, sub);
      }
    }
    q = qn;
  }
  return sk.flags;
}

// Expansion + statistics of one VALID collective instance whose head (rank 0) sits at
// ring position p; gidx is its global record index.  Rank-attributed rules (ct_common.cuh,
// SURVEY App. A): ring family -- the record at ring position q (rank order[q]) sends to
// order[q+1]; tree -- every rank sends to its peers in both trees; collnet -- every rank
// sends S to NET and receives S from it.  All edges leave through one emission site.
// Ring lanes start at different positions (j0) so their shared-memory reads spread over
// the banks.
template <bool SH>
__device__ __forceinline__ void expand_block(const FastParams& P, Sink<SH>& sk, const ct_record* R, const Rec& h,
                                             uint32_t p, uint64_t gidx, uint32_t j0, bool fastdev, bool packed,
                                             uint32_t devs, RingAcc& ra, int slot, SAE* sa, SAReq& sq) {
  const int n = (int)h.nranks, coll = h.coll();
  const unsigned long long base = min((unsigned long long)gidx, (1ull << 41) - 1) << 21;
  if (CT_UNLIKELY((h.count >> 40) != 0)) {
    for (int j = 0; j < n; j++) {
      Rec rc = h;
      rc.rank = (uint32_t)j;
      rc.dev = R[(p + j) & kRM].dev;
      sk.flags |= expand_wide<SH>(P, R, rc, p, base | ((unsigned long long)j << 11));
    }
    return;
  }
  const uint64_t blk = h.count * (uint64_t)dtype_width(h.dtype());
  const bool scatter = coll == CT_COLL_ALLGATHER || coll == CT_COLL_REDUCESCATTER;
  const uint64_t s = scatter ? blk * (uint64_t)n : blk;
  int algo = h.algo();
  if (coll == CT_COLL_ALLREDUCE) {
    if (algo == CT_ALGO_AUTO) algo = s < P.ex.tree_threshold ? CT_ALGO_TREE : CT_ALGO_RING;
  } else {
    if (algo == CT_ALGO_TREE || algo == CT_ALGO_COLLNET) { sk.flags |= F_WRONG_ALGO; return; }
    algo = CT_ALGO_RING;
  }
  const int g2 = P.g2;
  const bool ring = algo == CT_ALGO_RING, tree = algo == CT_ALGO_TREE;
  // ring family
  const bool rmap = ring && n == P.ex.ring_len;
  const uint64_t chunk = ring && coll == CT_COLL_ALLREDUCE ? ceil_div(s, (uint32_t)n) : 0;
  // allreduce blocks b[i] (decompose.py:104-107): chunk for i < n-1 and the remainder
  // s - (n-1)*chunk for i = n-1 unless s is tiny (then trailing blocks are empty)
  const bool simple = ring && coll == CT_COLL_ALLREDUCE && (uint64_t)(n - 1) * chunk < s;
  const uint64_t gen = 2 * s - 2 * chunk, dlt = chunk - (s - (uint64_t)(n - 1) * chunk);
  const uint64_t fixed = scatter ? s - blk : s;
  if (fastdev && packed && !rmap && n >= 2 && s != 0) {
    if (ring && (simple || scatter)) {  // per-lane register accumulator
      if (ra.add(sk, g2, (uint32_t)coll | ((uint32_t)n << 8), devs, simple ? gen : fixed, simple ? dlt : 0ull, s))
        return;
    }
    const bool rooted = coll == CT_COLL_BROADCAST || coll == CT_COLL_REDUCE;
    if (slot >= 0 && (!ring || simple || scatter || (rooted && h.has_root()))) {  // the warp's slot accumulator
      const uint32_t cls = tree ? 3u : (!ring ? 4u : (coll == CT_COLL_ALLREDUCE ? 0u : (coll == CT_COLL_ALLGATHER ? 1u
                           : (coll == CT_COLL_REDUCESCATTER ? 2u : (coll == CT_COLL_BROADCAST ? 5u : 6u)))));
      const uint32_t root = rooted ? h.aux & 7u : 0u;
      const uint32_t e = ((cls < 5u ? cls : (cls == 5u ? 8u : 16u) + root) + (uint32_t)slot * 5u) & (uint32_t)(kSE - 1);
      const uint32_t key =
          0x80000000u | (uint32_t)slot | (cls << 3) | ((uint32_t)coll << 6) | ((uint32_t)n << 9) | (root << 13);
      SAE& E = sa[e];
      if (E.key == key && E.devs == devs) {
        // low limbs and the count first (independent atomics in flight), then the carries
        const unsigned long long vg = tree ? s - s / 2 : (ring && !rooted ? (simple ? gen : fixed) : s);
        const unsigned long long vd = tree ? s / 2 : (simple ? dlt : 0ull);
        const uint32_t og = atomicAdd(&E.g[0], (uint32_t)vg);
        const uint32_t od = atomicAdd(&E.d[0], (uint32_t)vd);
        const uint32_t os = atomicAdd(&E.s[0], (uint32_t)s);
        const uint32_t oc = atomicAdd(&E.cnt, 1u);
        if (tree && s / 2 != 0) atomicAdd(&E.cnt2, 1u);
        const uint32_t hg = (uint32_t)(vg >> 32) + (og + (uint32_t)vg < og ? 1u : 0u);
        const uint32_t hd = (uint32_t)(vd >> 32) + (od + (uint32_t)vd < od ? 1u : 0u);
        const uint32_t hs = (uint32_t)(s >> 32) + (os + (uint32_t)s < os ? 1u : 0u);
        if (hg) atomicAdd(&E.g[1], hg);
        if (hd) atomicAdd(&E.d[1], hd);
        if (hs) atomicAdd(&E.s[1], hs);
        if (oc + 1 == P.sa_flush) { sq.e = e; sq.key = 0; sq.act = true; }  // write out after the batch
        return;
      }
      sq.e = e; sq.key = key; sq.act = true;  // re-key after the batch; this instance is expanded now
    }
  }
  sk.flags |= expand_direct<SH>(P, R, h, p, gidx, j0, fastdev, packed, devs, algo);
}

// nibble r of the result = nibble r ^ x of d (x < 8): the device word of a walk that
// visited rank k ^ x at step k, back in rank order
__device__ __forceinline__ uint32_t nibble_xor(uint32_t d, uint32_t x) {
  if (x & 1u) d = ((d >> 4) & 0x0F0F0F0Fu) | ((d << 4) & 0xF0F0F0F0u);
  if (x & 2u) d = __byte_perm(d, 0, 0x2301);
  if (x & 4u) d = __byte_perm(d, 0, 0x1032);
  return d;
}

__device__ __noinline__ void count_diag(uint32_t st) {
  if (st == ST_INCOMPAT) atomicAdd(&cta_mem().diag[CT_DIAG_INCOMPATIBLE], 1u);
  else if (st == ST_DUPDEV) atomicAdd(&cta_mem().diag[CT_DIAG_DUPLICATE_DEVICE], 1u);
  else if (st == ST_MISMATCH) atomicAdd(&cta_mem().diag[CT_DIAG_MISMATCHED_P2P], 1u);
}

}  // namespace

size_t fast_smem_bytes(int g2, int smem_hist) {
  size_t b = sizeof(WarpMem) * kWarps + sizeof(CtaMem);
  if (smem_hist) b += (size_t)kTypes * g2 * g2 * (sizeof(unsigned long long) + sizeof(unsigned int));
  return b;
}

template <bool SH>
// REGION kernel_init
__global__ void __launch_bounds__(kThreads, 1) fast_kernel(FastParams P) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  WarpMem* WM = reinterpret_cast<WarpMem*>(smem_raw);
  CtaMem& C = cta_mem();
  const int ncell = kTypes * P.g2 * P.g2;
  uint32_t* shl = hist_lo<true>(P);  // lo limbs, then hi limbs, then frequencies
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned lt = (1u << lane) - 1;
  WarpMem& W = WM[warp];

  // ---- init
  if (SH)
    for (int c = tid; c < 3 * ncell; c += kThreads) shl[c] = 0;
  if (tid < kTypes * 8) (&C.st[0][0])[tid] = 0;
  if (tid < 3) C.copy_first[tid] = kNone;
  if (tid < CT_NDIAG) C.diag[tid] = 0;
  if (tid < (kTreeLut + 1) * kTreeLut) {
    const int n = tid / kTreeLut, j = tid % kTreeLut;
    C.tree_lut[n][j] = j < n ? tree_pack(n, j) : 0ull;
  }
  if (tid == 0) {
    C.flags = 0; C.max_dev = -1; C.oor_key = kNone; C.of_cell = kNone;
  }
  if (lane < kSE) { W.sa[lane].key = 0; W.sa[lane].cnt = 0; }
  if (lane < kCS) {
    W.tag[lane] = kEmptyTag; W.sn[lane] = 0;
    W.cfirst[lane] = kNone; W.clast[lane] = kNone;
    for (int t = 0; t < 5; t++) W.tfirst[lane][t] = kNone;
  }
  const uint32_t gw = blockIdx.x * kWarps + warp;
  for (int e = lane; e < kPC; e += 32) P.chans.key((uint64_t)gw * kPC + e) = kNone;
  if (lane < kRing) mbar_init(&W.bar[lane], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();

  Sink<SH> sk(P);
  RingAcc racc;
  racc.tag = 0;
  racc.miss = 0;
  racc.thr = 8;
  int my_max_dev = -1;
  uint32_t copy_seen = 0;              // copy kinds this lane has seen (first index noted)
  uint32_t wflags = 0;
  unsigned long long tf_pend = (1ull << (kCS * 5)) - 1;  // (slot, type) first valid instance not yet noted
  uint32_t sc_comm = kEmptyTag;        // this lane's last (comm, slot) look-up
  int sc_slot = -1;

  // ---- this warp's range, cut at element starts
  const uint64_t NC = P.n_chunks;
  const uint64_t c0 = NC * gw / P.total_warps, c1 = NC * (gw + 1) / P.total_warps;
  bool bad0 = false;
  const uint64_t start = c0 == 0 ? 0 : first_start(P.recs, P.n, c0 * 32, bad0);
  const uint64_t end = c1 >= NC ? P.n : first_start(P.recs, P.n, c1 * 32, bad0);
  if (bad0) wflags |= F_NONCANON;
  if (start < end && !bad0) {
    // Positions are 32-bit, relative to the ring origin rb0 (chunk k0); relative chunk q
    // lives in ring slot q % kRing, so record rb0 + x sits at ring index x & kRM.
    const uint64_t k0 = start / 32;
    const uint64_t rb0 = k0 * 32;
    const uint32_t s0 = (uint32_t)(start - rb0);
    const uint32_t eo = (uint32_t)(end - rb0);
    const uint32_t lastc = (eo + 31) / 32;  // chunks [0, lastc) hold the range
    const ct_record* R = &W.ring[0][0];
    // chunk c of the range is gsrc[32c, 32c + 32): full below nfull, else the trace's tail
    const ct_record* gsrc = P.recs + rb0;
    const uint32_t nfull = (uint32_t)min((unsigned long long)((P.n - rb0) >> 5), 0xFFFFFFFFull);
    const uint32_t tail = (uint32_t)((P.n - rb0) & 31) * (uint32_t)sizeof(ct_record);
    auto chunk_bytes = [&](uint32_t c) -> uint32_t { return c < nfull ? 32u * (uint32_t)sizeof(ct_record) : tail; };
    for (uint32_t q = 0; q < (uint32_t)kRing && q < lastc; q++)
      if (lane == 0) bulk_load(W.ring[q], gsrc + (size_t)q * 32, chunk_bytes(q), &W.bar[q]);
    const uint32_t bar_a = smem_addr(&W.bar[0]), ring_a = smem_addr(&W.ring[0][0]);
    static_assert(sizeof(W.ring[0]) == 1024 && sizeof(W.bar[0]) == 8, "ring slot / barrier strides");
    uint32_t freed = 0;             // chunks released (slot re-issued)
    uint32_t qh = 0, qt = 0;        // element queue head / tail
    int cover = 0;                  // element lengths + copies (must equal the range's records)
    uint32_t cross = 0;             // 1: the last queued element extends past the scanned chunks
    uint32_t u = 0;                 // chunk of the oldest queued element (when the queue is not empty)
    uint32_t cnext = 0;             // next free entry of the seq-table pool
    const bool stream_only = (P.dbg & 4) != 0, no_expand = (P.dbg & 1) != 0;
    bool bail = false;
    uint32_t q = 0, waited = 0;  // next chunk to scan / chunks waited for
    uint32_t ns = 1;              // chunks scanned this step (two when both are in the ring)
    for (; q < lastc && !bail; q += ns) {
      ns = q + 1 < min(freed + (uint32_t)kRing, lastc) ? 2u : 1u;
      mbar_wait_a(bar_a + 8 * (q % kRing), (q / kRing) & 1);
      if (ns == 2) mbar_wait_a(bar_a + 8 * ((q + 1) % kRing), ((q + 1) / kRing) & 1);
      waited = q + ns;
      const uint32_t ql = q + ns - 1;  // last chunk of this step
      if (stream_only) {  // diagnostic: stream only (roofline experiments)
        for (uint32_t k = 0; k < ns; k++) {
          const uint32_t rel = (q + k) * 32 + lane;
          if (rel < eo) my_max_dev = max(my_max_dev, (int)(R[rel & kRM].dev ^ R[rel & kRM].rank));
        }
      } else {
        // REGION scan
        // ================= scan (lane = record; two chunks per step: records A and B)
        {
          // a copy: one transfer (decompose.py:397-406) and the first record of its kind
          auto copy_rec = [&](uint32_t rel, const uint4& b, int kind) {
            const unsigned long long cnt = reinterpret_cast<const unsigned long long*>(R + (rel & kRM))[0];
            const int ck = (int)(b.w >> 30);
            const uint32_t aux = b.z >> 16, aux2 = b.w & 0xFFFF;
            // d over copy GPU endpoints: with the CTA histogram, every in-table copy leaves a
            // cell with a frequency (read in the epilogue) and copy_edge_slow notes the rest
            if (!SH) {
              if (ck != CT_CKIND_H2D) my_max_dev = max(my_max_dev, (int)aux);
              if (ck != CT_CKIND_D2H) my_max_dev = max(my_max_dev, (int)aux2);
            }
            my_max_dev = max(my_max_dev, (int)(b.z & 0xFFFF));  // the record's own device (d, matrix.py:250-258)
            const int t = kind - CT_KIND_MEMCPY;  // statistics: the host sums the type's cells
            if (!no_expand) {
              const int src = ck == CT_CKIND_H2D ? -1 : (int)aux, dst = ck == CT_CKIND_D2H ? -1 : (int)aux2;
              // table rows: host 0, gpu g at g + 2 (an in-table endpoint is a row < g2)
              const uint32_t a = (uint32_t)(src + 2) & (src < 0 ? 0u : ~0u), bb = (uint32_t)(dst + 2) & (dst < 0 ? 0u : ~0u);
              if (max(a, bb) < (uint32_t)P.g2 && (cnt >> 63) == 0) {
                sk.add((uint32_t)((CT_T_EXPLICIT + t) * P.g2 * P.g2) + a * (uint32_t)P.g2 + bb, cnt);
              } else {  // an endpoint outside the table or >= 2^63 bytes (out of line)
                sk.flags |= copy_edge_slow<SH>(P, rb0 + rel, CT_T_EXPLICIT + t, src, dst, cnt);
              }
            }
            // first record of each copy kind: positions only grow, so a lane's first is its min
            const uint32_t bit = 1u << t;
            if (!(copy_seen & bit)) {
              copy_seen |= bit;
              atomicMin(&C.copy_first[t], rb0 + rel);
            }
          };
          const uint32_t relA = q * 32 + lane, relB = relA + 32;
          const bool actA = relA >= s0 && relA < eo, actB = ns == 2 && relB < eo;
          const uint4 bA = reinterpret_cast<const uint4*>(R + (relA & kRM))[1];  // any ring slot is readable
          const uint4 bB = reinterpret_cast<const uint4*>(R + (relB & kRM))[1];
          const int kindA = actA ? (int)((bA.w >> 16) & 7) : 7, kindB = actB ? (int)((bB.w >> 16) & 7) : 7;
          const bool isHA = (kindA == CT_KIND_COLLECTIVE && (bA.y >> 16) == 0) || kindA == CT_KIND_SEND;
          const bool isHB = (kindB == CT_KIND_COLLECTIVE && (bB.y >> 16) == 0) || kindB == CT_KIND_SEND;
          const bool isCpA = (uint32_t)(kindA - CT_KIND_MEMCPY) < 3u, isCpB = (uint32_t)(kindB - CT_KIND_MEMCPY) < 3u;
          const unsigned hmA = __ballot_sync(kFull, isHA), hmB = __ballot_sync(kFull, isHB);
          cover += (int)isCpA + (int)isCpB;  // copies tile the range too (summed over lanes at the end)
          const uint32_t nA = __popc(hmA);
          if (isHA) W.q[(qt + __popc(hmA & lt)) & kQM] = relA;
          if (isHB) W.q[(qt + nA + __popc(hmB & lt)) & kQM] = relB;
          if (qt == qh && (hmA | hmB)) u = hmA ? q : q + 1;  // the queue's oldest element starts here
          qt += nA + __popc(hmB);
          // only the step's last element can extend past it (else the layout is not canonical
          // and the tiling check fails): it waits for the next step
          const bool lastH = ns == 2 ? isHB : isHA;
          const uint32_t lrel = ns == 2 ? relB : relA;
          const uint4& lb = ns == 2 ? bB : bA;
          const uint32_t llen = (ns == 2 ? kindB : kindA) == CT_KIND_COLLECTIVE ? (lb.y & 0xFFFF) : 2u;
          cross = __any_sync(kFull, lastH && lrel + llen > (ql + 1) * 32) ? 1u : 0u;
          if (isCpA) copy_rec(relA, bA, kindA);
          if (isCpB) copy_rec(relB, bB, kindB);
        }
        __syncwarp();

        // REGION join_setup
        // ================= join + expand (lane = element), in batches of <= 32
        // elements wholly inside chunks <= q are joinable; join when 32 are ready or when
        // the ring is about to be full of unjoined records (the oldest one's chunk u)
        const bool pressure = ql + 1 + kDrainSlack >= u + kRing || ql + 1 == lastc;
        while (qt - qh - cross >= 32 || (pressure && qt - qh - cross > 0)) {
          const uint32_t nb = min(32u, qt - qh - cross);
          const bool act = (uint32_t)lane < nb;
          const uint32_t p = act ? W.q[(qh + lane) & kQM] : 0u;
          const Rec h = ring_rec(R, p);  // inactive lanes read slot 0 and are ignored
          const int kind = act ? h.kind() : 7;
          const bool isC = kind == CT_KIND_COLLECTIVE, isS = kind == CT_KIND_SEND;
          bool bad = false;

          // ---- comm slots of collective blocks
          int slot = -1;
          if (isC) {
            if (h.comm >= P.n_comms) { wflags |= F_COMM_RANGE; bad = true; }
            slot = h.comm == sc_comm ? sc_slot : find_slot(W, h.comm);
          }
          if (CT_UNLIKELY(__any_sync(kFull, isC && slot < 0))) {  // unseen comms (rare)
            slot = alloc_slots(W, isC && slot < 0, h.comm, slot, lane);
            if (slot == -2) { bad = true; slot = -1; }
          }
          if (isC) { sc_comm = h.comm; sc_slot = slot; }
          const int hs = slot < 0 ? 0 : slot;

          // ---- the comm's previous block: earlier in this batch (ring) or the slot table
          const unsigned same =
              __match_any_sync(kFull, isC ? (unsigned long long)h.comm : (0xFFFFFFFF00000000ull | lane));
          const unsigned lower = same & lt;
          const int pl = lower ? 31 - __clz(lower) : -1;
          const bool lastb = isC && (same >> lane) == 1u;  // no later block of this comm in the batch
          const uint32_t ppos = __shfl_sync(kFull, p, pl < 0 ? lane : pl);
          const uint32_t pn = __shfl_sync(kFull, h.nranks, pl < 0 ? lane : pl);
          const uint32_t tsn = isC ? W.sn[hs] : 0u;
          const bool hist = pl < 0 && tsn != 0;
          const uint32_t n = h.nranks;
          if (isC && (pl >= 0 ? pn != n : (tsn != 0 && tsn != n))) bad = true;  // grouping.py:104-108
          // a comm's first block in this range: its seq table gets n pooled entries
          for (unsigned need = __ballot_sync(kFull, isC && pl < 0 && tsn == 0 && n >= 1 && n <= (uint32_t)kMaxN);
               need; need &= need - 1) {
            const int L = __ffs(need) - 1;
            const uint32_t nL = __shfl_sync(kFull, n, L);
            const int sL = __shfl_sync(kFull, hs, L);
            if (lane == 0) W.cbase[sL] = cnext;
            cnext += nL;
          }
          if (CT_UNLIKELY(cnext > (uint32_t)kCP)) bad = true;  // more ranks in one range than the pool holds
          __syncwarp();
          const uint32_t cb = W.cbase[hs];
          {  // the element lies inside the range; lengths tile it (with the copies)
            const uint32_t len = isC ? n : (isS ? 2u : 0u);
            if (isC && (n == 0 || n > (uint32_t)kMaxN)) bad = true;
            if (p + len > eo) bad = true;
            cover += (int)len;
          }

          // REGION validate
          // ---- validation (lane walks its element)
          uint32_t st = ST_NONE;
          bool fastdev = false, packed = false;  // all devices < gcap / held in ``devs``
          bool uniform = true;                    // every rank of the block carries the head's seq
          uint32_t devs = 0;                    // device of rank j in bits [4j, 4j+4) (n <= 8, devices < 16)
          uint64_t rseq = 0;
          uint32_t rdev = 0;
          const uint32_t j0 = n == 0 ? 0u : ((n & (n - 1)) == 0 ? (uint32_t)lane & (n - 1) : (uint32_t)lane % n);
          // warp-uniform choice: every block of the batch has 8 ranks and none crosses the
          // ring's end (else one lane's fallback walk would run next to everyone's fast walk)
          const bool all8 = __all_sync(kFull, !isC || bad || (h.nranks == 8 && (p & kRM) <= (uint32_t)kRM - 7u));
          if (isC && !bad) {
            // compare raw words against the head: w4 comm, w5 nranks | rank << 16, w6 dev |
            // aux << 16 (aux = root when rooted), w7 aux2 | kc << 16 | ad << 24
            const uint4* R4 = reinterpret_cast<const uint4*>(R);
            const uint32_t hc0 = (uint32_t)h.count, hc1 = (uint32_t)(h.count >> 32);
            const uint32_t hw7 = h.aux2 | (h.kc << 16) | (h.ad << 24);
            const uint32_t rootm = h.has_root() ? 0xFFFF0000u : 0u, hw6 = h.aux << 16;
            uint32_t badw = 0, incw = 0, useqw = 0, m32 = 0;
            bool big = false, dup;
            const uint32_t hq0 = (uint32_t)h.seq, hq1 = (uint32_t)(h.seq >> 32);
            auto vrec = [&](uint32_t j) {  // one member record (independent across j)
              const uint32_t ix = (p + j) & kRM;
              const uint4 wa = R4[2 * ix], wb = R4[2 * ix + 1];
              const uint32_t x7 = wb.w ^ hw7;
              badw |= (wb.x ^ h.comm) | (wb.y ^ (n | (j << 16))) | (x7 & 0x00070000u);  // kind, comm, n, rank
              incw |= (wa.x ^ hc0) | (wa.y ^ hc1) | (x7 & 0x3F780000u) | ((wb.z ^ hw6) & rootm);  // signature
              useqw |= (wa.z ^ hq0) | (wa.w ^ hq1);  // every rank carries the head's seq
              const uint32_t dv = wb.z & 0xFFFF;
              big |= dv >= 32;
              m32 |= 1u << (dv & 31);
              devs |= (dv & 15u) << (4 * (j & 7));
            };
#ifndef CT_N8
#define CT_N8 1
#endif
            bool walked = false;
            if (CT_N8 && all8) {  // every block of the batch has 8 ranks: fully unrolled
              // The common case first: every member record is the head's record with its
              // own rank and device (same count, seq, comm, aux, aux2, kind byte and flags
              // byte).  One OR of XORs per word proves it; lane l visits rank k ^ (l & 7)
              // (bank spread) and keeps device nibbles in visit order.  Any difference or a
              // device >= 32 takes the field-by-field walk, which decides the same flags
              // exactly.
              const uint32_t jx = (uint32_t)lane & 7u;
              const uint32_t Bs = ring_a + 32u * (p & kRM), jx32 = jx << 5;
              const uint32_t nj = n | (jx << 16);
              uint32_t E = (p & kRM) > (uint32_t)kRM - 7u ? 1u : 0u, zor = 0, D = 0;  // (excluded by all8)
#pragma unroll
              for (uint32_t k = 0; k < 8; k++) {
                uint4 wa, wb;
                lds256(Bs + (jx32 ^ (k << 5)), wa, wb);
                E |= (wa.x ^ hc0) | (wa.y ^ hc1) | (wa.z ^ hq0) | (wa.w ^ hq1);
                E |= (wb.x ^ h.comm) | (wb.y ^ nj ^ (k << 16)) | ((wb.z ^ hw6) & 0xFFFF0000u) | (wb.w ^ hw7);
                zor |= wb.z;
                m32 |= 1u << (wb.z & 31u);
                D |= (wb.z & 15u) << (4 * k);
              }
              walked = E == 0 && (zor & 0xFFE0u) == 0;
              if (CT_LIKELY(walked)) devs = nibble_xor(D, jx);  // nibble r = device of rank r
              else m32 = 0;
            }
            if (!walked) {
              uint32_t j = j0;
              uint32_t i = 0;
              for (; i + 1 < n; i += 2) {
                const uint32_t j1 = j + 1 == n ? 0 : j + 1;
                vrec(j);
                vrec(j1);
                j = j1 + 1 == n ? 0 : j1 + 1;
              }
              if (i < n) vrec(j);
            }
            if (badw) bad = true;
            uniform = useqw == 0;
            if (CT_LIKELY(!big)) {  // devices < 32: the mask holds them all
              dup = __popc(m32) != (int)n;  // pairwise distinct devices
              fastdev = P.gcap >= 32 || (m32 >> P.gcap) == 0;
              my_max_dev = max(my_max_dev, 31 - __clz(m32));  // the block's devices (d)
            } else {
              const uint32_t info = block_devices(R, p, n, (uint32_t)P.gcap);
              dup = (info & 1u) != 0;
              fastdev = (info & 2u) != 0;
              my_max_dev = max(my_max_dev, (int)(info >> 16));
            }
            packed = !big && n <= 8 && (m32 >> 16) == 0;
            st = incw ? ST_INCOMPAT : (dup ? ST_DUPDEV : ST_VALID);
          } else if (isS) {
            const Rec r = ring_rec(R, p + 1);
            if (r.kind() != CT_KIND_RECV || r.comm != h.comm || r.aux != h.rank || r.rank != h.aux) bad = true;
            st = (r.count != h.count || r.dtype() != h.dtype()) ? ST_MISMATCH : ST_VALID;  // decompose.py:362-372
            rseq = r.seq;
            rdev = r.dev;
            my_max_dev = max(my_max_dev, (int)max(h.dev, rdev));
          }
          {  // per (comm, rank) seq strictly increasing from the comm's previous block
            const bool pu = __shfl_sync(kFull, uniform, pl < 0 ? lane : pl);
            const unsigned long long pq = __shfl_sync(kFull, h.seq, pl < 0 ? lane : pl);
            if (isC && !bad && (pl >= 0 || hist)) {
              const bool tu = pl < 0 && W.uni[hs];
              if (CT_LIKELY(uniform && (pl >= 0 ? pu : tu))) {  // one comparison per block
                if (!((pl >= 0 ? pq : W.useq[hs]) < h.seq)) bad = true;
              } else {  // rank by rank
                if (!seq_order_ranks(R, p, n, pl >= 0 ? ppos : 0u, pl >= 0, tu, W.useq[hs], W.cpool, cb)) bad = true;
              }
            }
          }
          if (CT_UNLIKELY(__any_sync(kFull, bad))) { wflags |= F_NONCANON; bail = true; break; }
          if (__any_sync(kFull, isS)) wflags |= p2p_order(P.chans, (uint64_t)gw * kPC, h, rseq, isS, lane);
          if (CT_UNLIKELY(st > ST_VALID)) count_diag(st);

          // REGION tables
          // ---- tables: the last block of each comm in the batch; first occurrences
          __syncwarp();  // every lane has read the tables
          if (isC) {
            const uint64_t gi = rb0 + p;
            if (pl < 0 && tsn == 0) W.cfirst[hs] = gi;  // first block of this comm in the range
            if (lastb) {
              W.sn[hs] = n;
              W.clast[hs] = gi;
              W.uni[hs] = uniform ? 1u : 0u;
              W.useq[hs] = h.seq;
            }
          }
          // the last block of each comm becomes the slot's seq table: one block per step,
          // lane = rank
          for (unsigned lb = __ballot_sync(kFull, lastb && !uniform); lb; lb &= lb - 1) {
            const int L = __ffs(lb) - 1;
            const uint32_t pL = __shfl_sync(kFull, p, L), nL = __shfl_sync(kFull, n, L);
            const int sL = __shfl_sync(kFull, hs, L);
            if ((uint32_t)lane < nL) W.cpool[(W.cbase[sL] + lane) & (kCP - 1)] = R[(pL + lane) & kRM].seq;
          }
          {  // first valid instance per (comm slot, type): only until recorded once
            const unsigned long long bit = (isC && st == ST_VALID) ? 1ull << (hs * 5 + h.coll()) : 0ull;
            const bool rec = (bit & tf_pend) != 0;
            if (CT_UNLIKELY(__any_sync(kFull, rec))) {
              if (rec) note_min_smem(&W.tfirst[hs][h.coll()], rb0 + p);
              const unsigned lo = __reduce_or_sync(kFull, rec ? (unsigned)bit : 0u);
              const unsigned hi = __reduce_or_sync(kFull, rec ? (unsigned)(bit >> 32) : 0u);
              tf_pend &= ~(((unsigned long long)hi << 32) | lo);
            }
          }
          __syncwarp();

          // REGION expand_call
          // ---- expansion + accumulation of valid elements
          SAReq sq{0u, 0u, false};
          if (st == ST_VALID && !no_expand) {
            if (isC) {
              expand_block<SH>(P, sk, R, h, p, rb0 + p, j0, fastdev, packed, devs, racc, slot, W.sa, sq);
            } else {  // matched send/recv pair (decompose.py:319-339)
              const unsigned __int128 nbytes = (unsigned __int128)h.count * (unsigned)dtype_width(h.dtype());
              sk.stat(CT_T_SENDRECV, nbytes);
              sk.rec_key = (1ull << 62) | (min((unsigned long long)(rb0 + p), (1ull << 41) - 1) << 21);
              if (rdev != h.dev) sk.edge(CT_T_SENDRECV, (int)h.dev, (int)rdev, nbytes);
            }
          }
          if (CT_UNLIKELY(__any_sync(kFull, sq.act))) {  // slot accumulators: one lane per entry writes out / re-keys
            __syncwarp();
            const unsigned grp = __match_any_sync(kFull, sq.act ? sq.e : (0x100u | (uint32_t)lane));
            if (sq.act && (grp >> lane) == 1u) sk.flags |= sa_flush<SH>(P, &W.sa[sq.e], sq.key, devs);
            __syncwarp();
          }
          qh += nb;
          if (qt != qh) u = W.q[qh & kQM] / 32;
        }
        if (bail) break;
      }

      // REGION release
      // ---- release chunks no element still needs; their slots refill
      const uint32_t keep = qt != qh ? u : ql + 1;
      if (keep > freed) {
        __syncwarp();
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        {  // lane j refills the slot of released chunk freed + j (keep - freed <= kRing)
          const uint32_t c = freed + (uint32_t)lane, nq = c + kRing;
          if (c < keep && nq < lastc)
            bulk_load_a(ring_a + 1024 * (c % kRing), gsrc + (size_t)nq * 32, chunk_bytes(nq), bar_a + 8 * (c % kRing));
          freed = keep;
        }
      }
    }
    if (!bail && !(P.dbg & 4)) {  // element lengths must tile the range exactly
      const int tot = __reduce_add_sync(kFull, cover);
      if (tot != (int)(eo - s0)) wflags |= F_NONCANON;
    }
    const uint32_t issued = min(freed + (uint32_t)kRing, lastc);
    for (uint32_t c = waited; c < issued; c++)  // drain outstanding bulk copies
      mbar_wait(&W.bar[c % kRing], (c / kRing) & 1);
  }

  // REGION epilogue
  // ---- per-warp summaries for the cross-range check and first-occurrence keys
  __syncwarp();
  if (lane < kCS) {
    WarpSlot& o = P.slots[(size_t)gw * kCS + lane];
    const uint32_t cm = W.tag[lane];
    o.comm = cm;
    o.n = W.sn[lane];
    o.coll_first = W.cfirst[lane];
    o.coll_last = W.clast[lane];
    if (cm != kEmptyTag && cm < P.n_comms) {
      if (W.cfirst[lane] != kNone) atomicMin(&P.comm_first[cm], W.cfirst[lane]);
      for (int t = 0; t < 5; t++)
        if (W.tfirst[lane][t] != kNone) atomicMin(&P.type_comm_first[(size_t)t * P.n_comms + cm], W.tfirst[lane][t]);
    }
  }

  // ---- CTA epilogue: drain caches, one global merge
  if (racc.tag) racc.flush(sk, P.g2);
  if (lane < kSE && W.sa[lane].key && W.sa[lane].cnt) sk.flags |= sa_flush<SH>(P, &W.sa[lane], 0u, 0ull);
  atomicMax(&C.max_dev, my_max_dev);
  if (sk.flags | wflags) atomicOr(&C.flags, sk.flags | wflags);
  __syncthreads();

  GlobalState* G = P.st;
  if (SH) {
    uint32_t of = 0;
    int cmx = -1;  // copy GPU endpoints (d inference): the copy planes' touched cells
    const int copy0 = CT_T_EXPLICIT * P.g2 * P.g2;
    for (int c = tid; c < ncell; c += kThreads) {
      const unsigned int f = shl[2 * ncell + c];
      if (!f) continue;
      if (c >= copy0) cmx = max(cmx, max((c / P.g2) % P.g2, c % P.g2) - 2);
      const unsigned long long bb = shl[c] | ((unsigned long long)shl[ncell + c] << 32);
      const unsigned long long old = atomicAdd(P.cells + c, bb);
      if (old + bb < old) { of |= F_OVERFLOW; atomicMin(&G->of_cell, (unsigned long long)c); }
      atomicAdd(P.freq + c, (unsigned long long)f);
    }
    if (of) atomicOr(&C.flags, of);
    if (cmx >= 0) atomicMax(&C.max_dev, cmx);
  }
  if (tid < kTypes) {
    const uint32_t* L = C.st[tid];
    const unsigned long long c = L[4] | ((unsigned long long)L[5] << 32);
    if (c) {
      const unsigned long long lo = L[0] | ((unsigned long long)L[1] << 32);
      const unsigned long long hi = L[2] | ((unsigned long long)L[3] << 32);
      const unsigned long long old = atomicAdd(&G->pay_lo[tid], lo);
      atomicAdd(&G->pay_hi[tid], hi + (old + lo < old ? 1ull : 0ull));
      atomicAdd(&G->calls[tid], c);
    }
  }
  if (tid < CT_NDIAG && C.diag[tid]) atomicAdd(&G->diag[tid], (unsigned long long)C.diag[tid]);
  if (tid < 3 && C.copy_first[tid] != kNone) atomicMin(&G->copy_first[tid], C.copy_first[tid]);
  __syncthreads();
  if (tid == 0) {
    if (C.flags) atomicOr(&G->flags, C.flags);
    atomicMax(&G->max_dev, C.max_dev);
    if (C.oor_key != kNone) atomicMin(&G->oor_key, C.oor_key);
    if (C.of_cell != kNone) atomicMin(&G->of_cell, C.of_cell);
  }
}

// REGION range_check
template __global__ void fast_kernel<true>(FastParams);
template __global__ void fast_kernel<false>(FastParams);

// Cross-range seq-order check, one thread per (warp range, item): items [0, kCS) are the
// collective comm slots (nranks equal and per-rank seq strictly increasing from the last
// block of the nearest earlier range holding the comm to this range's first block), items
// [kCS, kCS + kPC) the p2p channels (send and recv seqs non-decreasing across ranges).
__global__ void range_check_kernel(const ct_record* recs, const WarpSlot* slots, const Chans chans,
                                   uint32_t total_warps, GlobalState* st) {
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint32_t per = kCS + kPC;
  if (t >= (uint64_t)total_warps * per) return;
  const uint32_t w = (uint32_t)(t / per), item = (uint32_t)(t % per);
  if (w == 0) return;
  if (item < (uint32_t)kCS) {
    const WarpSlot& me = slots[(size_t)w * kCS + item];
    if (me.comm == kEmptyTag || me.n == 0) return;
    for (int32_t v = (int32_t)w - 1; v >= 0; v--)
      for (int q = 0; q < kCS; q++) {
        const WarpSlot& o = slots[(size_t)v * kCS + q];
        if (o.comm != me.comm || o.n == 0) continue;
        bool ok = o.n == me.n;
        for (uint32_t r = 0; ok && r < me.n; r++) ok = recs[o.coll_last + r].seq < recs[me.coll_first + r].seq;
        if (!ok) atomicOr(&st->flags, F_NONCANON);
        return;
      }
    return;
  }
  const uint64_t me = (uint64_t)w * kPC + (item - kCS);
  const uint64_t mk = chans.key(me);
  if (mk == kNone) return;
  // the nearest earlier range holding the channel: every table is open-addressed with the
  // same hash, so membership is a short probe sequence (stops at an empty entry)
  const uint32_t h0 = (uint32_t)((mk * 0x9E3779B97F4A7C15ull) >> 58) % kPC;
  for (int32_t v = (int32_t)w - 1; v >= 0; v--)
    for (uint32_t probe = 0, h = h0; probe < (uint32_t)kPC; probe++, h = (h + 1) % kPC) {
      const uint64_t o = (uint64_t)v * kPC + h;
      const uint64_t k = chans.key(o);
      if (k == kNone) break;
      if (k != mk) continue;
      if (chans.first_s(me) < chans.last_s(o) || chans.first_r(me) < chans.last_r(o)) atomicOr(&st->flags, F_NONCANON);
      return;
    }
}

}  // namespace ct
