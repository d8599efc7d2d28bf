// Fast path: warp-autonomous streaming layout check + join + expand + accumulate
// (design notes in ct_fast.cuh).
#include "ct_fast.cuh"

namespace ct {

namespace {

constexpr uint64_t kNone = ~0ull;
constexpr uint32_t kEmptyTag = 0xFFFFFFFFu;
constexpr unsigned kFull = 0xFFFFFFFFu;

struct __align__(16) WarpMem {
  ct_record ring[kRing][32];                 // TMA ring: chunk k lives in slot (k - k0) % kRing
  unsigned long long bar[kRing];
  unsigned long long cseq[kCS][kMaxN];       // last collective block: seq per rank
  unsigned long long cfirst[kCS], clast[kCS];
  unsigned long long tfirst[kCS][5];
  uint16_t cdev[kCS][kMaxN];                 // last collective block: device per rank
  uint32_t tag[kCS];                         // comm id of the slot
  uint32_t sn[kCS];                          // collective nranks of the slot (0: none yet)
  uint32_t sver[kCS];                        // last block's devices pairwise distinct
};

struct __align__(16) CtaMem {
  unsigned long long calls[kTypes], pay_lo[kTypes], pay_hi[kTypes];
  unsigned long long copy_first[3];
  unsigned int diag[CT_NDIAG];
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

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, unsigned long long* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
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

// conflict-free 32-B record read from shared memory: lanes alternate which 16-B half
// they fetch first so each quarter-warp covers all 32 banks
__device__ __forceinline__ Rec load_swz(const ct_record* base, int i) {
  const uint4* q = reinterpret_cast<const uint4*>(base + i);
  const int f = (i >> 2) & 1;
  const uint4 x = q[f], y = q[f ^ 1];
  return f ? unpack(y, x) : unpack(x, y);
}

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
template <bool SH>  // SH: CTA histogram in shared memory (else global atomics)
struct Acc {
  // two small register caches: transfer cells and per-type statistics; a miss evicts the
  // older entry into the CTA histogram (shared-memory atomics)
  uint32_t ctag[2], stag[2];
  unsigned long long csum[2], ssum[2];
  uint32_t ccnt[2], scnt[2];
  uint32_t flags;
  unsigned long long* hb;
  void* hf;
  bool smem;
  CtaMem* C;
  int g2, gcap;
  bool explicit_d;
  unsigned long long rec_key;  // (class << 62) | (element << 21) | (src rank << 11) for oor ordering
  unsigned long long oor_key;
  unsigned long long of_cell;

  __device__ void init(CtaMem* c, unsigned long long* b, void* f, bool sm, int g2_, int gcap_, bool ex) {
    ctag[0] = ctag[1] = stag[0] = stag[1] = kEmptyTag;
    csum[0] = csum[1] = ssum[0] = ssum[1] = 0;
    ccnt[0] = ccnt[1] = scnt[0] = scnt[1] = 0;
    flags = 0; hb = b; hf = f; smem = sm; C = c; g2 = g2_; gcap = gcap_; explicit_d = ex;
    rec_key = 0; oor_key = kNone; of_cell = kNone;
  }

  __device__ __forceinline__ void flush_cell(uint32_t key, unsigned long long v, uint32_t c) {
    const unsigned long long old = atomicAdd(hb + key, v);
    if (old + v < old) { flags |= F_OVERFLOW; if (key < of_cell) of_cell = key; }
    if (SH) atomicAdd(static_cast<unsigned int*>(hf) + key, c);
    else atomicAdd(static_cast<unsigned long long*>(hf) + key, (unsigned long long)c);
  }

  __device__ __forceinline__ void flush_stat(uint32_t t, unsigned long long v, uint32_t c) {
    const unsigned long long old = atomicAdd(&C->pay_lo[t], v);
    if (old + v < old) atomicAdd(&C->pay_hi[t], 1ull);
    atomicAdd(&C->calls[t], (unsigned long long)c);
  }

  __device__ __forceinline__ void add_cell(uint32_t key, unsigned long long v) {
    if (ctag[0] == key) {
      const unsigned long long s = csum[0] + v;
      if (s < v) { flags |= F_OVERFLOW; if (key < of_cell) of_cell = key; }
      csum[0] = s; ccnt[0]++;
    } else if (ctag[1] == key) {
      const unsigned long long s = csum[1] + v;
      if (s < v) { flags |= F_OVERFLOW; if (key < of_cell) of_cell = key; }
      csum[1] = s; ccnt[1]++;
    } else {
      if (ctag[1] != kEmptyTag) flush_cell(ctag[1], csum[1], ccnt[1]);
      ctag[1] = ctag[0]; csum[1] = csum[0]; ccnt[1] = ccnt[0];
      ctag[0] = key; csum[0] = v; ccnt[0] = 1;
    }
  }

  // payload sums are 128-bit in the CTA: flush before a register entry would wrap
  __device__ __forceinline__ void add_stat(uint32_t t, unsigned long long v) {
    if (stag[0] == t) {
      if (ssum[0] + v < v) { flush_stat(t, ssum[0], scnt[0]); ssum[0] = v; scnt[0] = 1; }
      else { ssum[0] += v; scnt[0]++; }
    } else if (stag[1] == t) {
      if (ssum[1] + v < v) { flush_stat(t, ssum[1], scnt[1]); ssum[1] = v; scnt[1] = 1; }
      else { ssum[1] += v; scnt[1]++; }
    } else {
      if (stag[1] != kEmptyTag) flush_stat(stag[1], ssum[1], scnt[1]);
      stag[1] = stag[0]; ssum[1] = ssum[0]; scnt[1] = scnt[0];
      stag[0] = t; ssum[0] = v; scnt[0] = 1;
    }
  }

  __device__ __forceinline__ void drain() {
    if (ctag[0] != kEmptyTag) flush_cell(ctag[0], csum[0], ccnt[0]);
    if (ctag[1] != kEmptyTag) flush_cell(ctag[1], csum[1], ccnt[1]);
    if (stag[0] != kEmptyTag) flush_stat(stag[0], ssum[0], scnt[0]);
    if (stag[1] != kEmptyTag) flush_stat(stag[1], ssum[1], scnt[1]);
    ctag[0] = ctag[1] = stag[0] = stag[1] = kEmptyTag;
  }

  // stats: calls += 1, payload += s (128-bit capable)
  __device__ __forceinline__ void stat(int type, unsigned __int128 s) {
    if ((s >> 63) == 0) { add_stat((uint32_t)type, (unsigned long long)s); return; }
    const unsigned long long lo = (unsigned long long)s;
    unsigned long long hi = (unsigned long long)(s >> 64);
    const unsigned long long old = atomicAdd(&C->pay_lo[type], lo);
    if (old + lo < old) hi += 1;
    atomicAdd(&C->pay_hi[type], hi);
    atomicAdd(&C->calls[type], 1ull);
  }

  __device__ __forceinline__ void out_of_range(unsigned long long k) {
    flags |= explicit_d ? F_OOR : F_CAP;
    if (k < oor_key) oor_key = k;
  }

  // endpoint: gpu g (>= 0), -1 host, -2 net.  ``sub`` orders transfers inside one
  // decomposition (destination rank of a collective edge, transfers are sorted by rank
  // pair, decompose.py:92; 0/1 for collnet) for the EndpointOutOfRange message.
  __device__ __forceinline__ void edge(int type, int src, int dst, unsigned __int128 bytes, int sub = 0) {
    const int a = src == -1 ? kHost : (src == -2 ? kNet : src + 2);
    const int b = dst == -1 ? kHost : (dst == -2 ? kNet : dst + 2);
    if (src >= gcap || dst >= gcap) {
      const unsigned long long k = rec_key | ((unsigned long long)min(sub, 1023) << 1);
      if (src >= gcap) out_of_range(k);
      if (dst >= gcap) out_of_range(k | 1);
      return;
    }
    if ((bytes >> 63) != 0) { flags |= F_OVERFLOW; return; }
    add_cell((uint32_t)((type * g2 + a) * g2 + b), (unsigned long long)bytes);
  }
};

constexpr uint32_t kRM = kRing * 32 - 1;  // ring index mask (kRing is a power of two)
static_assert((kRing & (kRing - 1)) == 0, "kRing must be a power of two");

// device of a trace record (absolute index) held in the warp's ring
struct WinDev {
  const ct_record* R;
  uint64_t rb0;  // record index of ring position 0
  __device__ __forceinline__ uint32_t dev_of(uint64_t abs) const { return R[(uint32_t)(abs - rb0) & kRM].dev; }
};

__device__ __forceinline__ int find_slot(const WarpMem& W, uint32_t comm) {
  int s = -1;
#pragma unroll
  for (int k = 0; k < kCS; k++)
    if (W.tag[k] == comm) s = k;
  return s;
}

// no set bit in [lo, lo + len) of a 64-bit window mask (lo + len <= 64)
__device__ __forceinline__ bool range_clear(unsigned long long mask64, uint32_t lo, uint32_t len) {
  if (len == 0) return true;
  const unsigned long long m = len >= 64 ? ~0ull : ((1ull << len) - 1);
  return ((mask64 >> lo) & m) == 0;
}

__device__ __forceinline__ void note_min_smem(unsigned long long* slot, unsigned long long v) {
  if (v < *slot) atomicMin(slot, v);
}

// Predecessor check of a non-start element member.  q0..q4 are the predecessor's words
// (comm | nranks, rank | kc, ad, aux | count lo | count hi); w2 is the member's own kc/ad/aux.
// Collective members must continue their block (same comm and nranks, rank + 1); the
// signature (coll, algo, count, dtype, root; grouping.py:78-79) must match, otherwise the
// block is incompatible.  A recv must follow its counterpart send (decompose.py:323-330);
// count/dtype disagreement makes the pair mismatched (decompose.py:362-372).
__device__ __forceinline__ void member_check(const Rec& me, uint32_t w2, uint32_t q0, uint32_t q1, uint32_t q2,
                                             uint32_t q3, uint32_t q4, bool& sfail, bool& gfail, bool& mis) {
  const int kind = me.kind();
  const uint32_t pk = q2 & 7;
  if (kind == CT_KIND_COLLECTIVE) {
    if (pk != CT_KIND_COLLECTIVE || q0 != me.comm || (q1 & 0xFFFF) != me.nranks || (q1 >> 16) + 1 != me.rank) {
      sfail = true;
      return;
    }
    const uint32_t m = 0x3F78u | (me.has_root() ? 0xFFFF0000u : 0u);
    if (((q2 ^ w2) & m) != 0 || q3 != (uint32_t)me.count || q4 != (uint32_t)(me.count >> 32)) gfail = true;
  } else if (kind == CT_KIND_RECV) {
    if (pk != CT_KIND_SEND || q0 != me.comm || (q1 >> 16) != me.aux || (q2 >> 16) != me.rank) {
      sfail = true;
      return;
    }
    if (q3 != (uint32_t)me.count || q4 != (uint32_t)(me.count >> 32) || ((q2 >> 10) & 15) != (uint32_t)me.dtype())
      mis = true;
  } else {
    sfail = true;  // sends, copies and unknown kinds never continue an element
  }
}

// seq order of a collective member against the same rank of the comm's previous block
// (in-window ``pseq`` or the per-warp table) and device inheritance from the table
__device__ __forceinline__ void order_check(const WarpMem& W, const Rec& me, uint32_t info, uint64_t pseq,
                                            uint32_t& wflags, bool& devf) {
  const int s = info & 15;
  const uint32_t r = me.rank;
  bool have = (info & (1u << 10)) != 0;
  if (!have && (info & (1u << 11))) { pseq = W.cseq[s][r]; have = true; }
  if (have && !(pseq < me.seq)) wflags |= F_NONCANON;  // strictly increasing per (comm, rank)
  devf = !((info & (1u << 12)) && W.cdev[s][r] == me.dev);
}

// pairwise-distinct devices of the block of n records starting at ring index i0
__device__ __noinline__ bool devices_distinct(const ct_record* R, uint32_t i0, uint32_t n) {
  uint64_t seen0 = 0, seen1 = 0, seen2 = 0, seen3 = 0;
  for (uint32_t m = 0; m < n; m++) {
    const uint32_t d = R[(i0 + m) & kRM].dev;
    if (d < 256) {
      const uint64_t bit = 1ull << (d & 63);
      const uint32_t wi = d >> 6;
      const uint64_t wd = wi == 0 ? seen0 : wi == 1 ? seen1 : wi == 2 ? seen2 : seen3;
      if (wd & bit) return false;
      if (wi == 0) seen0 |= bit; else if (wi == 1) seen1 |= bit; else if (wi == 2) seen2 |= bit; else seen3 |= bit;
    } else {
      for (uint32_t m2 = 0; m2 < m; m2++)
        if (R[(i0 + m2) & kRM].dev == d) return false;
    }
  }
  return true;
}

// p2p order: per (comm, src, dst) channel, send seqs and recv seqs non-decreasing in file
// order (then FIFO-by-position pairing equals the reference's seq-sorted pairing)
__device__ __forceinline__ void p2p_order(P2PEntry* chan, const Rec& ra, uint64_t next_seq, bool sendA, int lane,
                                          unsigned lt, unsigned gt, uint32_t& wflags) {
  uint64_t key = 0xFFFFFFFF00000000ull | lane, sseq = 0, rseq = 0;
  if (sendA) {  // the recv is the next record (elements are whole inside a window)
    key = ((uint64_t)ra.comm << 32) | ((uint64_t)ra.rank << 16) | ra.aux;
    sseq = ra.seq;
    rseq = next_seq;
  }
  const unsigned m = __match_any_sync(kFull, key);
  const unsigned lower = m & lt;
  const int pl = lower ? 31 - __clz(lower) : -1;  // in-window previous pair of the channel
  const uint64_t ps = __shfl_sync(kFull, sseq, pl < 0 ? lane : pl);
  const uint64_t pr = __shfl_sync(kFull, rseq, pl < 0 ? lane : pl);
  int e = -1;
  if (sendA && !lower) {  // first pair of the channel in this window: channel table
    uint32_t h = (uint32_t)((key * 0x9E3779B97F4A7C15ull) >> 58) % kPC;
    for (int probe = 0; probe < kPC; probe++, h = (h + 1) % kPC) {
      const unsigned long long old = atomicCAS(reinterpret_cast<unsigned long long*>(&chan[h].key), kNone, key);
      if (old == kNone) {  // first pair of the channel in this range
        chan[h].first_s = sseq; chan[h].first_r = rseq;
        chan[h].last_s = sseq; chan[h].last_r = rseq;
        e = (int)h;
        break;
      }
      if (old == key) {
        if (sseq < chan[h].last_s || rseq < chan[h].last_r) wflags |= F_NONCANON;
        e = (int)h;
        break;
      }
    }
    if (e < 0) wflags |= F_NONCANON;  // more channels than the table holds
  }
  if (sendA && pl >= 0 && (sseq < ps || rseq < pr)) wflags |= F_NONCANON;
  const int e_grp = __shfl_sync(kFull, e, sendA ? __ffs(m) - 1 : lane);
  __syncwarp();
  if (sendA && (m & gt) == 0 && e_grp >= 0) { chan[e_grp].last_s = sseq; chan[e_grp].last_r = rseq; }
  __syncwarp();
}

// expansion + accumulation of one record of a processed element (status ``st``)
template <bool SH>
__device__ __forceinline__ void expand_record(const FastParams& P, Acc<SH>& acc, const WinDev& wdv, const Rec& me,
                                              uint64_t abs, uint32_t st, uint64_t head, int& max_dev,
                                              unsigned long long& cf0, unsigned long long& cf1,
                                              unsigned long long& cf2) {
  const int kind = me.kind();
  max_dev = max(max_dev, (int)me.dev);
  if (kind == CT_KIND_COLLECTIVE) {
    if (st != ST_VALID) return;
    acc.rec_key = (min((unsigned long long)head, (1ull << 41) - 1) << 21) | ((unsigned long long)min(me.rank, 1023u) << 11);
    if ((me.count >> 40) == 0) expand_collective<uint64_t>(P.ex, wdv, acc, me, head);
    else expand_collective<unsigned __int128>(P.ex, wdv, acc, me, head);
  } else if (kind == CT_KIND_SEND) {
    if (st != ST_VALID) return;
    const unsigned __int128 nb = (unsigned __int128)me.count * (unsigned)dtype_width(me.dtype());
    acc.stat(CT_T_SENDRECV, nb);
    acc.rec_key = (1ull << 62) | (min((unsigned long long)abs, (1ull << 41) - 1) << 21);
    const int rdev = (int)wdv.dev_of(abs + 1);
    if (rdev != (int)me.dev) acc.edge(CT_T_SENDRECV, (int)me.dev, rdev, nb);
  } else if (kind >= CT_KIND_MEMCPY) {
    const int ck = me.ckind();
    if (ck != CT_CKIND_H2D) max_dev = max(max_dev, (int)me.aux);
    if (ck != CT_CKIND_D2H) max_dev = max(max_dev, (int)me.aux2);
    const int t = CT_T_EXPLICIT + (kind - CT_KIND_MEMCPY);
    acc.stat(t, (unsigned __int128)me.count);
    acc.rec_key = (2ull << 62) | (min((unsigned long long)abs, (1ull << 41) - 1) << 21);
    acc.edge(t, ck == CT_CKIND_H2D ? -1 : (int)me.aux, ck == CT_CKIND_D2H ? -1 : (int)me.aux2,
             (unsigned __int128)me.count);
    if (kind == CT_KIND_MEMCPY) cf0 = min(cf0, (unsigned long long)abs);
    else if (kind == CT_KIND_UM) cf1 = min(cf1, (unsigned long long)abs);
    else cf2 = min(cf2, (unsigned long long)abs);
  }
}

}  // namespace

size_t fast_smem_bytes(int g2, int smem_hist) {
  size_t b = sizeof(WarpMem) * kWarps + sizeof(CtaMem);
  if (smem_hist) b += (size_t)kTypes * g2 * g2 * (sizeof(unsigned long long) + sizeof(unsigned int));
  return b;
}

template <bool SH>
__global__ void __launch_bounds__(kThreads, 1) fast_kernel(FastParams P) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  WarpMem* WM = reinterpret_cast<WarpMem*>(smem_raw);
  CtaMem& C = *reinterpret_cast<CtaMem*>(smem_raw + sizeof(WarpMem) * kWarps);
  const int ncell = kTypes * P.g2 * P.g2;
  unsigned long long* shb = reinterpret_cast<unsigned long long*>(smem_raw + sizeof(WarpMem) * kWarps + sizeof(CtaMem));
  unsigned int* shf = reinterpret_cast<unsigned int*>(shb + ncell);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  WarpMem& W = WM[warp];
  const unsigned lt = (1u << lane) - 1;
  const unsigned gt = lane == 31 ? 0u : ~((2u << lane) - 1);

  // ---- init
  if (SH)
    for (int c = tid; c < ncell; c += kThreads) { shb[c] = 0; shf[c] = 0; }
  if (tid < kTypes) { C.calls[tid] = 0; C.pay_lo[tid] = 0; C.pay_hi[tid] = 0; }
  if (tid < 3) C.copy_first[tid] = kNone;
  if (tid < CT_NDIAG) C.diag[tid] = 0;
  if (tid == 0) { C.flags = 0; C.max_dev = -1; }
  if (lane < kCS) {
    W.tag[lane] = kEmptyTag; W.sn[lane] = 0; W.sver[lane] = 0;
    W.cfirst[lane] = kNone; W.clast[lane] = kNone;
    for (int t = 0; t < 5; t++) W.tfirst[lane][t] = kNone;
  }
  P2PEntry* chan = P.chans + (size_t)(blockIdx.x * kWarps + warp) * kPC;  // this warp's channel table
  for (int e = lane; e < kPC; e += 32) chan[e].key = kNone;
  if (lane < kRing) mbar_init(&W.bar[lane], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();

  Acc<SH> acc;
  acc.init(&C, SH ? shb : P.cells, SH ? (void*)shf : (void*)P.freq, SH, P.g2, P.gcap, P.explicit_d != 0);
  int my_max_dev = -1;
  uint32_t n_incompat = 0, n_dupdev = 0, n_mismatch = 0;
  unsigned long long cf0 = kNone, cf1 = kNone, cf2 = kNone;  // first record of each copy kind
  uint32_t wflags = 0;
  unsigned long long tf_pend = ~0ull;  // (slot, type) pairs whose first valid instance is not yet recorded
  uint32_t sc_comm = kEmptyTag;  // last (comm, slot) pair looked up (warp-uniform)
  int sc_slot = -1;

  // ---- this warp's range, cut at element starts
  const uint32_t gw = blockIdx.x * kWarps + warp;
  const uint64_t NC = P.n_chunks;
  const uint64_t c0 = NC * gw / P.total_warps, c1 = NC * (gw + 1) / P.total_warps;
  bool bad = false;
  const uint64_t start = c0 == 0 ? 0 : first_start(P.recs, P.n, c0 * 32, bad);
  const uint64_t end = c1 >= NC ? P.n : first_start(P.recs, P.n, c1 * 32, bad);
  if (bad) wflags |= F_NONCANON;
  if (start < end && !bad) {
    // The warp slides a 32-record window over its range.  A window always begins at an
    // element start and consumes exactly the elements that lie whole inside it (n <= 32
    // guarantees progress); the next window begins where the last one ended.  Chunk k of
    // the range lives in ring slot (k - k0) % kRing; a window touches at most two chunks.
    const uint64_t k0 = start / 32;
    const uint64_t rb0 = k0 * 32;                                  // record at ring index 0
    const uint64_t last_chunk = min(NC, (end + 31) / 32 + 1);      // chunks below this may be read
    const ct_record* R = &W.ring[0][0];
    const WinDev wdv{R, rb0};
    uint64_t issued = k0, ready = k0, freed = k0;
    {
      const uint64_t lim = min(k0 + kRing, last_chunk);
      for (; issued < lim; issued++)
        if (lane == 0)
          bulk_load(W.ring[(issued - k0) % kRing], P.recs + issued * 32,
                    (uint32_t)min((uint64_t)32, P.n - issued * 32) * (uint32_t)sizeof(ct_record),
                    &W.bar[(issued - k0) % kRing]);
    }

    uint64_t b = start;
    while (b < end) {
      const uint64_t kB = min((b + 31) / 32, last_chunk - 1);
      while (ready <= kB) {
        mbar_wait(&W.bar[(ready - k0) % kRing], (uint32_t)(((ready - k0) / kRing) & 1));
        ready++;
      }
      const uint32_t ri0 = (uint32_t)(b - rb0);                    // ring index of the window start
      const uint32_t nval = (uint32_t)min((uint64_t)32, P.n - b);  // records that exist
      const uint32_t lim = (uint32_t)min((uint64_t)32, end - b);   // heads this range owns
      const bool valid = (uint32_t)lane < nval;
      Rec ra{};
      int kind = 7;
      if (valid) { ra = load_swz(R, (ri0 + lane) & kRM); kind = ra.kind(); }
      uint64_t nb;
      if (P.dbg & 4) {  // diagnostic: stream only (roofline experiments)
        my_max_dev = max(my_max_dev, (int)(ra.dev ^ ra.rank));
        nb = b + 32;
      } else {
        // ---------------- elements: starts, lengths, whole-in-window heads, coverage
        const bool isS = valid && is_start(kind, ra.rank);
        uint32_t len = 0;
        bool badl = false;
        if (isS) {
          len = kind == CT_KIND_COLLECTIVE ? ra.nranks : (kind == CT_KIND_SEND ? 2u : 1u);
          if (len == 0 || len > (uint32_t)kMaxN) { badl = true; len = 1; }
        }
        const unsigned Sall = __ballot_sync(kFull, isS);
        const unsigned Sown = lim >= 32 ? Sall : Sall & ((1u << lim) - 1);
        const unsigned Inc = __ballot_sync(kFull, ((Sown >> lane) & 1) && (uint32_t)lane + len > 32);
        const unsigned H = Inc ? Sown & ((1u << (__ffs(Inc) - 1)) - 1) : Sown;  // heads processed now
        const bool head = (H >> lane) & 1;
        if (!(H & 1)) badl = true;  // the window must begin with an element start
        const int hL = H ? 31 - __clz(H) : 0;
        const uint32_t Pw = hL + __shfl_sync(kFull, len, hL);      // records consumed
        const bool mem = (uint32_t)lane < Pw;
        const unsigned below = H & (lt | (1u << lane));
        const int hA = below ? 31 - __clz(below) : 0;
        const uint32_t lenA = __shfl_sync(kFull, len, hA);
        if (mem && (uint32_t)lane >= (uint32_t)hA + lenA) badl = true;  // a record no element covers
        if (head && ((uint32_t)lane + len > nval || !range_clear((unsigned long long)Sall, (uint32_t)lane + 1, len - 1)))
          badl = true;  // runs past the trace, or another element starts inside this one

        // ---------------- member checks against the predecessor record (lane shuffles)
        // words: comm | nranks, rank | kc, ad, aux | count lo | count hi
        const uint32_t a2 = ra.kc | (ra.ad << 8) | (ra.aux << 16);
        bool gfail = false, mis = false;
        {
          const uint32_t q0 = __shfl_up_sync(kFull, ra.comm, 1);
          const uint32_t q1 = __shfl_up_sync(kFull, ra.nranks | (ra.rank << 16), 1);
          const uint32_t q2 = __shfl_up_sync(kFull, a2, 1);
          const uint32_t q3 = __shfl_up_sync(kFull, (uint32_t)ra.count, 1);
          const uint32_t q4 = __shfl_up_sync(kFull, (uint32_t)(ra.count >> 32), 1);
          if (mem && !head) member_check(ra, a2, q0, q1, q2, q3, q4, badl, gfail, mis);
        }
        if (__any_sync(kFull, badl)) { wflags |= F_NONCANON; break; }  // host re-runs the exact path
        const bool collH = head && kind == CT_KIND_COLLECTIVE;
        const bool sendH = head && kind == CT_KIND_SEND;
        const unsigned Hc = __ballot_sync(kFull, collH);
        const unsigned Hs = __ballot_sync(kFull, sendH);
        const unsigned sigmask = __ballot_sync(kFull, gfail);
        const unsigned mismask = Hs ? __ballot_sync(kFull, mis) : 0u;

        // ---------------- per-comm predecessor block, comm slot (uniform fast case)
        uint32_t info = 0;  // slot | ph << 4 | has_ph << 10 | hist << 11 | ver << 12 | last << 13
        if (Hc) {
          const uint32_t c_first = __shfl_sync(kFull, ra.comm, __ffs(Hc) - 1);
          if (__all_sync(kFull, !collH || ra.comm == c_first)) {
            int su = c_first == sc_comm ? sc_slot : find_slot(W, c_first);
            if (su < 0) {  // new comm in this range
              for (int s = kCS - 1; s >= 0; s--)
                if (W.tag[s] == kEmptyTag) su = s;
              __syncwarp();
              if (su < 0) wflags |= F_NONCANON;  // more comms than slots in one range
              else if (lane == 0) W.tag[su] = c_first;
              __syncwarp();
            }
            if (c_first >= P.n_comms) wflags |= F_COMM_RANGE | F_NONCANON;
            sc_comm = c_first;
            sc_slot = su;
            const int slot = su < 0 ? 0 : su;
            const uint32_t sn = W.sn[slot];
            const uint32_t base = (uint32_t)slot | (sn ? 1u << 11 : 0u) | (sn && W.sver[slot] ? 1u << 12 : 0u);
            const unsigned lower = Hc & ((1u << hA) - 1);
            const int ph = lower ? 31 - __clz(lower) : -1;
            info = base | ((uint32_t)(ph & 63) << 4) | (ph >= 0 ? 1u << 10 : 0u) | ((Hc >> hA) == 1u ? 1u << 13 : 0u);
          } else {
            // several comms start blocks in this window: per-head slots, MATCH for predecessors
            int slot = -1;
            if (collH) {
              if (ra.comm >= P.n_comms) wflags |= F_COMM_RANGE | F_NONCANON;
              slot = ra.comm == sc_comm ? sc_slot : find_slot(W, ra.comm);
            }
            while (true) {  // allocate slots for unseen comms (rare, warp-serial)
              const unsigned miss = __ballot_sync(kFull, collH && slot < 0);
              if (!miss) break;
              const uint32_t cm = __shfl_sync(kFull, ra.comm, __ffs(miss) - 1);
              int free_s = -1;
              for (int s = kCS - 1; s >= 0; s--)
                if (W.tag[s] == kEmptyTag) free_s = s;
              __syncwarp();
              if (free_s < 0) { wflags |= F_NONCANON; break; }
              if (lane == 0) W.tag[free_s] = cm;
              __syncwarp();
              if (collH && slot < 0 && ra.comm == cm) slot = free_s;
            }
            const unsigned same =
                __match_any_sync(kFull, collH ? (unsigned long long)ra.comm : (0xFFFFFFFF00000000ull | lane)) & Hc;
            const unsigned lower = same & lt;
            const int ph = lower ? 31 - __clz(lower) : -1;
            const int hs = slot < 0 ? 0 : slot;
            const bool hist = collH && W.sn[hs] != 0;
            const uint32_t hinfo = (uint32_t)hs | ((uint32_t)(ph & 63) << 4) | (ph >= 0 ? 1u << 10 : 0u) |
                                   (hist ? 1u << 11 : 0u) | (hist && W.sver[hs] ? 1u << 12 : 0u) |
                                   ((same & gt) == 0 ? 1u << 13 : 0u);
            info = __shfl_sync(kFull, hinfo, hA);
          }
        }
        if (collH) {  // nranks constant per comm (grouping.py:104-108)
          const uint32_t pn = (info & (1u << 10)) ? R[(ri0 + ((info >> 4) & 63)) & kRM].nranks
                                                  : ((info & (1u << 11)) ? W.sn[info & 15] : ra.nranks);
          if (pn != ra.nranks) wflags |= F_NONCANON;
        }

        // ---------------- per-member seq order and device inheritance from the last block
        bool devf = false;
        const bool cm = mem && kind == CT_KIND_COLLECTIVE;
        {
          const int src = (cm && (info & (1u << 10))) ? ((((info >> 4) & 63) + (int)ra.rank) & 31) : lane;
          const uint64_t pseq = ((uint64_t)__shfl_sync(kFull, (uint32_t)(ra.seq >> 32), src) << 32) |
                                __shfl_sync(kFull, (uint32_t)ra.seq, src);
          if (cm) order_check(W, ra, info, pseq, wflags, devf);
        }
        const unsigned devmask = __ballot_sync(kFull, devf);

        // ---------------- element status (every member derives its element's status)
        // collective: incompatible if any member's signature differs (grouping.py:144-155),
        // duplicate device if devices are not pairwise distinct (grouping.py:156-167)
        const unsigned needs_full = __ballot_sync(kFull, collH && !range_clear(devmask, (uint32_t)lane, ra.nranks));
        bool dist = true;
        if (needs_full) {  // devices changed since the comm's last block: full pairwise check
          if ((needs_full >> lane) & 1) dist = devices_distinct(R, ri0 + lane, ra.nranks);
        }
        const unsigned dupmask = __ballot_sync(kFull, !dist);  // heads with duplicate devices
        const uint32_t kindH = __shfl_sync(kFull, (uint32_t)kind, hA);
        uint32_t st = ST_NONE;
        if (mem) {
          if (kindH == CT_KIND_COLLECTIVE)
            st = !range_clear(sigmask, (uint32_t)hA + 1, lenA - 1) ? ST_INCOMPAT
                                                                   : (((dupmask >> hA) & 1) ? ST_DUPDEV : ST_VALID);
          else if (kindH == CT_KIND_SEND)
            st = ((mismask >> (hA + 1)) & 1) ? ST_MISMATCH : ST_VALID;
          else
            st = ST_VALID;
        }
        if (head) {
          n_incompat += st == ST_INCOMPAT;
          n_dupdev += st == ST_DUPDEV;
          n_mismatch += st == ST_MISMATCH;
        }

        // ---------------- p2p order: per (comm, src, dst) channel non-decreasing send and
        // recv seqs (decompose.py:359-361 sorts each side by seq; FIFO pairs by position)
        if (Hs) {
          const uint64_t nseq = ((uint64_t)__shfl_down_sync(kFull, (uint32_t)(ra.seq >> 32), 1) << 32) |
                                __shfl_down_sync(kFull, (uint32_t)ra.seq, 1);
          p2p_order(chan, ra, nseq, sendH, lane, lt, gt, wflags);
        }

        // ---------------- table update with the last block of each comm in the window
        __syncwarp();
        if (cm && (info & (1u << 13))) { W.cseq[info & 15][ra.rank] = ra.seq; W.cdev[info & 15][ra.rank] = (uint16_t)ra.dev; }
        if (collH) {
          const int hs = info & 15;
          const uint64_t gi = b + lane;
          if (!(info & (3u << 10))) W.cfirst[hs] = gi;  // first block of this comm in the range
          if (info & (1u << 13)) { W.sn[hs] = ra.nranks; W.sver[hs] = dist; W.clast[hs] = gi; }
        }
        if (Hc) {  // first valid instance per (comm slot, type): only until recorded once
          const unsigned long long bit = (collH && st == ST_VALID) ? 1ull << ((info & 15) * 5 + ra.coll()) : 0ull;
          const bool rec = (bit & tf_pend) != 0;
          if (rec) note_min_smem(&W.tfirst[info & 15][ra.coll()], b + lane);
          const unsigned lo = __reduce_or_sync(kFull, rec ? (unsigned)bit : 0u);
          const unsigned hi = __reduce_or_sync(kFull, rec ? (unsigned)(bit >> 32) : 0u);
          tf_pend &= ~(((unsigned long long)hi << 32) | lo);
        }
        __syncwarp();

        // ---------------- expansion + accumulation
        if (mem && !(P.dbg & 1)) expand_record(P, acc, wdv, ra, b + lane, st, b + (uint64_t)hA, my_max_dev, cf0, cf1, cf2);
        nb = b + Pw;
      }

      // ---------------- slide: chunks wholly behind the next window refill their slots
      const uint64_t kf = nb / 32;
      if (kf > freed) {
        __syncwarp();
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        do {
          const uint64_t q = freed + kRing;
          if (q < last_chunk) {
            if (lane == 0)
              bulk_load(W.ring[(freed - k0) % kRing], P.recs + q * 32,
                        (uint32_t)min((uint64_t)32, P.n - q * 32) * (uint32_t)sizeof(ct_record),
                        &W.bar[(freed - k0) % kRing]);
            issued = q + 1;
          }
          freed++;
        } while (freed < kf);
      }
      b = nb;
    }
    for (uint64_t q = ready; q < issued; q++)  // drain outstanding bulk copies
      mbar_wait(&W.bar[(q - k0) % kRing], (uint32_t)(((q - k0) / kRing) & 1));
  }

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
  acc.drain();
  atomicMax(&C.max_dev, my_max_dev);
  if (n_incompat) atomicAdd(&C.diag[CT_DIAG_INCOMPATIBLE], n_incompat);
  if (n_dupdev) atomicAdd(&C.diag[CT_DIAG_DUPLICATE_DEVICE], n_dupdev);
  if (n_mismatch) atomicAdd(&C.diag[CT_DIAG_MISMATCHED_P2P], n_mismatch);
  if (cf0 != kNone) atomicMin(&C.copy_first[0], cf0);
  if (cf1 != kNone) atomicMin(&C.copy_first[1], cf1);
  if (cf2 != kNone) atomicMin(&C.copy_first[2], cf2);
  if (acc.flags | wflags) atomicOr(&C.flags, acc.flags | wflags);
  if (acc.oor_key != kNone) atomicMin(&P.st->oor_key, acc.oor_key);
  if (acc.of_cell != kNone) atomicMin(&P.st->of_cell, acc.of_cell);
  __syncthreads();

  GlobalState* G = P.st;
  if (SH) {
    uint32_t of = 0;
    for (int c = tid; c < ncell; c += kThreads) {
      const unsigned int f = shf[c];
      if (!f) continue;
      const unsigned long long bb = shb[c];
      const unsigned long long old = atomicAdd(P.cells + c, bb);
      if (old + bb < old) { of |= F_OVERFLOW; atomicMin(&G->of_cell, (unsigned long long)c); }
      atomicAdd(P.freq + c, (unsigned long long)f);
    }
    if (of) atomicOr(&C.flags, of);
  }
  if (tid < kTypes) {
    const unsigned long long lo = C.pay_lo[tid], hi = C.pay_hi[tid], c = C.calls[tid];
    if (c) {
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
  }
}

template __global__ void fast_kernel<true>(FastParams);
template __global__ void fast_kernel<false>(FastParams);

// Cross-range seq-order check, one thread per (warp range, item): items [0, kCS) are the
// collective comm slots (nranks equal and per-rank seq strictly increasing from the last
// block of the nearest earlier range holding the comm to this range's first block), items
// [kCS, kCS + kPC) the p2p channels (send and recv seqs non-decreasing across ranges).
__global__ void range_check_kernel(const ct_record* recs, const WarpSlot* slots, const P2PEntry* chans,
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
  const P2PEntry& me = chans[(size_t)w * kPC + (item - kCS)];
  if (me.key == kNone) return;
  for (int32_t v = (int32_t)w - 1; v >= 0; v--)
    for (int q = 0; q < kPC; q++) {
      const P2PEntry& o = chans[(size_t)v * kPC + q];
      if (o.key != me.key) continue;
      if (me.first_s < o.last_s || me.first_r < o.last_r) atomicOr(&st->flags, F_NONCANON);
      return;
    }
}

}  // namespace ct
