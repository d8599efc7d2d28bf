// Fast path: warp-autonomous streaming layout check + join + expand + accumulate
// (design notes in ct_fast.cuh).
#include "ct_fast.cuh"

namespace ct {

namespace {

constexpr uint64_t kNone = ~0ull;
constexpr uint32_t kEmptyTag = 0xFFFFFFFFu;
constexpr unsigned kFull = 0xFFFFFFFFu;

// A block signature seen valid in the warp's steady communicator, and how many later
// blocks repeated it exactly (same signature and devices) without being expanded yet.
struct __align__(16) Tpl {
  unsigned long long count;
  uint32_t sig;   // coll_sig(); 0 = empty entry
  uint32_t ndef;  // deferred repeats
};
constexpr int kTSets = 16;          // 2-way set-associative template table
constexpr int kTE = 2 * kTSets;
static_assert(kTE == 32, "one template entry per lane");

struct __align__(16) WarpMem {
  ct_record ring[kRing][32];                 // TMA ring: chunk k lives in slot (k - k0) % kRing
  Tpl tpl[kTE];
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
  unsigned long long oor_key;   // min out-of-range ordering key seen by the CTA
  unsigned long long of_cell;   // min cell index whose 64-bit sum wrapped
  unsigned int diag[CT_NDIAG];
  uint32_t flags;
  int max_dev;
};
static_assert(sizeof(CtaMem) % 16 == 0, "histogram after CtaMem must stay aligned");
// the shared-memory histogram must fit for d <= 16 (g2 = 18), else the kernel falls back
// to global atomics
static_assert(sizeof(WarpMem) * kWarps + sizeof(CtaMem) + kTypes * 18 * 18 * 12 <= 227 * 1024,
              "shared memory budget: CTA histogram no longer fits for d <= 16");

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
// Histogram location: the CTA's shared-memory copy right after CtaMem (SH), else global.
template <bool SH>
__device__ __forceinline__ unsigned long long* hist_bytes(const FastParams& P) {
  return SH ? reinterpret_cast<unsigned long long*>(&cta_mem() + 1) : P.cells;
}
template <bool SH>
__device__ __forceinline__ void* hist_freq(const FastParams& P) {
  return SH ? static_cast<void*>(hist_bytes<SH>(P) + kTypes * P.g2 * P.g2) : static_cast<void*>(P.freq);
}

__device__ __forceinline__ void note_overflow(uint32_t& flags, unsigned long long key) {
  flags |= F_OVERFLOW;
  if (key < cta_mem().of_cell) atomicMin(&cta_mem().of_cell, key);
}

template <bool SH>  // SH: CTA histogram in shared memory (else global atomics)
struct Acc {
  // two small register caches: transfer cells and per-type statistics; a miss evicts the
  // older entry into the CTA histogram (shared-memory atomics).  Everything else (the
  // histogram, limits, first-error keys) comes from the kernel parameters / shared memory.
  uint32_t ctag[2], stag[2];
  unsigned long long csum[2], ssum[2];
  uint32_t ccnt[2], scnt[2];
  uint32_t flags;
  unsigned long long rec_key;  // (class << 62) | (element << 21) | (src rank << 11) for oor ordering
  const FastParams& P;

  __device__ __forceinline__ explicit Acc(const FastParams& p) : P(p) {
    ctag[0] = ctag[1] = stag[0] = stag[1] = kEmptyTag;
    csum[0] = csum[1] = ssum[0] = ssum[1] = 0;
    ccnt[0] = ccnt[1] = scnt[0] = scnt[1] = 0;
    flags = 0;
    rec_key = 0;
  }

  __device__ __forceinline__ void flush_cell(uint32_t key, unsigned long long v, uint32_t c) {
    const unsigned long long old = atomicAdd(hist_bytes<SH>(P) + key, v);
    if (old + v < old) note_overflow(flags, key);
    if (SH) atomicAdd(static_cast<unsigned int*>(hist_freq<SH>(P)) + key, c);
    else atomicAdd(static_cast<unsigned long long*>(hist_freq<SH>(P)) + key, (unsigned long long)c);
  }

  __device__ __forceinline__ void flush_stat(uint32_t t, unsigned long long v, uint32_t c) {
    CtaMem& C = cta_mem();
    const unsigned long long old = atomicAdd(&C.pay_lo[t], v);
    if (old + v < old) atomicAdd(&C.pay_hi[t], 1ull);
    atomicAdd(&C.calls[t], (unsigned long long)c);
  }

  __device__ __forceinline__ void add_cell(uint32_t key, unsigned long long v) {
    if (ctag[0] == key) {
      const unsigned long long s = csum[0] + v;
      if (s < v) note_overflow(flags, key);
      csum[0] = s; ccnt[0]++;
    } else if (ctag[1] == key) {
      const unsigned long long s = csum[1] + v;
      if (s < v) note_overflow(flags, key);
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
    CtaMem& C = cta_mem();
    const unsigned long long lo = (unsigned long long)s;
    unsigned long long hi = (unsigned long long)(s >> 64);
    const unsigned long long old = atomicAdd(&C.pay_lo[type], lo);
    if (old + lo < old) hi += 1;
    atomicAdd(&C.pay_hi[type], hi);
    atomicAdd(&C.calls[type], 1ull);
  }

  __device__ __forceinline__ void out_of_range(unsigned long long k) {
    flags |= P.explicit_d ? F_OOR : F_CAP;
    if (k < cta_mem().oor_key) atomicMin(&cta_mem().oor_key, k);
  }

  // endpoint: gpu g (>= 0), -1 host, -2 net.  ``sub`` orders transfers inside one
  // decomposition (destination rank of a collective edge, transfers are sorted by rank
  // pair, decompose.py:92; 0/1 for collnet) for the EndpointOutOfRange message.
  __device__ __forceinline__ void edge(int type, int src, int dst, unsigned __int128 bytes, int sub = 0) {
    const int a = src == -1 ? kHost : (src == -2 ? kNet : src + 2);
    const int b = dst == -1 ? kHost : (dst == -2 ? kNet : dst + 2);
    if (src >= P.gcap || dst >= P.gcap) {
      const unsigned long long k = rec_key | ((unsigned long long)min(sub, 1023) << 1);
      if (src >= P.gcap) out_of_range(k);
      if (dst >= P.gcap) out_of_range(k | 1);
      return;
    }
    if ((bytes >> 63) != 0) { flags |= F_OVERFLOW; return; }
    add_cell((uint32_t)((type * P.g2 + a) * P.g2 + b), (unsigned long long)bytes);
  }
};

// device of a record held in the warp's ring, by position relative to the ring origin
struct WinDev {
  const ct_record* R;
  __device__ __forceinline__ uint32_t dev_of(uint64_t rel) const { return R[(uint32_t)rel & kRM].dev; }
};

// signature word of a collective record: coll, has_root, algo, dtype, root when rooted
// (grouping.py:78-79 without count), bit 7 set so an empty entry (0) never matches
__device__ __forceinline__ uint32_t coll_sig(uint32_t a2 /* kc | ad << 8 | aux << 16 */) {
  return (a2 & (0x3F78u | ((a2 & 0x40u) ? 0xFFFF0000u : 0u))) | 0x80u;
}

__device__ __forceinline__ uint32_t tpl_set(unsigned long long count, uint32_t sig) {
  const uint32_t h = ((uint32_t)count ^ ((uint32_t)(count >> 32) * 0x85EBCA6Bu) ^ (sig * 0xC2B2AE35u)) * 0x9E3779B1u;
  return h >> 28;  // kTSets == 16
}

// ------------------------------------------------------------ out-of-line sinks
// Sink that adds every transfer ``c`` times straight into the CTA histogram: bytes * c
// into the cell, c into the frequency, S * c into the 128-bit payload and c calls.  Used
// for deferred repeats (c identical blocks) and for the rare > 2^40-element records.
template <bool SH>
struct DirectSink {
  unsigned long long* hb;
  void* hf;
  int g2, gcap, explicit_d;
  unsigned long long rec_key;
  unsigned long long c;
  uint32_t flags;
  __device__ __forceinline__ void stat(int type, unsigned __int128 s) {
    CtaMem& C = cta_mem();
    const unsigned __int128 v = s * c;
    const unsigned long long lo = (unsigned long long)v;
    unsigned long long hi = (unsigned long long)(v >> 64);
    const unsigned long long old = atomicAdd(&C.pay_lo[type], lo);
    if (old + lo < old) hi++;
    if (hi) atomicAdd(&C.pay_hi[type], hi);
    atomicAdd(&C.calls[type], c);
  }
  __device__ __forceinline__ void edge(int type, int src, int dst, unsigned __int128 bytes, int sub) {
    if (src >= gcap || dst >= gcap) {  // same ordering key as Acc::edge
      const unsigned long long k = rec_key | ((unsigned long long)min(sub, 1023) << 1);
      flags |= explicit_d ? F_OOR : F_CAP;
      const unsigned long long kk = src >= gcap ? k : (k | 1);
      if (kk < cta_mem().oor_key) atomicMin(&cta_mem().oor_key, kk);
      return;
    }
    const int a = src == -1 ? kHost : (src == -2 ? kNet : src + 2);
    const int b = dst == -1 ? kHost : (dst == -2 ? kNet : dst + 2);
    const unsigned long long key = (unsigned long long)((type * g2 + a) * g2 + b);
    const unsigned __int128 v = bytes * c;
    if ((v >> 63) != 0) {  // one transfer alone exceeds the cell (as Acc::edge); c repeats do by summing
      if (c == 1) flags |= F_OVERFLOW;
      else note_overflow(flags, key);
      return;
    }
    const unsigned long long old = atomicAdd(hb + key, (unsigned long long)v);
    if (old + (unsigned long long)v < old) note_overflow(flags, key);
    if (SH) atomicAdd(static_cast<unsigned int*>(hf) + key, (unsigned int)c);
    else atomicAdd(static_cast<unsigned long long*>(hf) + key, c);
  }
};

// a collective record with count >= 2^40 (128-bit byte counts): rare, kept out of line
template <bool SH>
__device__ __noinline__ uint32_t expand_wide(ExpandParams ex, unsigned long long* hb, void* hf, int g2, int gcap,
                                             int explicit_d, unsigned long long rec_key, Rec me, uint32_t head,
                                             const ct_record* R) {
  DirectSink<SH> ds{hb, hf, g2, gcap, explicit_d, rec_key, 1ull, 0u};
  const WinDev wdv{R};
  expand_collective<unsigned __int128>(ex, wdv, ds, me, head);
  return ds.flags;
}

struct TblDev {  // devices of the steady communicator's last block, by rank
  const uint16_t* cd;
  __device__ __forceinline__ uint32_t dev_of(uint64_t r) const { return cd[(uint32_t)r]; }
};

// Expand every template with deferred repeats (lane = rank) and clear the counters;
// returns error flags.
template <bool SH>
__device__ __noinline__ uint32_t flush_templates(ExpandParams ex, unsigned long long* hb, void* hf, int g2, WarpMem& W,
                                                 int ts, uint32_t tcomm, uint32_t tn) {
  const int lane = threadIdx.x & 31;
  uint32_t flags = 0;
  unsigned todo = __ballot_sync(kFull, W.tpl[lane].ndef != 0);  // kTE == 32
  while (todo) {
    const int e = __ffs(todo) - 1;
    todo &= todo - 1;
    const unsigned long long c = W.tpl[e].ndef;
    if ((uint32_t)lane < tn) {
      const uint32_t sg = W.tpl[e].sig;
      Rec rc;
      rc.count = W.tpl[e].count;
      rc.seq = 0;
      rc.comm = tcomm;
      rc.nranks = tn;
      rc.rank = (uint32_t)lane;
      rc.dev = W.cdev[ts][lane];
      rc.aux = sg >> 16;
      rc.aux2 = 0;
      rc.kc = sg & 0x78u;
      rc.ad = (sg >> 8) & 0x3Fu;
      DirectSink<SH> ds{hb, hf, g2, 1 << 30, 0, 0ull, c, 0u};  // steady devices are < gcap
      const TblDev td{W.cdev[ts]};
      if ((rc.count >> 40) == 0) expand_collective<uint64_t>(ex, td, ds, rc, 0);
      else expand_collective<unsigned __int128>(ex, td, ds, rc, 0);
      flags |= ds.flags;
    }
  }
  __syncwarp();
  W.tpl[lane].ndef = 0;
  __syncwarp();
  return flags;
}

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
                                          uint32_t& wflags) {
  const unsigned lt = (1u << lane) - 1;
  const unsigned gt = lane == 31 ? 0u : ~((2u << lane) - 1);
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

// expansion + accumulation of one record of a processed element (status ``st``); ``rel``
// and ``head`` are positions relative to the ring origin ``rb0``
template <bool SH>
__device__ __forceinline__ void expand_record(const FastParams& P, Acc<SH>& acc, const WinDev& wdv, const Rec& me,
                                              uint64_t rb0, uint32_t rel, uint32_t st, uint32_t head, int& max_dev,
                                              uint32_t& copy_seen) {
  const int kind = me.kind();
  max_dev = max(max_dev, (int)me.dev);
  if (kind == CT_KIND_COLLECTIVE) {
    if (st != ST_VALID) return;
    acc.rec_key = (min((unsigned long long)(rb0 + head), (1ull << 41) - 1) << 21) | ((unsigned long long)min(me.rank, 1023u) << 11);
    if ((me.count >> 40) == 0) expand_collective<uint64_t>(P.ex, wdv, acc, me, head);
    else acc.flags |= expand_wide<SH>(P.ex, hist_bytes<SH>(P), hist_freq<SH>(P), P.g2, P.gcap, P.explicit_d,
                                      acc.rec_key, me, head, wdv.R);
  } else if (kind == CT_KIND_SEND) {
    if (st != ST_VALID) return;
    const unsigned __int128 nb = (unsigned __int128)me.count * (unsigned)dtype_width(me.dtype());
    acc.stat(CT_T_SENDRECV, nb);
    acc.rec_key = (1ull << 62) | (min((unsigned long long)(rb0 + rel), (1ull << 41) - 1) << 21);
    const int rdev = (int)wdv.dev_of(rel + 1);
    if (rdev != (int)me.dev) acc.edge(CT_T_SENDRECV, (int)me.dev, rdev, nb);
  } else if (kind >= CT_KIND_MEMCPY) {
    const int ck = me.ckind();
    if (ck != CT_CKIND_H2D) max_dev = max(max_dev, (int)me.aux);
    if (ck != CT_CKIND_D2H) max_dev = max(max_dev, (int)me.aux2);
    const int t = CT_T_EXPLICIT + (kind - CT_KIND_MEMCPY);
    acc.stat(t, (unsigned __int128)me.count);
    acc.rec_key = (2ull << 62) | (min((unsigned long long)(rb0 + rel), (1ull << 41) - 1) << 21);
    acc.edge(t, ck == CT_CKIND_H2D ? -1 : (int)me.aux, ck == CT_CKIND_D2H ? -1 : (int)me.aux2,
             (unsigned __int128)me.count);
    // first record of each copy kind: positions only grow, so a lane's first is its min
    const uint32_t bit = 1u << (kind - CT_KIND_MEMCPY);
    if (!(copy_seen & bit)) {
      copy_seen |= bit;
      atomicMin(&cta_mem().copy_first[kind - CT_KIND_MEMCPY], rb0 + rel);
    }
  }
}

__device__ __forceinline__ void count_diag(uint32_t st) {
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
__global__ void __launch_bounds__(kThreads, 1) fast_kernel(FastParams P) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  WarpMem* WM = reinterpret_cast<WarpMem*>(smem_raw);
  CtaMem& C = cta_mem();
  const int ncell = kTypes * P.g2 * P.g2;
  unsigned long long* shb = hist_bytes<true>(P);
  unsigned int* shf = static_cast<unsigned int*>(hist_freq<true>(P));
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  WarpMem& W = WM[warp];

  // ---- init
  if (SH)
    for (int c = tid; c < ncell; c += kThreads) { shb[c] = 0; shf[c] = 0; }
  if (tid < kTypes) { C.calls[tid] = 0; C.pay_lo[tid] = 0; C.pay_hi[tid] = 0; }
  if (tid < 3) C.copy_first[tid] = kNone;
  if (tid < CT_NDIAG) C.diag[tid] = 0;
  if (tid == 0) { C.flags = 0; C.max_dev = -1; C.oor_key = kNone; C.of_cell = kNone; }
  W.tpl[lane].sig = 0;  // kTE == 32
  W.tpl[lane].ndef = 0;
  if (lane < kCS) {
    W.tag[lane] = kEmptyTag; W.sn[lane] = 0; W.sver[lane] = 0;
    W.cfirst[lane] = kNone; W.clast[lane] = kNone;
    for (int t = 0; t < 5; t++) W.tfirst[lane][t] = kNone;
  }
  const uint32_t gw = blockIdx.x * kWarps + warp;
  for (int e = lane; e < kPC; e += 32) P.chans[(size_t)gw * kPC + e].key = kNone;
  if (lane < kRing) mbar_init(&W.bar[lane], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();

  const long long t_start = clock64();
  Acc<SH> acc(P);
  int my_max_dev = -1;
  uint32_t copy_seen = 0;              // copy kinds this lane has seen (first index noted)
  uint32_t wflags = 0;
  unsigned long long tf_pend = ~0ull;  // (slot, type) pairs whose first valid instance is not yet recorded
  uint32_t sc_comm = kEmptyTag;        // last (comm, slot) pair looked up (warp-uniform)
  int sc_slot = -1;

  // ---- this warp's range, cut at element starts
  const uint64_t NC = P.n_chunks;
  const uint64_t c0 = NC * gw / P.total_warps, c1 = NC * (gw + 1) / P.total_warps;
  bool bad = false;
  const uint64_t start = c0 == 0 ? 0 : first_start(P.recs, P.n, c0 * 32, bad);
  const uint64_t end = c1 >= NC ? P.n : first_start(P.recs, P.n, c1 * 32, bad);
  if (bad) wflags |= F_NONCANON;
  if (start < end && !bad) {
    // The warp slides a 32-record window over its range.  A window always begins at an
    // element start and consumes exactly the elements that lie whole inside it (n <= 32
    // guarantees progress); the next window begins where the last one ended.  Positions
    // are 32-bit, relative to the ring origin rb0 (chunk k0); relative chunk q lives in
    // ring slot q % kRing, so record rb0 + x sits at ring index x & kRM.
    const uint64_t k0 = start / 32;
    const uint64_t rb0 = k0 * 32;
    const uint32_t lastc = (uint32_t)(min(NC, (end + 31) / 32 + 1) - k0);  // chunks below this may be read
    const uint32_t eo = (uint32_t)(end - rb0);
    const uint32_t no = (uint32_t)min((unsigned long long)(P.n - rb0), 0xFFFFFFFFull);
    const ct_record* R = &W.ring[0][0];
    const WinDev wdv{R};
    uint32_t issued = 0, ready = 0, freed = 0;
    for (; issued < (uint32_t)kRing && issued < lastc; issued++)
      if (lane == 0) {
        const uint64_t first = (k0 + issued) * 32;
        bulk_load(W.ring[issued], P.recs + first, (uint32_t)min((uint64_t)32, P.n - first) * (uint32_t)sizeof(ct_record),
                  &W.bar[issued]);
      }

    int ts = -1;                     // steady comm slot (-1: none)
    uint32_t tcomm = 0, tn = 0;      // its comm id and nranks
    uint32_t pending = 0;            // deferred blocks not yet expanded
    uint32_t skip = 0, backoff = 0;  // steady attempts back off after misses
    uint32_t bo = (uint32_t)(start - rb0);
    while (bo < eo) {
      const uint32_t kB = min((bo + 31) / 32, lastc - 1);
      while (ready <= kB) {
        mbar_wait(&W.bar[ready % kRing], (ready / kRing) & 1);
        ready++;
      }
      const uint32_t nval = min(32u, no - bo);  // records that exist
      const uint32_t lim = min(32u, eo - bo);   // heads this range owns
      const bool valid = (uint32_t)lane < nval;
      Rec ra{};
      int kind = 7;
      if (valid) { ra = load_swz(R, (bo + lane) & kRM); kind = ra.kind(); }
      uint32_t nbo;
      if (P.dbg & 4) {  // diagnostic: stream only (roofline experiments)
        my_max_dev = max(my_max_dev, (int)(ra.dev ^ ra.rank));
        nbo = bo + 32;
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
        const unsigned below = H & (0xFFFFFFFFu >> (31 - lane));
        const int hA = below ? 31 - __clz(below) : 0;
        const uint32_t lenA = __shfl_sync(kFull, len, hA);
        if (mem && (uint32_t)lane >= (uint32_t)hA + lenA) badl = true;  // a record no element covers
        if (head && ((uint32_t)lane + len > nval || !range_clear((unsigned long long)Sall, (uint32_t)lane + 1, len - 1)))
          badl = true;  // runs past the trace, or another element starts inside this one
        const uint32_t a2 = ra.kc | (ra.ad << 8) | (ra.aux << 16);

        // ---------------- steady window: every element is a copy or a block of the steady
        // communicator repeating a known-valid signature with the devices of its last block
        // and increasing seqs.  Such blocks are valid instances with identical transfers:
        // count them per template and expand once, multiplied, at the next flush.
        bool steady = false;
        if (ts >= 0 && skip == 0) {
          bool okl = !badl;
          uint32_t ti = 0;
          const bool cl = mem && kind == CT_KIND_COLLECTIVE;
          if (cl) {
            const uint32_t sg = coll_sig(a2);
            const uint32_t set = tpl_set(ra.count, sg);
            const Tpl e0 = W.tpl[2 * set], e1 = W.tpl[2 * set + 1];
            const bool h0 = e0.count == ra.count && e0.sig == sg;
            const bool h1 = e1.count == ra.count && e1.sig == sg;
            ti = 2 * set + (h0 ? 0u : 1u);
            okl = okl && (h0 || h1) && ra.comm == tcomm && ra.nranks == tn && ra.rank == (uint32_t)(lane - hA) &&
                  ra.dev == W.cdev[ts][ra.rank & 31] && ra.dev < (uint32_t)P.gcap;
          } else if (mem) {
            okl = okl && kind >= CT_KIND_MEMCPY && kind <= CT_KIND_ZEROCOPY;
          }
          const unsigned Hc = __ballot_sync(kFull, head && kind == CT_KIND_COLLECTIVE);
          const uint32_t tiH = __shfl_sync(kFull, ti, hA);
          const unsigned lower = Hc & ((1u << hA) - 1);
          const int ph = lower ? 31 - __clz(lower) : -1;  // previous block of the comm in the window
          const int src = ph >= 0 ? ((ph + (int)ra.rank) & 31) : lane;
          const uint64_t pseq = ((uint64_t)__shfl_sync(kFull, (uint32_t)(ra.seq >> 32), src) << 32) |
                                __shfl_sync(kFull, (uint32_t)ra.seq, src);
          if (cl) {
            const uint64_t prev = ph >= 0 ? pseq : W.cseq[ts][ra.rank & 31];
            okl = okl && ti == tiH && prev < ra.seq;
          }
          if ((P.dbg & 8) && !okl) {  // diagnostic: why a steady attempt failed
            uint32_t why = badl ? 1u : 0u;
            if (cl) {
              const uint32_t sg = coll_sig(a2);
              const uint32_t set = tpl_set(ra.count, sg);
              const bool hit = (W.tpl[2 * set].count == ra.count && W.tpl[2 * set].sig == sg) ||
                               (W.tpl[2 * set + 1].count == ra.count && W.tpl[2 * set + 1].sig == sg);
              if (!hit) why |= 2;
              if (ra.comm != tcomm || ra.nranks != tn) why |= 4;
              if (ra.rank != (uint32_t)(lane - hA)) why |= 8;
              if (ra.dev != W.cdev[ts][ra.rank & 31]) why |= 16;
              if (ti != tiH) why |= 128;
              if (!((ph >= 0 ? pseq : W.cseq[ts][ra.rank & 31]) < ra.seq)) why |= 256;
            } else if (mem) {
              why |= 64;
            }
            atomicOr(&P.st->pad, why);
          }
          if (__all_sync(kFull, okl)) {
            steady = true;
            backoff = 0;
            if ((P.dbg & 8) && lane == 0) atomicAdd(&P.st->n_chain, 1u);
            if (Hc) {
              const int hLc = 31 - __clz(Hc);
              if (head && kind == CT_KIND_COLLECTIVE) atomicAdd(&W.tpl[ti].ndef, 1u);
              pending += __popc(Hc);
              if (cl && hA == hLc) W.cseq[ts][ra.rank] = ra.seq;
              if (lane == 0) W.clast[ts] = rb0 + bo + hLc;
              __syncwarp();
            }
            if (Hc != H && mem && kind != CT_KIND_COLLECTIVE && !(P.dbg & 1))
              expand_record(P, acc, wdv, ra, rb0, bo + lane, ST_VALID, bo + lane, my_max_dev, copy_seen);
          } else {
            if (backoff == 63) {  // long miss streak: drop stale templates
              W.tpl[lane].sig = 0;
              __syncwarp();
            }
            backoff = min(2 * backoff + 1, 63u);
            skip = backoff;
          }
        } else if (skip) {
          skip--;
        }

        if (!steady) {
          if (pending) {  // the general path may change the steady comm's devices: expand first
            acc.flags |= flush_templates<SH>(P.ex, hist_bytes<SH>(P), hist_freq<SH>(P), P.g2, W, ts, tcomm, tn);
            pending = 0;
          }
          // ---------------- member checks against the predecessor record (lane shuffles)
          // words: comm | nranks, rank | kc, ad, aux | count lo | count hi
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
          int uslot = -1;     // the single comm slot of the window's blocks (uniform case)
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
              uslot = su;
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
              const unsigned lt = (1u << lane) - 1;
              const unsigned same =
                  __match_any_sync(kFull, collH ? (unsigned long long)ra.comm : (0xFFFFFFFF00000000ull | lane)) & Hc;
              const unsigned lower = same & lt;
              const int ph = lower ? 31 - __clz(lower) : -1;
              const int hs = slot < 0 ? 0 : slot;
              const bool hist = collH && W.sn[hs] != 0;
              const uint32_t hinfo = (uint32_t)hs | ((uint32_t)(ph & 63) << 4) | (ph >= 0 ? 1u << 10 : 0u) |
                                     (hist ? 1u << 11 : 0u) | (hist && W.sver[hs] ? 1u << 12 : 0u) |
                                     ((same & ~lt & ~(1u << lane)) == 0 ? 1u << 13 : 0u);
              info = __shfl_sync(kFull, hinfo, hA);
            }
          }
          if (collH) {  // nranks constant per comm (grouping.py:104-108)
            const uint32_t pn = (info & (1u << 10)) ? R[(bo + ((info >> 4) & 63)) & kRM].nranks
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
            if ((needs_full >> lane) & 1) dist = devices_distinct(R, bo + lane, ra.nranks);
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
          if (head && st != ST_VALID) count_diag(st);

          // ---------------- p2p order: per (comm, src, dst) channel non-decreasing send and
          // recv seqs (decompose.py:359-361 sorts each side by seq; FIFO pairs by position)
          if (Hs) {
            const uint64_t nseq = ((uint64_t)__shfl_down_sync(kFull, (uint32_t)(ra.seq >> 32), 1) << 32) |
                                  __shfl_down_sync(kFull, (uint32_t)ra.seq, 1);
            p2p_order(P.chans + (size_t)gw * kPC, ra, nseq, sendH, lane, wflags);
          }

          // ---------------- table update with the last block of each comm in the window
          __syncwarp();
          if (cm && (info & (1u << 13))) { W.cseq[info & 15][ra.rank] = ra.seq; W.cdev[info & 15][ra.rank] = (uint16_t)ra.dev; }
          if (collH) {
            const int hs = info & 15;
            const uint64_t gi = rb0 + bo + lane;
            if (!(info & (3u << 10))) W.cfirst[hs] = gi;  // first block of this comm in the range
            if (info & (1u << 13)) { W.sn[hs] = ra.nranks; W.sver[hs] = dist; W.clast[hs] = gi; }
          }
          if (Hc) {  // first valid instance per (comm slot, type): only until recorded once
            const unsigned long long bit = (collH && st == ST_VALID) ? 1ull << ((info & 15) * 5 + ra.coll()) : 0ull;
            const bool rec = (bit & tf_pend) != 0;
            if (rec) note_min_smem(&W.tfirst[info & 15][ra.coll()], rb0 + bo + lane);
            const unsigned lo = __reduce_or_sync(kFull, rec ? (unsigned)bit : 0u);
            const unsigned hi = __reduce_or_sync(kFull, rec ? (unsigned)(bit >> 32) : 0u);
            tf_pend &= ~(((unsigned long long)hi << 32) | lo);
          }
          __syncwarp();

          // ---------------- expansion + accumulation
          if (mem && !(P.dbg & 1))
            expand_record(P, acc, wdv, ra, rb0, bo + lane, st, bo + (uint32_t)hA, my_max_dev, copy_seen);

          // ---------------- steady comm and templates: the window's last block, when valid
          if (ts >= 0 && !W.sver[ts]) ts = -1;  // duplicate devices: repeats are not valid
          if (Hc && uslot >= 0) {
            const int hLc = 31 - __clz(Hc);
            if (__shfl_sync(kFull, st, hLc) == ST_VALID && W.sver[uslot] && uslot != ts) {
              W.tpl[lane].sig = 0;
              ts = uslot;
              tcomm = __shfl_sync(kFull, ra.comm, hLc);
              tn = __shfl_sync(kFull, ra.nranks, hLc);
              skip = backoff = 0;
            }
            __syncwarp();
            if (ts == uslot && skip <= 3 && collH && st == ST_VALID) {  // valid signatures before an attempt
              const uint32_t sg = coll_sig(a2);
              const uint32_t set = tpl_set(ra.count, sg);
              Tpl* e = &W.tpl[2 * set];
              const bool in0 = e[0].count == ra.count && e[0].sig == sg;
              const bool in1 = e[1].count == ra.count && e[1].sig == sg;
              if (!in0 && !in1) {  // empty way first, else replace way (seq & 1); racing lanes only cost hits
                const int way = e[0].sig == 0 ? 0 : (e[1].sig == 0 ? 1 : (int)(ra.seq & 1));
                e[way].count = ra.count;
                e[way].sig = sg;
                e[way].ndef = 0;
              }
            }
            __syncwarp();
          }
        }  // general path
        nbo = bo + Pw;
      }

      // ---------------- slide: chunks wholly behind the next window refill their slots
      const uint32_t kf = nbo / 32;
      if (kf > freed) {
        __syncwarp();
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        do {
          const uint32_t q = freed + kRing;
          if (q < lastc) {
            if (lane == 0) {
              const uint64_t first = (k0 + q) * 32;
              bulk_load(W.ring[freed % kRing], P.recs + first,
                        (uint32_t)min((uint64_t)32, P.n - first) * (uint32_t)sizeof(ct_record), &W.bar[freed % kRing]);
            }
            issued = q + 1;
          }
          freed++;
        } while (freed < kf);
      }
      bo = nbo;
    }
    if (pending) acc.flags |= flush_templates<SH>(P.ex, hist_bytes<SH>(P), hist_freq<SH>(P), P.g2, W, ts, tcomm, tn);
    for (uint32_t q = ready; q < issued; q++)  // drain outstanding bulk copies
      mbar_wait(&W.bar[q % kRing], (q / kRing) & 1);
  }

  if ((P.dbg & 16) && lane == 0)  // diagnostic: slowest warp (cycles << 24 | warp)
    atomicMax(&P.st->err_index, ((unsigned long long)(clock64() - t_start) << 24) | gw);

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
  if (acc.flags | wflags) atomicOr(&C.flags, acc.flags | wflags);
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
    if (C.oor_key != kNone) atomicMin(&G->oor_key, C.oor_key);
    if (C.of_cell != kNone) atomicMin(&G->of_cell, C.of_cell);
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
