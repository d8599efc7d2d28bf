// The fused layout-check + join + expand + accumulate kernel (fast path).
//
// Element-parallel streaming design (no block-wide barriers in the main loop):
//   * every warp owns a contiguous range of the packed trace, cut at element starts
//     (a collective rank-0 record, a send, or a copy), and streams it through its own
//     ring of 1 KB TMA bulk copies (cp.async.bulk + mbarrier, kRing slots deep);
//   * scan (lane = record, one 32-record chunk at a time): element heads appended to a
//     per-warp element queue, copies expanded in place (one transfer each);
//   * join (lane = element, up to 32 queued elements, run when the ring is full): each
//     lane walks its block's records comparing raw words with the head -- membership,
//     signature (grouping.py:78-79, 132-155), one seq per block or per rank against the
//     comm's previous block (same batch: the ring; else the per-warp table), distinct
//     devices (grouping.py:156-167) -- and the element lengths plus copies must tile the
//     range exactly;
//   * expansion of valid instances (rank-attributed rules, ct_common.cuh): repeated
//     uniform-ring instances go to a per-lane register accumulator, repeated ring / tree
//     / collnet / broadcast / reduce instances to per-warp shared slot accumulators, the
//     rest edge by edge -- all into the CTA's shared-memory histogram (32-bit limbs);
//   * each CTA merges its histogram and statistics into global memory once at the end.
// Seq-order preconditions (exactly when the reference's seq-sorted grouping and FIFO
// matching coincide with file order, grouping.py:118-131, decompose.py:357-361):
//   collectives: per (comm, rank) strictly increasing seq, constant nranks per comm;
//   p2p:         per (comm, src, dst) channel non-decreasing send seqs and recv seqs.
// Violations (and anything else non-canonical) raise F_NONCANON; the host then runs the
// exact sort-based join (ct_exact.cu) and feeds its canonical stream back through here.
#pragma once
#include "ct_expand.cuh"

namespace ct {

#ifndef CT_WARPS
#define CT_WARPS 16
#endif
constexpr int kThreads = 32 * CT_WARPS;  // one CTA per SM
constexpr int kWarps = kThreads / 32;
#ifndef CT_RING_SLOTS
#define CT_RING_SLOTS 8
#endif
constexpr int kRing = CT_RING_SLOTS;  // per-warp TMA ring slots of 32 records (1 KB each)
constexpr int kCS = 8;          // collective communicator slots per warp
constexpr int kPC = 64;         // p2p channel table entries per warp (open addressing, global memory)
constexpr int kMaxN = 32;       // largest communicator the fast path handles
constexpr int kQ = 128;         // element queue entries per warp (< 32 carried + 2 chunks of heads)

struct GlobalState {
  uint32_t flags;
  int32_t max_dev;
  uint32_t unused0;
  uint32_t unused1;
  unsigned long long diag[CT_NDIAG];
  unsigned long long calls[kTypes];
  unsigned long long pay_lo[kTypes];
  unsigned long long pay_hi[kTypes];
  unsigned long long copy_first[3];
  unsigned long long err_index;
  unsigned long long oor_key;   // min (class, element, src rank, dst rank, which) of an out-of-range endpoint
  unsigned long long of_cell;   // min internal cell index whose 64-bit sum wrapped
};

// Per (warp range, comm slot) summary for the cross-range seq-order check.
struct WarpSlot {
  uint32_t comm;        // ~0u: unused
  uint32_t n;           // collective nranks (0: no collectives)
  uint64_t coll_first;  // first / last collective block head of this comm in the range
  uint64_t coll_last;
};

// Per (warp range, p2p channel): the channel key (comm << 32 | src << 16 | dst; ~0 unused)
// and its first / last send and recv seq in the range, as structure-of-arrays over one
// buffer of 5 * n u64 (lookups touch only the keys and last seqs: 24 B per entry in L1).
struct Chans {
  uint64_t* base;
  uint64_t n;  // entries (total warps * kPC)
  __device__ __forceinline__ uint64_t& key(uint64_t i) const { return base[i]; }
  __device__ __forceinline__ uint64_t& last_s(uint64_t i) const { return base[n + 2 * i]; }
  __device__ __forceinline__ uint64_t& last_r(uint64_t i) const { return base[n + 2 * i + 1]; }
  __device__ __forceinline__ uint64_t& first_s(uint64_t i) const { return base[3 * n + 2 * i]; }
  __device__ __forceinline__ uint64_t& first_r(uint64_t i) const { return base[3 * n + 2 * i + 1]; }
};
constexpr int kChanWords = 5;  // u64 per channel entry

struct FastParams {
  const ct_record* recs;      // analyzed array (device)
  uint64_t n;                 // records
  int gcap;                   // GPUs covered by the histogram
  int g2;                     // gcap + 2
  int explicit_d;             // 1: gcap == d, gpu >= d raises EndpointOutOfRange
  ExpandParams ex;            // ring order / inverse (device), tree threshold
  uint32_t n_comms;
  int smem_hist;              // 1: CTA histogram in shared memory
  GlobalState* st;
  unsigned long long* cells;  // [kTypes][g2][g2] bytes
  unsigned long long* freq;   // [kTypes][g2][g2]
  unsigned long long* type_comm_first;  // [5][n_comms] first valid head per (type, comm)
  unsigned long long* comm_first;       // [n_comms] first collective head per comm
  WarpSlot* slots;            // [total warps][kCS]
  Chans chans;                // [total warps][kPC] entries
  uint32_t total_warps;
  uint64_t n_chunks;          // ceil(n / 32)
  uint32_t sa_flush;          // slot accumulator write-out threshold (instances, <= 2^14)
  int dbg;                    // diagnostic knobs (CT_DEBUG_MODE): 1 skip expansion, 4 stream only
};

size_t fast_smem_bytes(int g2, int smem_hist);

}  // namespace ct
