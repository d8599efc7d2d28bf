// The fused layout-check + join + expand + accumulate kernel (fast path).
//
// Warp-autonomous streaming design (no block-wide barriers in the main loop):
//   * every warp owns a contiguous range of the packed trace, cut at element starts
//     (a collective rank-0 record, a send, or a copy), and streams it through its own
//     ring of 1 KB TMA bulk copies (cp.async.bulk + mbarrier, kRing slots deep);
//   * it walks the range in 64-record windows: elements starting in the first 32
//     positions are processed whole (n <= 32 keeps every element inside the window),
//     the window then slides by 32 and the carry skips the records already consumed;
//   * element structure, instance validity (signature equality, distinct devices,
//     grouping.py:132-167), pair matching and the seq-order preconditions are decided
//     with ballots over the window and broadcast shared-memory reads of the heads;
//   * per-(comm, rank) state of the last block (seq, device) lives in a small per-warp
//     table, so a block is validated against its predecessor in O(1) per record;
//   * transfers go into a per-thread register cache and spill to a per-CTA shared
//     histogram; each CTA merges into global memory once at the end.
// Seq-order preconditions (exactly when the reference's seq-sorted grouping and FIFO
// matching coincide with file order, grouping.py:118-131, decompose.py:357-361):
//   collectives: per (comm, rank) strictly increasing seq, constant nranks per comm;
//   p2p:         per (comm, src, dst) channel non-decreasing send seqs and recv seqs.
// Violations (and anything else non-canonical) raise F_NONCANON; the host then runs the
// exact sort-based join (ct_exact.cu) and feeds its canonical stream back through here.
#pragma once
#include "ct_expand.cuh"

namespace ct {

constexpr int kThreads = 512;   // 16 warps, one CTA per SM
constexpr int kWarps = kThreads / 32;
#ifndef CT_RING_SLOTS
#define CT_RING_SLOTS 8
#endif
constexpr int kRing = CT_RING_SLOTS;  // per-warp TMA ring slots of 32 records (1 KB each)
constexpr int kCS = 8;          // collective communicator slots per warp
constexpr int kPC = 64;         // p2p channel table entries per warp
constexpr int kMaxN = 32;       // largest communicator the fast path handles
constexpr int kCacheE = 4;      // register cache entries per thread

struct GlobalState {
  uint32_t flags;
  int32_t max_dev;
  uint32_t n_chain;
  uint32_t pad;
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

// Per (warp range, p2p channel) summary: first / last send and recv seq in the range.
struct P2PEntry {
  uint64_t key;         // comm << 32 | src << 16 | dst; ~0: unused
  uint64_t first_s, first_r, last_s, last_r;
};

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
  P2PEntry* chans;            // [total warps][kPC]
  uint32_t total_warps;
  uint64_t n_chunks;          // ceil(n / 32)
  int dbg;                    // diagnostic knobs (CT_DEBUG_MODE): 1 skip expansion, 4 stream only
};

size_t fast_smem_bytes(int g2, int smem_hist);

}  // namespace ct
