// The fused expand + accumulate kernel (fast path) and its parameters.
//
// One persistent CTA per SM streams a contiguous range of the packed trace through
// shared memory with 1-D TMA bulk copies (cp.async.bulk + mbarrier, STAGES deep).
// Per sub-tile of SUB records:
//   A1  decode; verify the canonical layout locally (collective records form blocks
//       of ranks 0..n-1 on one comm; every send is followed by its recv); block heads
//       compute instance validity (grouping.py:144-167); sends compute pair status.
//   A2  compact chain elements (block heads, sends) in position order.
//   A3  chain check, partitioned across warps by key hash: consecutive blocks of one
//       comm must have strictly increasing seq per rank and equal nranks, consecutive
//       pairs of one (comm, src, dst) channel non-decreasing seqs — exactly the
//       conditions under which the reference's seq-sorted grouping/matching
//       (grouping.py:118-131, decompose.py:357-361) coincides with file order.
//   B   per-record expansion (ct_common.cuh) into a per-thread register cache of
//       (cell, bytes, count) entries; evictions go to a shared-memory histogram.
// At the end each CTA flushes its caches and merges its histogram and statistics into
// global memory once.  Chain first/last elements per CTA go to a small list that
// ct_chain_check validates across CTAs.  Any failed precondition raises F_NONCANON and
// the host reruns through the exact (sort-based) path.
#pragma once
#include "ct_expand.cuh"

namespace ct {

constexpr int kSub = 1024;      // records per sub-tile (32 KB)
constexpr int kStages = 3;      // TMA ring depth
constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int kPer = kSub / kThreads;
constexpr int kCacheE = 4;      // register cache entries per thread
constexpr int kChainW = 32;     // chain-table entries per warp
constexpr int kCommSm = 64;     // comms tracked in shared memory for first-occurrence keys
constexpr uint32_t kChainSortMax = 4096;  // single-CTA cross-CTA chain sort capacity

struct ChainEntry {
  uint64_t key, first, last;
};

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

struct FastParams {
  const ct_record* recs;      // analyzed array (device)
  uint64_t n;                 // records
  uint64_t base;              // global index of recs[0] (multi-GPU shards)
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
  ChainEntry* chain;          // cross-CTA chain list
  uint32_t chain_cap;
  uint32_t subs_per_cta;
  uint32_t n_subs;
};

size_t fast_smem_bytes(int g2, int smem_hist);

}  // namespace ct
