// Exact path: sort-based join that canonicalizes an arbitrary trace.
//
// The reference groups collectives by (comm, ordinal) where the ordinal is the
// record's position in its (comm, rank) stream sorted by seq (grouping.py:82-183), and
// pairs sends with recvs FIFO per (comm, src, dst) in seq order (decompose.py:342-394).
// This path computes both joins on the device with CUB radix sorts and writes a
// canonical record stream the fast kernel accepts:
//   [complete collective groups, ranks 0..n-1 consecutive, in (comm first-seen,
//    ordinal) order] [send,recv adjacent pairs per channel in FIFO order]
//   [copies in file order]
// Incomplete groups and unmatched sends/recvs are counted here (they never reach the
// canonical stream); incompatible / duplicate-device groups and mismatched pairs are
// carried through and classified by the fast kernel exactly as on canonical input.
// Fatal conditions (nranks disagreement, duplicate seq) are detected here with the
// reference's precedence and message fields.
#pragma once
#include <vector>

#include "ct_common.cuh"

namespace ct {

struct GroupRow {      // one reference-ordered collective group (for materialisation)
  uint64_t comm, ordinal, status, n_members, member_off;
};
struct P2PDiagRow {    // one p2p diagnostic (mismatched / unmatched)
  uint64_t reason, comm, src, dst, k, send_idx, recv_idx;
};

struct ExactResult {
  ct_record* canon = nullptr;   // device, cudaFreeAsync by caller
  uint64_t m = 0;               // canonical records
  uint64_t n_incomplete = 0, n_unmatched_send = 0, n_unmatched_recv = 0;
  int fatal = 0;                // 0 none, CT_ERR_INVARIANT
  int fatal_kind = 0;           // 1 nranks disagreement, 2 duplicate seq
  uint64_t err_index = 0, err_aux[4] = {0, 0, 0, 0};
  uint32_t launches = 0;
  // materialisation (filled when requested)
  std::vector<GroupRow> groups;
  std::vector<uint64_t> members;      // original record indices, rows concatenated
  std::vector<P2PDiagRow> p2p_diags;
  std::vector<uint64_t> canon_src;    // canonical position -> original record index
};

// Returns cudaError_t as int; ``res`` filled.  ``materialize`` also returns the
// group / diagnostic lists and the canonical->original index map.
// exact_canonicalize's return value when a per-(comm, rank) ordinal would not fit the
// 32-bit group key (>= 2^32 collective records): the caller reports CT_ERR_CAPACITY
constexpr int kExactCapacity = 0x7FFF0001;

int exact_canonicalize(const ct_record* recs, uint64_t n, uint32_t n_comms, cudaStream_t st,
                       bool materialize, ExactResult* res);

}  // namespace ct
