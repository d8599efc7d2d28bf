// Rank-attributed expansion of one collective record of a VALID instance, shared by
// the accumulate kernel (fast path) and the emit kernel (decompose_* API).
// ``Sink`` provides stat(type, S), edge(type, src, dst, bytes) and flags; endpoints are
// gpu ids, -1 host, -2 net.  ``DevOf`` maps a record index to its device.
#pragma once
#include "ct_common.cuh"

namespace ct {

struct ExpandParams {
  int ring_len;
  int ring_valid;
  const uint16_t* ring_order;
  const uint16_t* ring_inv;
  uint64_t tree_threshold;
};

// Expand one collective record of a valid instance (rank-attributed).
template <typename U, typename Sink, typename DevOf>
__device__ void expand_collective(const ExpandParams& P, const DevOf& v, Sink& acc, const Rec& rc,
                                  uint64_t head) {
  const int n = rc.nranks, r = rc.rank, coll = rc.coll();
  const U blk = (U)rc.count * (U)dtype_width(rc.dtype());
  const bool scatter = coll == CT_COLL_ALLGATHER || coll == CT_COLL_REDUCESCATTER;
  const U s = scatter ? blk * (U)n : blk;
  int algo = rc.algo();
  if (coll == CT_COLL_ALLREDUCE) {
    if (algo == CT_ALGO_AUTO) algo = s < (U)P.tree_threshold ? CT_ALGO_TREE : CT_ALGO_RING;
  } else {
    if (algo == CT_ALGO_TREE || algo == CT_ALGO_COLLNET) { acc.flags |= F_WRONG_ALGO; return; }
    algo = CT_ALGO_RING;
  }
  const int type = coll;
  if (r == 0) acc.stat(type, (unsigned __int128)s);
  const int me = (int)rc.dev;
  if (algo == CT_ALGO_COLLNET) {
    if (s != 0) {
      acc.edge(type, me, -2, (unsigned __int128)s, 0);
      acc.edge(type, -2, me, (unsigned __int128)s, 1);
    }
    return;
  }
  if ((coll == CT_COLL_BROADCAST || coll == CT_COLL_REDUCE) && !rc.has_root()) {
    acc.flags |= F_MISSING_ROOT;
    return;
  }
  if (n == 1 || s == 0) return;
  if (algo == CT_ALGO_TREE) {
    // T1 carries ceil(S/2), T2 floor(S/2) (skipped when 0); an edge present in both
    // trees is one transfer carrying S (decompose.py:242-255).  Scalars only, so the
    // neighbour lists stay in registers.
    const U share1 = s - s / 2, share2 = s / 2;
    int a0, a1, a2, b0, b1, b2;
    tree_links(n, r, a0, a1, a2);  // T1: rank == position
    if (share2 != 0) {
      int q0, q1, q2;
      tree_links(n, r == 0 ? n - 1 : r - 1, q0, q1, q2);  // T2: rank at position q is (q + 1) % n
      b0 = q0 < 0 ? -1 : (q0 + 1 == n ? 0 : q0 + 1);
      b1 = q1 < 0 ? -1 : (q1 + 1 == n ? 0 : q1 + 1);
      b2 = q2 < 0 ? -1 : (q2 + 1 == n ? 0 : q2 + 1);
    } else {
      b0 = b1 = b2 = -1;
    }
#pragma unroll
    for (int i = 0; i < 3; i++) {
      const int x = i == 0 ? a0 : i == 1 ? a1 : a2;
      if (x < 0) continue;
      const bool both = x == b0 || x == b1 || x == b2;
      acc.edge(type, me, (int)v.dev_of(head + x), (unsigned __int128)(both ? share1 + share2 : share1), x);
    }
#pragma unroll
    for (int i = 0; i < 3; i++) {
      const int y = i == 0 ? b0 : i == 1 ? b1 : b2;
      if (y < 0 || y == a0 || y == a1 || y == a2) continue;
      acc.edge(type, me, (int)v.dev_of(head + y), (unsigned __int128)share2, y);
    }
    return;
  }
  int p, succ, root_pos = 0;
  if (n == P.ring_len) {
    if (!P.ring_valid) { acc.flags |= F_BAD_RING; return; }
    p = P.ring_inv[r];
    succ = P.ring_order[p + 1 == n ? 0 : p + 1];
    if (rc.has_root()) root_pos = P.ring_inv[rc.aux];
  } else {
    p = r;
    succ = r + 1 == n ? 0 : r + 1;
    root_pos = rc.aux;
  }
  U bytes;
  switch (coll) {
    case CT_COLL_ALLREDUCE: {
      const U chunk = ceil_div(s, (uint32_t)n);
      int p1 = p + 1 == n ? 0 : p + 1;
      int p2 = p1 + 1 == n ? 0 : p1 + 1;
      U o1 = (U)p1 * chunk, o2 = (U)p2 * chunk;
      U b1 = o1 >= s ? (U)0 : (s - o1 < chunk ? s - o1 : chunk);
      U b2 = o2 >= s ? (U)0 : (s - o2 < chunk ? s - o2 : chunk);
      bytes = 2 * s - b1 - b2;
      break;
    }
    case CT_COLL_ALLGATHER:
    case CT_COLL_REDUCESCATTER:
      bytes = s - blk;
      break;
    case CT_COLL_BROADCAST:
      if (p == (root_pos == 0 ? n - 1 : root_pos - 1)) return;
      bytes = s;
      break;
    default:  // reduce
      if (p == root_pos) return;
      bytes = s;
      break;
  }
  if (bytes != 0) acc.edge(type, me, (int)v.dev_of(head + succ), (unsigned __int128)bytes, succ);
}


}  // namespace ct
