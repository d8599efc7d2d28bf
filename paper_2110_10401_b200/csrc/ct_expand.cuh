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
    const U share1 = s - s / 2, share2 = s / 2;
    TreeEdges te;
    tree_edges(n, r, share2 != 0, te);
#pragma unroll 1
    for (int e = 0; e < te.n; e++) {
      const U b = ((te.trees[e] & 1) ? share1 : (U)0) + ((te.trees[e] & 2) ? share2 : (U)0);
      acc.edge(type, me, (int)v.dev_of(head + te.dst[e]), (unsigned __int128)b, te.dst[e]);
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
