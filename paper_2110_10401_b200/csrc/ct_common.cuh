// Shared device definitions: record decoding, the reference's algorithm models in
// rank-attributed (per-record) form, and accumulation helpers.
//
// Every collective transfer of a valid instance has exactly one source rank, so
// emitting from each record only the edges whose source is its own rank reproduces
// the reference's per-instance decompositions exactly:
//   ring AR   decompose.py:130-153   edge p -> p+1 : 2S - b[p+1] - b[p+2]
//   AG / RS   decompose.py:156-189   S - b[p+1] / S - b[p]  (== (n-1)*block)
//   bcast     decompose.py:192-224   every position except root-1 sends S
//   reduce    decompose.py:200-224   every position except root sends S
//   tree      decompose.py:227-255   to parent and children in T1 (ceil S/2) and T2
//                                    (floor S/2, skipped if 0); same-peer edges merge
//   collnet   decompose.py:258-273   dev->NET and NET->dev, S each (incl. n == 1)
//   auto      decompose.py:276-289   allreduce: tree if S < threshold else ring
//   p2p       decompose.py:319-339   send dev -> recv dev if they differ, 0 kept
//   copy      decompose.py:397-406   src -> dst, 0 kept
// 0-byte collective edges are dropped (decompose.py:96).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/commtrace_b200.h"

namespace ct {

constexpr int kTypes = CT_NTYPES;
constexpr uint32_t kStatsKeyBit = 0x80000000u;

// internal endpoint indices (independent of d): host 0, net 1, gpu g -> g + 2
constexpr int kHost = 0;
constexpr int kNet = 1;

// status codes written per element (block head / send)
enum : uint8_t { ST_NONE = 0, ST_VALID = 1, ST_INCOMPAT = 2, ST_DUPDEV = 3, ST_MISMATCH = 4 };

// flag bits in State::flags
enum : uint32_t {
  F_NONCANON = 1u << 0,   // fast-path layout precondition failed
  F_OVERFLOW = 1u << 1,   // a cell sum exceeded 2^63-1 (or wrapped)
  F_OOR = 1u << 2,        // accumulated transfer endpoint gpu >= d (explicit d)
  F_CAP = 1u << 3,        // gpu id >= g_cap with inferred d: rerun with larger g_cap
  F_BAD_RING = 1u << 4,   // invalid ring order used by a ring instance
  F_WRONG_ALGO = 1u << 5,
  F_MISSING_ROOT = 1u << 6,
  F_COMM_RANGE = 1u << 8, // comm id >= n_comms
};

__host__ __device__ inline int dtype_width(int code) {
  // int8 uint8 int32 uint32 int64 uint64 float16 bfloat16 float32 float64 (events.py:109-120)
  return (int)((0x8422884411ull >> (4 * code)) & 0xF);
}

struct Rec {  // register view of ct_record (two 128-bit words)
  uint64_t count, seq;
  uint32_t comm;
  uint32_t nranks, rank, dev, aux, aux2;
  uint32_t kc, ad;
  __device__ __forceinline__ int kind() const { return kc & 7; }
  __device__ __forceinline__ int coll() const { return (kc >> 3) & 7; }
  __device__ __forceinline__ bool has_root() const { return (kc >> 6) & 1; }
  __device__ __forceinline__ int algo() const { return ad & 3; }
  __device__ __forceinline__ int dtype() const { return (ad >> 2) & 15; }
  __device__ __forceinline__ int ckind() const { return (ad >> 6) & 3; }
};

__device__ __forceinline__ Rec unpack(uint4 a, uint4 b) {
  Rec r;
  r.count = ((uint64_t)a.y << 32) | a.x;
  r.seq = ((uint64_t)a.w << 32) | a.z;
  r.comm = b.x;
  r.nranks = b.y & 0xFFFF;
  r.rank = b.y >> 16;
  r.dev = b.z & 0xFFFF;
  r.aux = b.z >> 16;
  r.aux2 = b.w & 0xFFFF;
  r.kc = (b.w >> 16) & 0xFF;
  r.ad = b.w >> 24;
  return r;
}

__device__ __forceinline__ Rec load_global(const ct_record* p) {
  const uint4* q = reinterpret_cast<const uint4*>(p);
  return unpack(__ldg(q), __ldg(q + 1));
}

__device__ __forceinline__ Rec load_shared(const ct_record* p) {
  const uint4* q = reinterpret_cast<const uint4*>(p);
  return unpack(q[0], q[1]);
}

// collective signature equality (grouping.py:78-79): coll, algo, count, dtype, root
__device__ __forceinline__ bool same_sig(const Rec& a, const Rec& b) {
  return ((a.kc ^ b.kc) & 0x78) == 0 && ((a.ad ^ b.ad) & 0x3F) == 0 && a.count == b.count &&
         (!a.has_root() || a.aux == b.aux);
}

// in-order binary tree over positions [0, n) (trees.py:57-78): parent and children of pos
__device__ __forceinline__ int subtree_root(int lo, int hi) {
  return lo + (1 << (31 - __clz(hi - lo))) - 1;
}

__device__ __forceinline__ void tree_links(int n, int pos, int& parent, int& left, int& right) {
  int lo = 0, hi = n;
  parent = -1;
  while (true) {
    int root = subtree_root(lo, hi);
    if (pos == root) {
      left = root > lo ? subtree_root(lo, root) : -1;
      right = root + 1 < hi ? subtree_root(root + 1, hi) : -1;
      return;
    }
    parent = root;
    if (pos < root) hi = root; else lo = root + 1;
  }
}

// Up to 6 peer edges of a tree-allreduce record, merged per peer: bit 0 of ``trees``
// = the edge exists in T1 (carries ceil(S/2)), bit 1 = in T2 (carries floor(S/2)).
struct TreeEdges {
  int dst[6];
  uint32_t trees[6];
  int n;
  __device__ __forceinline__ void add(int d, uint32_t t) {
#pragma unroll
    for (int e = 0; e < 6; e++)
      if (e < n && dst[e] == d) { trees[e] |= t; return; }
    dst[n] = d; trees[n] = t; n++;
  }
};

// Peers of rank r in the double binary tree over n ranks (trees.py:81-106); T2 edges
// are included only when its share floor(S/2) is non-zero (decompose.py:245-246).
__device__ __forceinline__ void tree_edges(int n, int r, bool with_t2, TreeEdges& te) {
  te.n = 0;
  int p, l, rr;
  tree_links(n, r, p, l, rr);  // T1: rank == position
  if (p >= 0) te.add(p, 1);
  if (l >= 0) te.add(l, 1);
  if (rr >= 0) te.add(rr, 1);
  if (with_t2) {  // T2: rank at position q is (q + 1) % n
    int q = r == 0 ? n - 1 : r - 1;
    tree_links(n, q, p, l, rr);
    if (p >= 0) te.add(p + 1 == n ? 0 : p + 1, 2);
    if (l >= 0) te.add(l + 1 == n ? 0 : l + 1, 2);
    if (rr >= 0) te.add(rr + 1 == n ? 0 : rr + 1, 2);
  }
}

// floor(s / n) for a small divisor without the 64-bit integer division sequence: one
// double-precision reciprocal multiply (exact to +-1 for s < 2^52) and one correction.
__device__ __forceinline__ uint64_t udiv_small(uint64_t s, uint32_t n) {
  if (s < (1ull << 52)) {
    uint64_t q = (uint64_t)((double)s * __drcp_rn((double)n));
    const int64_t r = (int64_t)(s - q * n);
    if (r < 0) q--;
    else if (r >= (int64_t)n) q++;
    return q;
  }
  return s / n;
}

__device__ __forceinline__ uint64_t ceil_div(uint64_t s, uint32_t n) {
  if ((n & (n - 1)) == 0) {  // power-of-two communicators (the common 2 / 4 / 8): a shift
    const uint32_t k = 31 - __clz(n);
    return (s >> k) + ((s & (n - 1)) != 0 ? 1 : 0);
  }
  const uint64_t q = udiv_small(s, n);
  return q + (q * n != s ? 1 : 0);
}

__device__ __forceinline__ unsigned __int128 ceil_div(unsigned __int128 s, uint32_t n) {
  return (s + (unsigned __int128)(n - 1)) / (unsigned __int128)n;
}

// ring block size b[i] for an n-way split of s with chunk = ceil(s/n) (decompose.py:104-107)
__device__ __forceinline__ uint64_t ring_block(uint64_t s, uint64_t chunk, int i) {
  uint64_t off = (uint64_t)i * chunk;
  if (off >= s) return 0;
  uint64_t rest = s - off;
  return rest < chunk ? rest : chunk;
}

}  // namespace ct
