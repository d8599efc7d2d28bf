// Device JSONL loader: reference wire text -> packed ct_record stream.
//
// Replaces the bulk of parse_trace (reference events.py:352-384, field readers
// events.py:294-349, validate events.py:166-236) followed by the record packing of
// packed.pack_events.  Three phases, all on the device:
//   1. line breaks: every byte position that starts a str.splitlines() terminator
//      (\n, \r, \r\n, \v, \f, \x1c-\x1e, U+0085, U+2028, U+2029) -> ordered list
//   2. one thread per line: JSON grammar, the reference's key/type reading order and
//      TraceEvent.validate rules, packed-range checks -> record + ts, or "blank", or
//      "deferred"
//   3. comm interning in first-seen order: 64-bit FNV-1a key per record, stable radix
//      sort, segment heads, byte-exact verification against each segment's first
//      name, segments ranked by first record index.
// A line is deferred whenever the device cannot prove that the reference accepts it
// unchanged: non-ASCII bytes, backslash escapes, control characters, floats / bools /
// null / big integers in consulted keys, missing keys, any grammar or validation
// failure.  The host parses exactly those lines with the reference-mirroring reader
// (events._parse_line), which raises the reference's exception for the first bad
// line; device-accepted lines can never raise, so error order is preserved.
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/commtrace_b200.h"

namespace {

constexpr uint64_t kNoKey = ~0ull;  // sort key of records without a device comm name

enum : uint8_t { L_BLANK = 0, L_OK = 1, L_DEFER = 2 };

// ---------------------------------------------------------------- phase 1: breaks

struct BreakPred {
  const uint8_t* s;
  uint64_t n;
  __device__ __forceinline__ bool operator()(uint64_t i) const {
    const uint8_t b = s[i];
    if (b == '\n') return i == 0 || s[i - 1] != '\r';  // \r\n is one terminator
    if (b == '\r' || b == 0x0b || b == 0x0c || b == 0x1c || b == 0x1d || b == 0x1e) return true;
    if (b == 0xC2) return i + 1 < n && s[i + 1] == 0x85;
    if (b == 0xE2) return i + 2 < n && s[i + 1] == 0x80 && (s[i + 2] == 0xA8 || s[i + 2] == 0xA9);
    return false;
  }
};

struct BreakCount {
  BreakPred p;
  __device__ __forceinline__ uint64_t operator()(uint64_t i) const { return p(i) ? 1u : 0u; }
};

__device__ __forceinline__ uint64_t break_len(const uint8_t* s, uint64_t n, uint64_t i) {
  const uint8_t b = s[i];
  if (b == '\r') return i + 1 < n && s[i + 1] == '\n' ? 2 : 1;
  if (b == 0xC2) return 2;
  if (b == 0xE2) return 3;
  return 1;
}

// ---------------------------------------------------------------- phase 2: parse

// top-level keys the reader consults (events.py:294-349)
enum Key : int { K_SEQ, K_TS, K_KIND, K_COMM, K_NRANKS, K_RANK, K_DEV, K_COLL, K_ALGO, K_COUNT,
                 K_DTYPE, K_ROOT, K_PEER, K_CKIND, K_SRC, K_DST, K_BYTES, K_N };

__constant__ char kKeyNames[K_N][8] = {"seq", "ts", "kind", "comm", "nranks", "rank", "dev", "coll",
                                       "algo", "count", "dtype", "root", "peer", "ckind", "src",
                                       "dst", "bytes"};
__constant__ char kKinds[6][12] = {"collective", "send", "recv", "memcpy", "um", "zerocopy"};
__constant__ char kColls[5][14] = {"allreduce", "broadcast", "reduce", "reducescatter", "allgather"};
__constant__ char kAlgos[4][8] = {"ring", "tree", "collnet", "auto"};
__constant__ char kDtypes[10][9] = {"int8", "uint8", "int32", "uint32", "int64", "uint64",
                                    "float16", "bfloat16", "float32", "float64"};
__constant__ char kCkinds[3][4] = {"h2d", "d2h", "d2d"};
__constant__ char kEpKinds[3][5] = {"host", "gpu", "net"};

// value types: absent, int >= 0 (fits u64), int < 0 (fits i64), plain string, endpoint
// object, anything else (float, bool, null, array, other object, huge int)
enum : uint8_t { V_NONE = 0, V_UINT, V_NINT, V_STR, V_EP, V_OTHER };

struct Val {
  uint8_t t;
  uint64_t u;        // V_UINT value / V_NINT two's complement
  uint32_t off, len;  // V_STR
  // V_EP: endpoint kind code (-1 invalid / absent) and index (-1 invalid / absent)
  int ep_kind;
  int64_t ep_idx;
};

__device__ __forceinline__ bool is_ws(uint8_t c) { return c == ' ' || c == '\t'; }

__device__ __forceinline__ uint64_t skip_ws(const uint8_t* s, uint64_t p, uint64_t e) {
  while (p < e && is_ws(s[p])) p++;
  return p;
}

template <int N, int W>
__device__ __forceinline__ int match(const uint8_t* s, uint32_t off, uint32_t len, const char (&tab)[N][W]) {
  for (int k = 0; k < N; k++) {
    uint32_t j = 0;
    while (j < len && j < (uint32_t)W && tab[k][j] != 0 && (uint8_t)tab[k][j] == s[off + j]) j++;
    if (j == len && (j == (uint32_t)W || tab[k][j] == 0)) return k;
  }
  return -1;
}

// string body after the opening quote (the line holds no backslash / control byte /
// non-ASCII byte; a raw tab is invalid in a strict JSON string): position after the
// closing quote, or 0 on failure
__device__ __forceinline__ uint64_t skip_string(const uint8_t* s, uint64_t p, uint64_t e) {
  while (p < e) {
    const uint8_t c = s[p++];
    if (c == '"') return p;
    if (c == '\t') return 0;
  }
  return 0;
}

// JSON number at p: position after it (0 on failure); is_int / value / negative /
// fits as the reference's json.loads would type it (int unless fraction or exponent)
__device__ uint64_t scan_number(const uint8_t* s, uint64_t p, uint64_t e, bool& is_int, uint64_t& mag,
                                bool& neg, bool& fits) {
  neg = false; is_int = true; fits = true; mag = 0;
  if (p < e && s[p] == '-') { neg = true; p++; }
  if (p >= e) return 0;
  if (s[p] == '0') {
    p++;
  } else if (s[p] >= '1' && s[p] <= '9') {
    while (p < e && s[p] >= '0' && s[p] <= '9') {
      const uint64_t dgt = s[p] - '0';
      if (mag > (~0ull - dgt) / 10) fits = false;
      else mag = mag * 10 + dgt;
      p++;
    }
  } else {
    return 0;
  }
  if (p < e && s[p] == '.') {
    is_int = false; p++;
    if (p >= e || s[p] < '0' || s[p] > '9') return 0;
    while (p < e && s[p] >= '0' && s[p] <= '9') p++;
  }
  if (p < e && (s[p] == 'e' || s[p] == 'E')) {
    is_int = false; p++;
    if (p < e && (s[p] == '+' || s[p] == '-')) p++;
    if (p >= e || s[p] < '0' || s[p] > '9') return 0;
    while (p < e && s[p] >= '0' && s[p] <= '9') p++;
  }
  return p;
}

__device__ __forceinline__ uint64_t skip_literal(const uint8_t* s, uint64_t p, uint64_t e) {
  const char* lit = s[p] == 't' ? "true" : s[p] == 'f' ? "false" : s[p] == 'n' ? "null" : nullptr;
  if (!lit) return 0;
  for (int k = 0; lit[k]; k++, p++)
    if (p >= e || s[p] != (uint8_t)lit[k]) return 0;
  return p;
}

// Any JSON value (grammar-checked, nesting <= 64): position after it, 0 on failure.
__device__ uint64_t skip_value(const uint8_t* s, uint64_t p, uint64_t e) {
  uint64_t stack = 0;  // bit d: container at depth d is an object
  int depth = 0;
  bool neg, is_int, fits;
  uint64_t mag;
value:
  p = skip_ws(s, p, e);
  if (p >= e) return 0;
  switch (s[p]) {
    case '{':
      p = skip_ws(s, p + 1, e);
      if (p < e && s[p] == '}') { p++; goto after; }
      if (depth == 64) return 0;
      stack |= 1ull << depth; depth++;
      goto key;
    case '[':
      p = skip_ws(s, p + 1, e);
      if (p < e && s[p] == ']') { p++; goto after; }
      if (depth == 64) return 0;
      stack &= ~(1ull << depth); depth++;
      goto value;
    case '"':
      p = skip_string(s, p + 1, e);
      if (!p) return 0;
      goto after;
    case 't': case 'f': case 'n':
      p = skip_literal(s, p, e);
      if (!p) return 0;
      goto after;
    default:
      p = scan_number(s, p, e, is_int, mag, neg, fits);
      if (!p) return 0;
      goto after;
  }
key:
  p = skip_ws(s, p, e);
  if (p >= e || s[p] != '"') return 0;
  p = skip_string(s, p + 1, e);
  if (!p) return 0;
  p = skip_ws(s, p, e);
  if (p >= e || s[p] != ':') return 0;
  p++;
  goto value;
after:
  if (depth == 0) return p;
  p = skip_ws(s, p, e);
  if (p >= e) return 0;
  {
    const bool obj = (stack >> (depth - 1)) & 1;
    if (s[p] == ',') { p++; if (obj) goto key; goto value; }
    if (s[p] == (obj ? '}' : ']')) { p++; depth--; goto after; }
  }
  return 0;
}

// A value of a consulted key: scalar types recorded, anything else skipped as V_OTHER.
__device__ uint64_t read_value(const uint8_t* s, uint64_t p, uint64_t e, Val& v) {
  p = skip_ws(s, p, e);
  if (p >= e) return 0;
  const uint8_t c = s[p];
  if (c == '"') {
    const uint64_t q = skip_string(s, p + 1, e);
    if (!q) return 0;
    v.t = V_STR; v.off = (uint32_t)(p + 1); v.len = (uint32_t)(q - p - 2);
    return q;
  }
  if (c == '-' || (c >= '0' && c <= '9')) {
    bool neg, is_int, fits;
    uint64_t mag;
    const uint64_t q = scan_number(s, p, e, is_int, mag, neg, fits);
    if (!q) return 0;
    if (!is_int || !fits) v.t = V_OTHER;
    else if (!neg || mag == 0) { v.t = V_UINT; v.u = mag; }      // "-0" is the int 0
    else if (mag <= (1ull << 63)) { v.t = V_NINT; v.u = 0ull - mag; }
    else v.t = V_OTHER;
    return q;
  }
  v.t = V_OTHER;
  return skip_value(s, p, e);
}

// Endpoint object {"kind": <str>, "idx": <int>} (events.py:271-284); other members
// are grammar-checked and ignored; duplicate keys: last wins (json.loads).
__device__ uint64_t read_endpoint(const uint8_t* s, uint64_t p, uint64_t e, Val& v) {
  p = skip_ws(s, p, e);
  if (p >= e) return 0;
  if (s[p] != '{') { v.t = V_OTHER; return skip_value(s, p, e); }
  v.t = V_EP; v.ep_kind = -2; v.ep_idx = -2;  // -2: absent, -1: wrong type / value
  p = skip_ws(s, p + 1, e);
  if (p < e && s[p] == '}') return p + 1;
  while (true) {
    p = skip_ws(s, p, e);
    if (p >= e || s[p] != '"') return 0;
    const uint64_t k0 = p + 1;
    p = skip_string(s, k0, e);
    if (!p) return 0;
    const uint32_t klen = (uint32_t)(p - k0 - 1);
    p = skip_ws(s, p, e);
    if (p >= e || s[p] != ':') return 0;
    p++;
    const bool is_kind = klen == 4 && s[k0] == 'k' && s[k0 + 1] == 'i' && s[k0 + 2] == 'n' && s[k0 + 3] == 'd';
    const bool is_idx = klen == 3 && s[k0] == 'i' && s[k0 + 1] == 'd' && s[k0 + 2] == 'x';
    if (is_kind || is_idx) {
      Val w;
      w.t = V_NONE;
      p = read_value(s, p, e, w);
      if (!p) return 0;
      if (is_kind) v.ep_kind = w.t == V_STR ? match(s, w.off, w.len, kEpKinds) : -1;
      else v.ep_idx = w.t == V_UINT && w.u < (1ull << 62) ? (int64_t)w.u : -1;
    } else {
      p = skip_value(s, p, e);
      if (!p) return 0;
    }
    p = skip_ws(s, p, e);
    if (p >= e) return 0;
    if (s[p] == ',') { p++; continue; }
    if (s[p] == '}') return p + 1;
    return 0;
  }
}

struct LineOut {
  ct_record r;
  int64_t ts;
  uint64_t hash;
  uint32_t comm_off, comm_len;
};

// Parse line [b, e) of s; L_OK with `o` filled, L_BLANK, or L_DEFER.
__device__ uint8_t parse_line(const uint8_t* s, uint64_t b, uint64_t e, LineOut& o) {
  // blank per str.strip (the ASCII whitespace left inside a line: space, tab, \x1f);
  // anything the device does not decode itself defers the line
  bool blank = true, plain = true;
  for (uint64_t p = b; p < e; p++) {
    const uint8_t c = s[p];
    if (c != ' ' && c != '\t' && c != 0x1f) blank = false;
    if (c >= 0x80 || c == '\\' || (c < 0x20 && c != '\t')) plain = false;
  }
  if (blank) return L_BLANK;
  if (!plain) return L_DEFER;

  Val v[K_N];
#pragma unroll
  for (int k = 0; k < K_N; k++) v[k].t = V_NONE;
  uint64_t p = skip_ws(s, b, e);
  if (p >= e || s[p] != '{') return L_DEFER;
  p = skip_ws(s, p + 1, e);
  if (p < e && s[p] == '}') return L_DEFER;  // {}: "kind" missing
  while (true) {
    p = skip_ws(s, p, e);
    if (p >= e || s[p] != '"') return L_DEFER;
    const uint64_t k0 = p + 1;
    p = skip_string(s, k0, e);
    if (!p) return L_DEFER;
    const int key = match(s, (uint32_t)k0, (uint32_t)(p - k0 - 1), kKeyNames);
    p = skip_ws(s, p, e);
    if (p >= e || s[p] != ':') return L_DEFER;
    p++;
    if (key < 0) {
      p = skip_value(s, p, e);
    } else {
      v[key].t = V_NONE;
      p = (key == K_SRC || key == K_DST) ? read_endpoint(s, p, e, v[key]) : read_value(s, p, e, v[key]);
    }
    if (!p) return L_DEFER;
    p = skip_ws(s, p, e);
    if (p >= e) return L_DEFER;
    if (s[p] == ',') { p++; continue; }
    if (s[p] == '}') { p++; break; }
    return L_DEFER;
  }
  if (skip_ws(s, p, e) != e) return L_DEFER;  // "Extra data"

  // the reader's consulted keys and TraceEvent.validate, in effect (events.py:287-310)
  auto str_code = [&](int k, int which) -> int {
    if (v[k].t != V_STR) return -1;
    switch (which) {
      case 0: return match(s, v[k].off, v[k].len, kKinds);
      case 1: return match(s, v[k].off, v[k].len, kColls);
      case 2: return match(s, v[k].off, v[k].len, kAlgos);
      case 3: return match(s, v[k].off, v[k].len, kDtypes);
      default: return match(s, v[k].off, v[k].len, kCkinds);
    }
  };
  const int kind = str_code(K_KIND, 0);
  if (kind < 0) return L_DEFER;
  if (v[K_SEQ].t != V_UINT || v[K_COMM].t != V_STR || v[K_NRANKS].t != V_UINT || v[K_RANK].t != V_UINT ||
      v[K_DEV].t != V_UINT)
    return L_DEFER;
  if (v[K_TS].t == V_UINT) {
    if (v[K_TS].u >= (1ull << 63)) return L_DEFER;
  } else if (v[K_TS].t != V_NINT) {
    return L_DEFER;
  }
  const uint64_t n = v[K_NRANKS].u, rank = v[K_RANK].u, dev = v[K_DEV].u;
  if (n < 1 || n > 0xFFFF || rank >= n || dev > 0xFFFF) return L_DEFER;
  ct_record& r = o.r;
  r.seq = v[K_SEQ].u;
  r.comm = 0;
  r.nranks = (uint16_t)n;
  r.rank = (uint16_t)rank;
  r.dev = (uint16_t)dev;
  r.aux = 0;
  r.aux2 = 0;
  if (kind == CT_KIND_COLLECTIVE) {
    const int coll = str_code(K_COLL, 1), algo = str_code(K_ALGO, 2), dt = str_code(K_DTYPE, 3);
    if (coll < 0 || algo < 0 || dt < 0 || v[K_COUNT].t != V_UINT) return L_DEFER;
    const bool rooted = coll == CT_COLL_BROADCAST || coll == CT_COLL_REDUCE;
    if (v[K_ROOT].t != V_NONE || rooted) {
      if (v[K_ROOT].t != V_UINT) return L_DEFER;
      if (!rooted || v[K_ROOT].u >= n) return L_DEFER;  // root only for bcast/reduce, in [0, N)
      r.aux = (uint16_t)v[K_ROOT].u;
    }
    if ((algo == CT_ALGO_TREE || algo == CT_ALGO_COLLNET) && coll != CT_COLL_ALLREDUCE) return L_DEFER;
    r.count = v[K_COUNT].u;
    r.kc = (uint8_t)(kind | (coll << 3) | (rooted ? 1 << 6 : 0));
    r.ad = (uint8_t)(algo | (dt << 2));
  } else if (kind == CT_KIND_SEND || kind == CT_KIND_RECV) {
    const int dt = str_code(K_DTYPE, 3);
    if (v[K_PEER].t != V_UINT || v[K_COUNT].t != V_UINT || dt < 0) return L_DEFER;
    if (v[K_PEER].u == rank || v[K_PEER].u >= n) return L_DEFER;
    r.aux = (uint16_t)v[K_PEER].u;
    r.count = v[K_COUNT].u;
    r.kc = (uint8_t)kind;
    r.ad = (uint8_t)(dt << 2);
  } else {
    const int ck = str_code(K_CKIND, 4);
    if (ck < 0 || v[K_SRC].t != V_EP || v[K_DST].t != V_EP || v[K_BYTES].t != V_UINT) return L_DEFER;
    const Val &sv = v[K_SRC], &dv = v[K_DST];
    if (sv.ep_kind < 0 || sv.ep_idx < 0 || dv.ep_kind < 0 || dv.ep_idx < 0) return L_DEFER;
    const int want_s = ck == CT_CKIND_H2D ? 0 : 1, want_d = ck == CT_CKIND_D2H ? 0 : 1;  // host 0, gpu 1
    if (sv.ep_kind != want_s || dv.ep_kind != want_d) return L_DEFER;
    if ((want_s == 0 && sv.ep_idx != 0) || (want_d == 0 && dv.ep_idx != 0)) return L_DEFER;
    if (sv.ep_idx > 0xFFFF || dv.ep_idx > 0xFFFF) return L_DEFER;
    if (ck == CT_CKIND_D2D && sv.ep_idx == dv.ep_idx) return L_DEFER;
    r.aux = (uint16_t)sv.ep_idx;
    r.aux2 = (uint16_t)dv.ep_idx;
    r.count = v[K_BYTES].u;
    r.kc = (uint8_t)kind;
    r.ad = (uint8_t)(ck << 6);
  }
  o.ts = (int64_t)v[K_TS].u;
  o.comm_off = v[K_COMM].off;
  o.comm_len = v[K_COMM].len;
  uint64_t h = 0xcbf29ce484222325ull;  // FNV-1a over the name bytes
  for (uint32_t j = 0; j < o.comm_len; j++) h = (h ^ s[o.comm_off + j]) * 0x100000001b3ull;
  o.hash = h == kNoKey ? kNoKey - 1 : h;
  return L_OK;
}

__global__ void k_parse(const uint8_t* s, uint64_t size, const uint64_t* brk, uint64_t nb, uint64_t n_lines,
                        uint8_t* status, LineOut* out) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < n_lines;
       k += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t b = k == 0 ? 0 : brk[k - 1] + break_len(s, size, brk[k - 1]);
    const uint64_t e = k < nb ? brk[k] : size;
    LineOut o;
    const uint8_t st = parse_line(s, b, e, o);
    status[k] = st;
    if (st == L_OK) out[k] = o;
  }
}

struct NonBlank {
  const uint8_t* st;
  __device__ __forceinline__ uint64_t operator()(uint64_t k) const { return st[k] != L_BLANK ? 1u : 0u; }
};
struct IsDeferred {
  const uint8_t* st;
  __device__ __forceinline__ bool operator()(uint64_t k) const { return st[k] == L_DEFER; }
};

// line k -> record slot ridx[k]: record, ts, comm (key, slot) pair
__global__ void k_scatter(uint64_t n_lines, const uint8_t* status, const LineOut* lo, const uint64_t* ridx,
                          ct_record* recs, int64_t* ts, uint64_t* keys, uint64_t* vals, uint64_t* coff) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < n_lines;
       k += (uint64_t)gridDim.x * blockDim.x) {
    const uint8_t st = status[k];
    if (st == L_BLANK) continue;
    const uint64_t i = ridx[k];
    vals[i] = i;
    if (st == L_OK) {
      recs[i] = lo[k].r;
      ts[i] = lo[k].ts;
      keys[i] = lo[k].hash;
      coff[i] = ((uint64_t)lo[k].comm_len << 40) | lo[k].comm_off;
    } else {
      recs[i] = ct_record{};
      ts[i] = 0;
      keys[i] = kNoKey;
      coff[i] = 0;
    }
  }
}

struct SegHead {
  const uint64_t* k;
  __device__ __forceinline__ uint32_t operator()(uint64_t i) const {
    return k[i] != kNoKey && (i == 0 || k[i] != k[i - 1]) ? 1u : 0u;
  }
};

// sorted position i: segment id seg[i] - 1 (inclusive scan of heads); heads record
// their position and first record slot; every member's name is compared byte-for-byte
// with its head's (a 64-bit key collision fails the load loudly)
__global__ void k_heads(uint64_t m, const uint64_t* keys, const uint64_t* vals, const uint32_t* seg,
                        uint64_t* seg_first, uint64_t* seg_coff, const uint64_t* coff) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
    if (keys[i] == kNoKey) continue;
    if (i == 0 || keys[i] != keys[i - 1]) {
      seg_first[seg[i] - 1] = vals[i];
      seg_coff[seg[i] - 1] = coff[vals[i]];
    }
  }
}

__global__ void k_iota(uint64_t n, uint64_t* out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = i;
}

__global__ void k_verify(uint64_t m, const uint64_t* keys, const uint64_t* vals, const uint32_t* seg,
                         const uint64_t* seg_coff, const uint64_t* coff, const uint8_t* s, unsigned int* collide) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
    if (keys[i] == kNoKey) continue;
    const uint64_t a = coff[vals[i]], h = seg_coff[seg[i] - 1];
    if (a == h) continue;
    const uint32_t la = (uint32_t)(a >> 40), lh = (uint32_t)(h >> 40);
    bool same = la == lh;
    const uint64_t oa = a & ((1ull << 40) - 1), oh = h & ((1ull << 40) - 1);
    for (uint32_t j = 0; same && j < la; j++) same = s[oa + j] == s[oh + j];
    if (!same) atomicOr(collide, 1u);
  }
}

// ranked segments: comm id of segment seg_order[r] is r; names gathered contiguously
__global__ void k_rank(uint64_t u, const uint64_t* seg_order, uint32_t* seg_id) {
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < u; r += (uint64_t)gridDim.x * blockDim.x)
    seg_id[seg_order[r]] = (uint32_t)r;
}

__global__ void k_assign(uint64_t m, const uint64_t* keys, const uint64_t* vals, const uint32_t* seg,
                         const uint32_t* seg_id, ct_record* recs) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x)
    if (keys[i] != kNoKey) recs[vals[i]].comm = seg_id[seg[i] - 1];
}

struct NameLen {
  const uint64_t* seg_coff;
  const uint64_t* seg_order;
  __device__ __forceinline__ uint64_t operator()(uint64_t r) const { return seg_coff[seg_order[r]] >> 40; }
};

__global__ void k_names(uint64_t u, const uint64_t* seg_order, const uint64_t* seg_first, const uint64_t* seg_coff,
                        const uint64_t* name_off, const uint8_t* s, uint8_t* names, uint64_t* rows) {
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < u; r += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t g = seg_order[r], c = seg_coff[g];
    const uint64_t len = c >> 40, off = c & ((1ull << 40) - 1);
    for (uint64_t j = 0; j < len; j++) names[name_off[r] + j] = s[off + j];
    rows[3 * r] = seg_first[g];
    rows[3 * r + 1] = name_off[r];
    rows[3 * r + 2] = len;
  }
}

__global__ void k_deferred_rows(uint64_t nd, const uint64_t* lines, const uint64_t* ridx, const uint8_t* s,
                                uint64_t size, const uint64_t* brk, uint64_t nb, uint64_t* rows) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < nd; j += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t k = lines[j];
    const uint64_t b = k == 0 ? 0 : brk[k - 1] + break_len(s, size, brk[k - 1]);
    const uint64_t e = k < nb ? brk[k] : size;
    rows[4 * j] = k + 1;  // 1-based line number
    rows[4 * j + 1] = ridx[k];
    rows[4 * j + 2] = b;
    rows[4 * j + 3] = e - b;
  }
}

__global__ void k_nonascii(const uint8_t* s, uint64_t n, unsigned int* flag) {
  bool any = false;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    any |= s[i] >= 0x80;
  if (__any_sync(0xffffffffu, any) && (threadIdx.x & 31) == 0) atomicOr(flag, 1u);
}

}  // namespace

// ---------------------------------------------------------------- handle + C ABI

struct ct_jsonl {
  int device = 0;
  cudaStream_t st = nullptr;
  std::string err;
  ct_jsonl_info info{};
  ct_record* recs = nullptr;
  int64_t* ts = nullptr;
  uint64_t* deferred_rows = nullptr;  // device, 4 per deferred line
  uint64_t* comm_rows = nullptr;      // device, 3 per comm
  uint8_t* names = nullptr;
  std::vector<void*> owned;
};

namespace {

struct Pool {
  ct_jsonl* j;
  template <class T>
  T* alloc(uint64_t n) {
    void* p = nullptr;
    if (cudaMallocAsync(&p, (n ? n : 1) * sizeof(T), j->st) != cudaSuccess) return nullptr;
    j->owned.push_back(p);
    return static_cast<T*>(p);
  }
  void* temp(size_t bytes) { return alloc<uint8_t>(bytes); }
};

#define JL_TRY(x)                                                                    \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess) {                                                         \
      j->err = std::string(#x) + ": " + cudaGetErrorString(e_);                      \
      return CT_ERR_CUDA;                                                            \
    }                                                                                \
  } while (0)
#define JL_NN(p)                                                                     \
  do {                                                                               \
    if (!(p)) { j->err = "device allocation failed"; return CT_ERR_CUDA; }           \
  } while (0)

int grid_for(uint64_t n, int threads = 256) {
  const uint64_t g = (n + threads - 1) / threads;
  return (int)(g < 1 ? 1 : g > 148 * 32 ? 148 * 32 : g);
}

int run(ct_jsonl* j, const uint8_t* text, uint64_t size, int on_device) {
  Pool pool{j};
  cudaEvent_t e0, e1;
  JL_TRY(cudaEventCreate(&e0));
  JL_TRY(cudaEventCreate(&e1));
  const uint8_t* s = text;
  if (!on_device) {
    uint8_t* d = pool.alloc<uint8_t>(size + 1);
    JL_NN(d);
    JL_TRY(cudaMemcpyAsync(d, text, size, cudaMemcpyHostToDevice, j->st));
    s = d;
  }
  JL_TRY(cudaEventRecord(e0, j->st));
  uint64_t* scal = pool.alloc<uint64_t>(8);  // device scalars
  JL_NN(scal);
  JL_TRY(cudaMemsetAsync(scal, 0, 8 * sizeof(uint64_t), j->st));
  unsigned int* flags = reinterpret_cast<unsigned int*>(scal + 6);

  // 1. terminators
  thrust::counting_iterator<uint64_t> idx(0);
  BreakPred bp{s, size};
  auto cnt_it = thrust::make_transform_iterator(idx, BreakCount{bp});
  size_t tb = 0;
  JL_TRY(cub::DeviceReduce::Sum(nullptr, tb, cnt_it, scal, (int64_t)size, j->st));
  void* t = pool.temp(tb);
  JL_NN(t);
  JL_TRY(cub::DeviceReduce::Sum(t, tb, cnt_it, scal, (int64_t)size, j->st));
  uint64_t nb = 0;
  JL_TRY(cudaMemcpyAsync(&nb, scal, sizeof(uint64_t), cudaMemcpyDeviceToHost, j->st));
  JL_TRY(cudaStreamSynchronize(j->st));
  uint64_t* brk = pool.alloc<uint64_t>(nb);
  JL_NN(brk);
  if (nb) {
    tb = 0;
    JL_TRY(cub::DeviceSelect::If(nullptr, tb, idx, brk, scal + 1, (int64_t)size, bp, j->st));
    t = pool.temp(tb);
    JL_NN(t);
    JL_TRY(cub::DeviceSelect::If(t, tb, idx, brk, scal + 1, (int64_t)size, bp, j->st));
  }
  uint64_t last_end = 0;  // first byte after the last terminator
  if (nb) {
    uint64_t lb = 0;
    uint8_t tailb[3] = {0, 0, 0};
    JL_TRY(cudaMemcpyAsync(&lb, brk + nb - 1, sizeof(uint64_t), cudaMemcpyDeviceToHost, j->st));
    JL_TRY(cudaStreamSynchronize(j->st));
    JL_TRY(cudaMemcpyAsync(tailb, s + lb, size - lb < 3 ? size - lb : 3, cudaMemcpyDeviceToHost, j->st));
    JL_TRY(cudaStreamSynchronize(j->st));
    uint64_t bl = 1;
    if (tailb[0] == '\r') bl = size - lb >= 2 && tailb[1] == '\n' ? 2 : 1;
    else if (tailb[0] == 0xC2) bl = 2;
    else if (tailb[0] == 0xE2) bl = 3;
    last_end = lb + bl;
  }
  const uint64_t n_lines = nb + (last_end < size ? 1 : 0);
  j->info.n_lines = n_lines;
  k_nonascii<<<grid_for(size), 256, 0, j->st>>>(s, size, flags + 1);

  // 2. parse, one thread per line
  uint8_t* status = pool.alloc<uint8_t>(n_lines + 1);  // + a blank terminator for the scan
  LineOut* lo = pool.alloc<LineOut>(n_lines);
  uint64_t* ridx = pool.alloc<uint64_t>(n_lines + 1);
  JL_NN(status); JL_NN(lo); JL_NN(ridx);
  JL_TRY(cudaMemsetAsync(status + n_lines, L_BLANK, 1, j->st));
  if (n_lines) k_parse<<<grid_for(n_lines, 128), 128, 0, j->st>>>(s, size, brk, nb, n_lines, status, lo);
  JL_TRY(cudaGetLastError());
  auto nb_it = thrust::make_transform_iterator(idx, NonBlank{status});
  tb = 0;
  JL_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tb, nb_it, ridx, (int64_t)n_lines + 1, j->st));
  t = pool.temp(tb);
  JL_NN(t);
  JL_TRY(cub::DeviceScan::ExclusiveSum(t, tb, nb_it, ridx, (int64_t)n_lines + 1, j->st));
  uint64_t n_rec = 0;
  JL_TRY(cudaMemcpyAsync(&n_rec, ridx + n_lines, sizeof(uint64_t), cudaMemcpyDeviceToHost, j->st));
  JL_TRY(cudaStreamSynchronize(j->st));
  j->info.n_records = n_rec;
  if (n_rec >= (1ull << 32)) { j->err = "more than 2^32 - 1 records in one text"; return CT_ERR_CAPACITY; }

  // deferred lines
  uint64_t* dlines = pool.alloc<uint64_t>(n_lines);
  JL_NN(dlines);
  if (n_lines) {
    tb = 0;
    IsDeferred isd{status};
    JL_TRY(cub::DeviceSelect::If(nullptr, tb, idx, dlines, scal + 2, (int64_t)n_lines, isd, j->st));
    t = pool.temp(tb);
    JL_NN(t);
    JL_TRY(cub::DeviceSelect::If(t, tb, idx, dlines, scal + 2, (int64_t)n_lines, isd, j->st));
  }
  uint64_t nd = 0;
  JL_TRY(cudaMemcpyAsync(&nd, scal + 2, sizeof(uint64_t), cudaMemcpyDeviceToHost, j->st));
  JL_TRY(cudaStreamSynchronize(j->st));
  j->info.n_deferred = nd;
  j->deferred_rows = pool.alloc<uint64_t>(4 * nd);
  JL_NN(j->deferred_rows);
  if (nd) k_deferred_rows<<<grid_for(nd), 256, 0, j->st>>>(nd, dlines, ridx, s, size, brk, nb, j->deferred_rows);

  // records + comm keys
  j->recs = pool.alloc<ct_record>(n_rec);
  j->ts = pool.alloc<int64_t>(n_rec);
  uint64_t* keys = pool.alloc<uint64_t>(n_rec);
  uint64_t* vals = pool.alloc<uint64_t>(n_rec);
  uint64_t* coff = pool.alloc<uint64_t>(n_rec);
  uint64_t* keys2 = pool.alloc<uint64_t>(n_rec);
  uint64_t* vals2 = pool.alloc<uint64_t>(n_rec);
  JL_NN(j->recs); JL_NN(j->ts); JL_NN(keys); JL_NN(vals); JL_NN(coff); JL_NN(keys2); JL_NN(vals2);
  if (n_lines) k_scatter<<<grid_for(n_lines), 256, 0, j->st>>>(n_lines, status, lo, ridx, j->recs, j->ts, keys, vals, coff);
  JL_TRY(cudaGetLastError());

  // 3. comm interning in first-seen order
  uint64_t u = 0;
  uint32_t* seg = pool.alloc<uint32_t>(n_rec);
  JL_NN(seg);
  if (n_rec) {
    tb = 0;
    JL_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, keys2, vals, vals2, (int64_t)n_rec, 0, 64, j->st));
    t = pool.temp(tb);
    JL_NN(t);
    JL_TRY(cub::DeviceRadixSort::SortPairs(t, tb, keys, keys2, vals, vals2, (int64_t)n_rec, 0, 64, j->st));
    auto head_it = thrust::make_transform_iterator(idx, SegHead{keys2});
    tb = 0;
    JL_TRY(cub::DeviceScan::InclusiveSum(nullptr, tb, head_it, seg, (int64_t)n_rec, j->st));
    t = pool.temp(tb);
    JL_NN(t);
    JL_TRY(cub::DeviceScan::InclusiveSum(t, tb, head_it, seg, (int64_t)n_rec, j->st));
    uint32_t u32 = 0;
    JL_TRY(cudaMemcpyAsync(&u32, seg + n_rec - 1, sizeof(uint32_t), cudaMemcpyDeviceToHost, j->st));
    JL_TRY(cudaStreamSynchronize(j->st));
    u = u32;
  }
  j->info.n_comms = u;
  uint64_t* seg_first = pool.alloc<uint64_t>(u);
  uint64_t* seg_coff = pool.alloc<uint64_t>(u);
  uint64_t* seg_ids = pool.alloc<uint64_t>(u);
  uint64_t* first_sorted = pool.alloc<uint64_t>(u);
  uint64_t* seg_order = pool.alloc<uint64_t>(u);
  uint32_t* seg_id = pool.alloc<uint32_t>(u);
  uint64_t* name_off = pool.alloc<uint64_t>(u + 1);
  j->comm_rows = pool.alloc<uint64_t>(3 * u);
  JL_NN(seg_first); JL_NN(seg_coff); JL_NN(seg_ids); JL_NN(first_sorted); JL_NN(seg_order); JL_NN(seg_id);
  JL_NN(name_off); JL_NN(j->comm_rows);
  uint64_t name_bytes = 0;
  if (u) {
    const int g = grid_for(n_rec);
    k_heads<<<g, 256, 0, j->st>>>(n_rec, keys2, vals2, seg, seg_first, seg_coff, coff);
    k_verify<<<g, 256, 0, j->st>>>(n_rec, keys2, vals2, seg, seg_coff, coff, s, flags);
    JL_TRY(cudaGetLastError());
    k_iota<<<grid_for(u), 256, 0, j->st>>>(u, seg_ids);
    tb = 0;
    JL_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tb, seg_first, first_sorted, seg_ids, seg_order, (int64_t)u, 0, 64, j->st));
    t = pool.temp(tb);
    JL_NN(t);
    JL_TRY(cub::DeviceRadixSort::SortPairs(t, tb, seg_first, first_sorted, seg_ids, seg_order, (int64_t)u, 0, 64, j->st));
    k_rank<<<grid_for(u), 256, 0, j->st>>>(u, seg_order, seg_id);
    k_assign<<<g, 256, 0, j->st>>>(n_rec, keys2, vals2, seg, seg_id, j->recs);
    auto len_it = thrust::make_transform_iterator(idx, NameLen{seg_coff, seg_order});
    tb = 0;
    JL_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tb, len_it, name_off, (int64_t)u, j->st));
    t = pool.temp(tb);
    JL_NN(t);
    JL_TRY(cub::DeviceScan::ExclusiveSum(t, tb, len_it, name_off, (int64_t)u, j->st));
    uint64_t lastoff = 0, lastc = 0, lastg = 0;
    JL_TRY(cudaMemcpyAsync(&lastoff, name_off + u - 1, sizeof(uint64_t), cudaMemcpyDeviceToHost, j->st));
    JL_TRY(cudaMemcpyAsync(&lastg, seg_order + u - 1, sizeof(uint64_t), cudaMemcpyDeviceToHost, j->st));
    JL_TRY(cudaStreamSynchronize(j->st));
    JL_TRY(cudaMemcpyAsync(&lastc, seg_coff + lastg, sizeof(uint64_t), cudaMemcpyDeviceToHost, j->st));
    JL_TRY(cudaStreamSynchronize(j->st));
    name_bytes = lastoff + (lastc >> 40);
    j->names = pool.alloc<uint8_t>(name_bytes);
    JL_NN(j->names);
    k_names<<<grid_for(u), 256, 0, j->st>>>(u, seg_order, seg_first, seg_coff, name_off, s, j->names, j->comm_rows);
    JL_TRY(cudaGetLastError());
  }
  j->info.comm_bytes = name_bytes;
  JL_TRY(cudaEventRecord(e1, j->st));
  unsigned int hflags[2] = {0, 0};
  JL_TRY(cudaMemcpyAsync(hflags, flags, sizeof(hflags), cudaMemcpyDeviceToHost, j->st));
  JL_TRY(cudaStreamSynchronize(j->st));
  float ms = 0;
  JL_TRY(cudaEventElapsedTime(&ms, e0, e1));
  j->info.ms_device = ms;
  j->info.non_ascii = hflags[1] ? 1 : 0;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (hflags[0]) {
    j->err = "comm name hash collision (64-bit FNV-1a): two different names share a key";
    return CT_ERR_CAPACITY;
  }
  return CT_OK;
}

}  // namespace

extern "C" {

int ct_jsonl_parse(int device, const char* text, uint64_t size, int on_device, ct_jsonl** out,
                   ct_jsonl_info* info) {
  if (!out) return CT_ERR_ARGUMENT;
  ct_jsonl* j = new ct_jsonl();
  *out = j;
  j->device = device;
  if (!text && size) { j->err = "null text"; return CT_ERR_ARGUMENT; }
  if (size >= (1ull << 40)) { j->err = "text larger than 2^40 bytes"; return CT_ERR_ARGUMENT; }
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&j->st, cudaStreamNonBlocking);
  if (e != cudaSuccess) { j->err = cudaGetErrorString(e); return CT_ERR_CUDA; }
  const int rc = run(j, reinterpret_cast<const uint8_t*>(text), size, on_device);
  if (info) *info = j->info;
  return rc;
}

int ct_jsonl_records(ct_jsonl* j, ct_record* dev_out, int64_t* host_ts) {
  if (!j) return CT_ERR_ARGUMENT;
  const uint64_t n = j->info.n_records;
  cudaError_t e = cudaSuccess;
  if (n && dev_out) e = cudaMemcpyAsync(dev_out, j->recs, n * sizeof(ct_record), cudaMemcpyDeviceToDevice, j->st);
  if (e == cudaSuccess && n && host_ts)
    e = cudaMemcpyAsync(host_ts, j->ts, n * sizeof(int64_t), cudaMemcpyDeviceToHost, j->st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(j->st);
  if (e != cudaSuccess) { j->err = cudaGetErrorString(e); return CT_ERR_CUDA; }
  return CT_OK;
}

int ct_jsonl_deferred(ct_jsonl* j, uint64_t* rows) {
  if (!j) return CT_ERR_ARGUMENT;
  const uint64_t n = j->info.n_deferred;
  cudaError_t e = cudaSuccess;
  if (n) e = cudaMemcpyAsync(rows, j->deferred_rows, 4 * n * sizeof(uint64_t), cudaMemcpyDeviceToHost, j->st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(j->st);
  if (e != cudaSuccess) { j->err = cudaGetErrorString(e); return CT_ERR_CUDA; }
  return CT_OK;
}

int ct_jsonl_comms(ct_jsonl* j, uint64_t* rows, char* names) {
  if (!j) return CT_ERR_ARGUMENT;
  const uint64_t u = j->info.n_comms;
  cudaError_t e = cudaSuccess;
  if (u) e = cudaMemcpyAsync(rows, j->comm_rows, 3 * u * sizeof(uint64_t), cudaMemcpyDeviceToHost, j->st);
  if (e == cudaSuccess && j->info.comm_bytes)
    e = cudaMemcpyAsync(names, j->names, j->info.comm_bytes, cudaMemcpyDeviceToHost, j->st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(j->st);
  if (e != cudaSuccess) { j->err = cudaGetErrorString(e); return CT_ERR_CUDA; }
  return CT_OK;
}

const char* ct_jsonl_error(const ct_jsonl* j) { return j ? j->err.c_str() : "null handle"; }

void ct_jsonl_free(ct_jsonl* j) {
  if (!j) return;
  if (j->st) {
    for (void* p : j->owned) cudaFreeAsync(p, j->st);
    cudaStreamSynchronize(j->st);
    cudaStreamDestroy(j->st);
  }
  delete j;
}

}  // extern "C"
