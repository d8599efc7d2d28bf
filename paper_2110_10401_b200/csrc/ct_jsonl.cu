// Device JSONL loader: reference wire text -> packed ct_record stream.
//
// Replaces the bulk of parse_trace (reference events.py:352-384, field readers
// events.py:294-349, validate events.py:166-236) followed by the record packing of
// packed.pack_events.  Three phases, all on the device:
//   1. line breaks: every byte position that starts a str.splitlines() terminator
//      (\n, \r, \r\n, \v, \f, \x1c-\x1e, U+0085, U+2028, U+2029) -> ordered list;
//      16 bytes per thread, per-tile counts, a scan, then in-order writes
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

#include <omp.h>

#include <algorithm>
#include <array>
#include <mutex>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/commtrace_b200.h"

namespace {

constexpr uint64_t kNoKey = ~0ull;  // sort key of records without a device comm name

// L_ESC: the line holds backslash escapes; the main parse leaves it to k_parse_esc (the
// same parser with escape decoding compiled in), so the common path carries no escape code
enum : uint8_t { L_BLANK = 0, L_OK = 1, L_DEFER = 2, L_ESC = 3 };

// ---------------------------------------------------------------- phase 1: breaks

// 16 bytes at i0 (i0 % 16 == 0): bit j set iff a terminator starts at i0 + j; non-ASCII
// bytes noted.  Neighbour bytes outside the 16 are read only for the rare cases.
constexpr int kTileThreads = 256;
constexpr int kTileReps = 1;  // 16-byte chunks per thread (4 measured slower)
constexpr uint64_t kChunkRow = kTileThreads * 16;
constexpr uint64_t kTileBytes = kChunkRow * kTileReps;

__device__ __forceinline__ uint4 load16(const uint8_t* s, uint64_t n, uint64_t i0, bool aligned) {
  if (aligned && i0 + 16 <= n) return *reinterpret_cast<const uint4*>(s + i0);
  return make_uint4(0, 0, 0, 0);  // handled bytewise in break_mask16
}

// 16 bytes at i0 (i0 % 16 == 0, pre-loaded in v when aligned and in range): bit j set
// iff a terminator starts at i0 + j; non-ASCII bytes noted.  Neighbour bytes outside
// the 16 are read only for the rare cases.
__device__ __forceinline__ uint32_t break_mask16(const uint8_t* s, uint64_t n, uint64_t i0, bool aligned,
                                                 const uint4 v, bool& non_ascii) {
  non_ascii = false;
  if (i0 >= n) return 0;
  uint8_t b[16];
  if (aligned && i0 + 16 <= n) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    // candidates are bytes < 0x20 or >= 0x80 (a superset: borrow artefacts above a true
    // candidate are re-checked): most 16-byte chunks have none, a line end has one
    uint32_t cand = 0;
#pragma unroll
    for (int q = 0; q < 4; q++) {
      const uint32_t t = (((w[q] - 0x20202020u) & ~w[q]) | w[q]) & 0x80808080u;
      cand |= (((t >> 7) & 1u) | ((t >> 14) & 2u) | ((t >> 21) & 4u) | ((t >> 28) & 8u)) << (4 * q);
    }
    if (!cand) return 0;
    uint32_t m = 0;
    bool hi = false;
    while (cand) {
      const int j = __ffs(cand) - 1;
      cand &= cand - 1;
      const uint32_t c = (w[j >> 2] >> (8 * (j & 3))) & 0xFF;
      auto at = [&](int k) -> uint32_t {  // byte k of the chunk, or of the text beyond it
        return k < 16 ? (w[k >> 2] >> (8 * (k & 3))) & 0xFF : (i0 + k < n ? s[i0 + k] : 0u);
      };
      const uint64_t i = i0 + j;
      hi |= c >= 0x80;
      bool brk;
      if (c == '\n') brk = j > 0 ? at(j - 1) != '\r' : (i == 0 || s[i - 1] != '\r');
      else if (c == '\r' || c == 0x0b || c == 0x0c || c == 0x1c || c == 0x1d || c == 0x1e) brk = true;
      else if (c == 0xC2) brk = at(j + 1) == 0x85;
      else if (c == 0xE2) brk = at(j + 1) == 0x80 && (at(j + 2) == 0xA8 || at(j + 2) == 0xA9);
      else brk = false;
      if (brk) m |= 1u << j;
    }
    non_ascii = hi;
    return m;
  } else {
#pragma unroll
    for (int j = 0; j < 16; j++) b[j] = i0 + j < n ? s[i0 + j] : (uint8_t)'x';
  }
  uint32_t m = 0;
  bool hi = false;
#pragma unroll
  for (int j = 0; j < 16; j++) {
    const uint8_t c = b[j];
    hi |= c >= 0x80;
    if (c < 0x20 || c >= 0xC2) {  // candidates only
      const uint64_t i = i0 + j;
      if (i >= n) continue;
      bool brk;
      if (c == '\n') brk = j > 0 ? b[j - 1] != '\r' : (i == 0 || s[i - 1] != '\r');
      else if (c == '\r' || c == 0x0b || c == 0x0c || c == 0x1c || c == 0x1d || c == 0x1e) brk = true;
      else if (c == 0xC2) brk = i + 1 < n && (j + 1 < 16 ? b[j + 1] : s[i + 1]) == 0x85;
      else if (c == 0xE2) brk = i + 2 < n && (j + 1 < 16 ? b[j + 1] : s[i + 1]) == 0x80 &&
                                ((j + 2 < 16 ? b[j + 2] : s[i + 2]) == 0xA8 || (j + 2 < 16 ? b[j + 2] : s[i + 2]) == 0xA9);
      else brk = false;
      if (brk) m |= 1u << j;
    }
  }
  non_ascii = hi;
  return m;
}

__global__ void __launch_bounds__(kTileThreads) k_brk_count(const uint8_t* s, uint64_t n, bool aligned,
                                                            uint32_t* tile_cnt, unsigned int* flags) {
  using BR = cub::BlockReduce<uint32_t, kTileThreads>;
  __shared__ typename BR::TempStorage tmp;
  const uint64_t base = blockIdx.x * kTileBytes + threadIdx.x * 16ull;
  uint4 v[kTileReps];
#pragma unroll
  for (int r = 0; r < kTileReps; r++) v[r] = load16(s, n, base + r * kChunkRow, aligned);
  uint32_t c = 0;
  bool hi = false;
#pragma unroll
  for (int r = 0; r < kTileReps; r++) {
    bool h;
    c += __popc(break_mask16(s, n, base + r * kChunkRow, aligned, v[r], h));
    hi |= h;
  }
  if (__any_sync(0xffffffffu, hi) && (threadIdx.x & 31) == 0) atomicOr(flags + 1, 1u);
  const uint32_t tot = BR(tmp).Sum(c);
  if (threadIdx.x == 0) tile_cnt[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kTileThreads) k_brk_write(const uint8_t* s, uint64_t n, bool aligned,
                                                            const uint64_t* tile_off, uint64_t* brk) {
  using BS = cub::BlockScan<uint32_t, kTileThreads>;
  __shared__ typename BS::TempStorage tmp;
  const uint64_t base = blockIdx.x * kTileBytes + threadIdx.x * 16ull;
  uint4 v[kTileReps];
#pragma unroll
  for (int r = 0; r < kTileReps; r++) v[r] = load16(s, n, base + r * kChunkRow, aligned);
  uint64_t o0 = tile_off[blockIdx.x];
#pragma unroll
  for (int r = 0; r < kTileReps; r++) {  // rows of chunks in text order
    bool h;
    uint32_t m = break_mask16(s, n, base + r * kChunkRow, aligned, v[r], h);
    uint32_t before, total;
    BS(tmp).ExclusiveSum((uint32_t)__popc(m), before, total);
    __syncthreads();
    uint64_t o = o0 + before;
    while (m) {
      const int j = __ffs(m) - 1;
      m &= m - 1;
      brk[o++] = base + r * kChunkRow + j;
    }
    o0 += total;
  }
}

__device__ __forceinline__ uint64_t break_len(const uint8_t* s, uint64_t n, uint64_t i) {
  const uint8_t b = s[i];
  if (b == '\r') return i + 1 < n && s[i + 1] == '\n' ? 2 : 1;
  if (b == 0xC2) return 2;
  if (b == 0xE2) return 3;
  return 1;
}

// ---------------------------------------------------------------- phase 2: parse

// Strings are compared as (length, first 16 bytes packed little-endian): every name the
// reader knows is <= 13 bytes, so two 64-bit compares against immediates decide it.
constexpr uint64_t pk8(const char* str, int off) {
  uint64_t v = 0;
  int n = 0;
  while (str[n]) n++;
  for (int i = 0; i < 8 && off + i < n; i++) v |= (uint64_t)(uint8_t)str[off + i] << (8 * i);
  return v;
}
constexpr uint32_t slen(const char* str) { return str[0] ? 1 + slen(str + 1) : 0; }

struct Str {
  uint32_t len;
  uint64_t w0, w1;
  bool esc = false;  // the JSON text held escapes (len / w0 / w1 are the decoded string's)
};

// Comm names are referenced as (offset | length << 40); names decoded from escapes live
// in a side buffer, marked by kSideBit in the offset (texts are < 2^39 bytes).
constexpr uint64_t kSideBit = 1ull << 39;
constexpr uint64_t kOffMask = (1ull << 40) - 1;
constexpr uint32_t kMaxEscName = 256;  // longest escaped comm name decoded on the device

__device__ __forceinline__ const uint8_t* name_ptr(const uint8_t* s, const uint8_t* side, uint64_t c) {
  const uint64_t off = c & kOffMask;
  return (off & kSideBit) ? side + (off & (kSideBit - 1)) : s + off;
}

struct Side {  // decoded comm names (escapes): bump-allocated, a full buffer defers the line
  uint8_t* buf;
  unsigned long long* used;
  uint64_t cap;
};

__device__ __forceinline__ int hexv(uint8_t c) {
  return c >= '0' && c <= '9' ? c - '0' : (c | 0x20) >= 'a' && (c | 0x20) <= 'f' ? (c | 0x20) - 'a' + 10 : -1;
}

// String body after the opening quote, WITH escapes (json.loads, strict): the decoded
// string's first 16 bytes / length in ``out`` and, when ``buf`` is given, its UTF-8
// bytes (up to ``cap``; lone surrogates encoded like Python's "surrogatepass").
// Position after the closing quote, 0 on failure (invalid escape, raw control byte).
struct EscOut {
  uint64_t pos, w0, w1;
  uint32_t len;
};

__device__ __noinline__ EscOut scan_str_esc_impl(const uint8_t* s, uint64_t p, uint64_t e, uint8_t* buf,
                                                 uint32_t cap) {
  EscOut r{0, 0, 0, 0};
  uint32_t n = 0;
  uint64_t w0 = 0, w1 = 0;
  auto put = [&](uint32_t b) {
    if (n < 8) w0 |= (uint64_t)b << (8 * n);
    else if (n < 16) w1 |= (uint64_t)b << (8 * (n - 8));
    if (buf && n < cap) buf[n] = (uint8_t)b;
    n++;
  };
  auto hex4 = [&](uint64_t q) -> int {
    if (q + 4 > e) return -1;
    int v = 0;
    for (int k = 0; k < 4; k++) {
      const int h = hexv(s[q + k]);
      if (h < 0) return -1;
      v = v * 16 + h;
    }
    return v;
  };
  while (p < e) {
    const uint8_t c = s[p];
    if (c == '"') {
      r.pos = p + 1;
      r.w0 = w0;
      r.w1 = w1;
      r.len = n;
      return r;
    }
    if (c < 0x20) return r;  // raw control characters are invalid in strict JSON strings
    if (c != '\\') { put(c); p++; continue; }
    if (p + 1 >= e) return r;
    const uint8_t x = s[p + 1];
    p += 2;
    switch (x) {
      case '"': put('"'); break;
      case '\\': put('\\'); break;
      case '/': put('/'); break;
      case 'b': put(8); break;
      case 'f': put(12); break;
      case 'n': put(10); break;
      case 'r': put(13); break;
      case 't': put(9); break;
      case 'u': {
        int cp = hex4(p);
        if (cp < 0) return r;
        p += 4;
        if (cp >= 0xD800 && cp <= 0xDBFF && p + 6 <= e && s[p] == '\\' && s[p + 1] == 'u') {
          const int lo = hex4(p + 2);
          if (lo >= 0xDC00 && lo <= 0xDFFF) {  // a surrogate pair is one code point
            cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
            p += 6;
          }
        }
        if (cp < 0x80) {
          put((uint32_t)cp);
        } else if (cp < 0x800) {
          put(0xC0 | (cp >> 6)); put(0x80 | (cp & 0x3F));
        } else if (cp < 0x10000) {
          put(0xE0 | (cp >> 12)); put(0x80 | ((cp >> 6) & 0x3F)); put(0x80 | (cp & 0x3F));
        } else {
          put(0xF0 | (cp >> 18)); put(0x80 | ((cp >> 12) & 0x3F)); put(0x80 | ((cp >> 6) & 0x3F));
          put(0x80 | (cp & 0x3F));
        }
        break;
      }
      default:
        return r;
    }
  }
  return r;
}

__device__ __forceinline__ uint64_t scan_str_esc(const uint8_t* s, uint64_t p, uint64_t e, Str& out, uint8_t* buf,
                                                 uint32_t cap) {
  const EscOut r = scan_str_esc_impl(s, p, e, buf, cap);
  out.len = r.len;
  out.w0 = r.w0;
  out.w1 = r.w1;
  out.esc = true;
  return r.pos;
}

#define CT_IS(x, lit) ((x).len == slen(lit) && (x).w0 == pk8(lit, 0) && (x).w1 == pk8(lit, 8))

// top-level keys the reader consults (events.py:294-349)
enum Key : int { K_SEQ, K_TS, K_KIND, K_COMM, K_NRANKS, K_RANK, K_DEV, K_COLL, K_ALGO, K_COUNT,
                 K_DTYPE, K_ROOT, K_PEER, K_CKIND, K_SRC, K_DST, K_BYTES, K_N };

__device__ __forceinline__ int key_of(const Str& k) {
  if (k.len > 6) return -1;
  if (CT_IS(k, "seq")) return K_SEQ;
  if (CT_IS(k, "ts")) return K_TS;
  if (CT_IS(k, "kind")) return K_KIND;
  if (CT_IS(k, "comm")) return K_COMM;
  if (CT_IS(k, "nranks")) return K_NRANKS;
  if (CT_IS(k, "rank")) return K_RANK;
  if (CT_IS(k, "dev")) return K_DEV;
  if (CT_IS(k, "coll")) return K_COLL;
  if (CT_IS(k, "algo")) return K_ALGO;
  if (CT_IS(k, "count")) return K_COUNT;
  if (CT_IS(k, "dtype")) return K_DTYPE;
  if (CT_IS(k, "root")) return K_ROOT;
  if (CT_IS(k, "peer")) return K_PEER;
  if (CT_IS(k, "ckind")) return K_CKIND;
  if (CT_IS(k, "src")) return K_SRC;
  if (CT_IS(k, "dst")) return K_DST;
  if (CT_IS(k, "bytes")) return K_BYTES;
  return -1;
}

// enum codes (packed.py KIND_CODE / COLL_CODE / ALGO_CODE / DTYPE_CODE / CKIND_CODE)
__device__ __forceinline__ int enum_of(int key, const Str& v) {
  switch (key) {
    case K_KIND:
      if (CT_IS(v, "collective")) return 0;
      if (CT_IS(v, "send")) return 1;
      if (CT_IS(v, "recv")) return 2;
      if (CT_IS(v, "memcpy")) return 3;
      if (CT_IS(v, "um")) return 4;
      if (CT_IS(v, "zerocopy")) return 5;
      return -1;
    case K_COLL:
      if (CT_IS(v, "allreduce")) return 0;
      if (CT_IS(v, "broadcast")) return 1;
      if (CT_IS(v, "reduce")) return 2;
      if (CT_IS(v, "reducescatter")) return 3;
      if (CT_IS(v, "allgather")) return 4;
      return -1;
    case K_ALGO:
      if (CT_IS(v, "ring")) return 0;
      if (CT_IS(v, "tree")) return 1;
      if (CT_IS(v, "collnet")) return 2;
      if (CT_IS(v, "auto")) return 3;
      return -1;
    case K_DTYPE:
      if (CT_IS(v, "float32")) return 8;
      if (CT_IS(v, "bfloat16")) return 7;
      if (CT_IS(v, "float16")) return 6;
      if (CT_IS(v, "int8")) return 0;
      if (CT_IS(v, "uint8")) return 1;
      if (CT_IS(v, "int32")) return 2;
      if (CT_IS(v, "uint32")) return 3;
      if (CT_IS(v, "int64")) return 4;
      if (CT_IS(v, "uint64")) return 5;
      if (CT_IS(v, "float64")) return 9;
      return -1;
    case K_CKIND:
      if (CT_IS(v, "h2d")) return 0;
      if (CT_IS(v, "d2h")) return 1;
      if (CT_IS(v, "d2d")) return 2;
      return -1;
    default:
      return -1;
  }
}

// value types: absent, int >= 0 (fits u64), int < 0 (fits i64), enum code, comm name,
// endpoint object, anything else (float, bool, null, array, other object, other
// string, huge int)
enum : uint8_t { V_NONE = 0, V_UINT, V_NINT, V_ENUM, V_NAME, V_EP, V_OTHER };

__device__ __forceinline__ bool is_ws(uint8_t c) { return c == ' ' || c == '\t'; }

__device__ __forceinline__ uint64_t skip_ws(const uint8_t* s, uint64_t p, uint64_t e) {
  while (p < e && is_ws(s[p])) p++;
  return p;
}

__device__ __forceinline__ uint32_t has_byte(uint32_t w, uint32_t rep) {
  const uint32_t x = w ^ rep;  // lowest set bit is exact (higher ones may be borrow artefacts)
  return (x - 0x01010101u) & ~x & 0x80808080u;
}

// string body after the opening quote, packing its first 16 bytes: position after the
// closing quote, or 0 on failure (the line holds no backslash / control / non-ASCII
// byte; a raw tab is invalid in a strict JSON string).  ``wl``: bytes below wl may be
// read as aligned 32-bit words (0: byte path only).
template <bool ESC>
__device__ __forceinline__ uint64_t scan_str(const uint8_t* s, uint64_t p, uint64_t e, Str& out, uint64_t wl) {
  const uint64_t p0 = p;
  if (p0 + 24 <= wl) {
    const uint64_t a = p0 & ~3ull;
    const uint32_t sh = (uint32_t)(p0 & 3) * 8;
    const uint32_t lowm = (1u << sh) - 1;
    uint64_t q = a;
    uint32_t w = (*reinterpret_cast<const uint32_t*>(s + a) & ~lowm) | (0x78787878u & lowm);
    uint64_t pos = 0;
    while (true) {
      const uint32_t hit = has_byte(w, 0x22222222u) | has_byte(w, 0x09090909u) | has_byte(w, 0x5C5C5C5Cu);
      if (hit) {
        const uint32_t j = (uint32_t)(__ffs(hit) - 1) >> 3;
        pos = q + j;
        if (pos >= e) return 0;
        const uint32_t c = (w >> (8 * j)) & 0xFF;
        if (c == '\\') return ESC ? scan_str_esc(s, p0, e, out, nullptr, 0) : 0;
        if (c != '"') return 0;
        break;
      }
      q += 4;
      if (q >= e) return 0;
      if (q + 4 > wl) {  // long string near the readable limit: finish bytewise
        pos = q;
        while (pos < e && s[pos] != '"') {
          if (s[pos] == '\t') return 0;
          if (s[pos] == '\\') return ESC ? scan_str_esc(s, p0, e, out, nullptr, 0) : 0;
          pos++;
        }
        if (pos >= e) return 0;
        break;
      }
      w = *reinterpret_cast<const uint32_t*>(s + q);
    }
    const uint32_t* wp = reinterpret_cast<const uint32_t*>(s + a);
    const uint64_t A = wp[0] | ((uint64_t)wp[1] << 32), B = wp[2] | ((uint64_t)wp[3] << 32), C4 = wp[4];
    uint64_t lo = A, hi = B;
    if (sh) {
      lo = (A >> sh) | (B << (64 - sh));
      hi = (B >> sh) | (C4 << (64 - sh));
    }
    const uint64_t len = pos - p0;
    if (len < 8) { lo &= (1ull << (8 * len)) - 1; hi = 0; }
    else if (len < 16) { hi &= (1ull << (8 * (len - 8))) - 1; }
    out.len = (uint32_t)len;
    out.w0 = lo;
    out.w1 = hi;
    return pos + 1;
  }
  uint64_t w0 = 0, w1 = 0;
  while (p < e) {
    const uint8_t c = s[p];
    if (c == '"') {
      out.len = (uint32_t)(p - p0);
      out.w0 = w0;
      out.w1 = w1;
      return p + 1;
    }
    if (c == '\t') return 0;
    if (c == '\\') return ESC ? scan_str_esc(s, p0, e, out, nullptr, 0) : 0;
    const uint64_t i = p - p0;
    if (i < 8) w0 |= (uint64_t)c << (8 * i);
    else if (i < 16) w1 |= (uint64_t)c << (8 * (i - 8));
    p++;
  }
  return 0;
}

// string body after the opening quote (the line holds no backslash / control byte /
// non-ASCII byte; a raw tab is invalid in a strict JSON string): position after the
// closing quote, or 0 on failure
template <bool ESC>
__device__ __forceinline__ uint64_t skip_string(const uint8_t* s, uint64_t p, uint64_t e) {
  const uint64_t p0 = p;
  while (p < e) {
    const uint8_t c = s[p++];
    if (c == '"') return p;
    if (c == '\t') return 0;
    if (c == '\\') {  // escapes are validated by the decoding scanner
      if (!ESC) return 0;
      Str x;
      return scan_str_esc(s, p0, e, x, nullptr, 0);
    }
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
    int nd = 0;
    while (p < e && s[p] >= '0' && s[p] <= '9') {
      const uint64_t dgt = s[p] - '0';
      if (nd < 19) mag = mag * 10 + dgt;  // < 10^19 cannot overflow
      else if (fits && mag <= (~0ull - dgt) / 10) mag = mag * 10 + dgt;
      else fits = false;
      nd++;
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
template <bool ESC>
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
      p = skip_string<ESC>(s, p + 1, e);
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
  p = skip_string<ESC>(s, p + 1, e);
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

// A value of a consulted key -> (type, payload): ints as values, enum strings as codes,
// the comm name as (offset | length << 40), anything else skipped as V_OTHER.
template <bool ESC>
__device__ uint64_t read_value(const uint8_t* s, uint64_t p, uint64_t e, int key, uint8_t& t, uint64_t& v,
                           uint64_t wl, const Side* side = nullptr) {
  p = skip_ws(s, p, e);
  if (p >= e) return 0;
  const uint8_t c = s[p];
  if (c == '"') {
    Str x;
    const uint64_t q = scan_str<ESC>(s, p + 1, e, x, wl);
    if (!q) return 0;
    if (key == K_COMM) {
      t = V_NAME;
      v = (p + 1) | ((uint64_t)x.len << 40);
      if (ESC && x.esc) {  // decoded name into the side buffer (too long / buffer full: the host reads the line)
        t = V_OTHER;
        if (side && x.len <= kMaxEscName) {
          const unsigned long long off = atomicAdd(side->used, (unsigned long long)x.len);
          if (off + x.len <= side->cap) {  // decode again, straight into the side buffer
            Str y;
            scan_str_esc(s, p + 1, e, y, side->buf + off, x.len);
            t = V_NAME;
            v = (off | kSideBit) | ((uint64_t)x.len << 40);
          }
        }
      }
    } else {
      const int code = enum_of(key, x);
      t = code >= 0 ? V_ENUM : V_OTHER;
      v = (uint64_t)code;
    }
    return q;
  }
  if (c == '-' || (c >= '0' && c <= '9')) {
    bool neg, is_int, fits;
    uint64_t mag;
    const uint64_t q = scan_number(s, p, e, is_int, mag, neg, fits);
    if (!q) return 0;
    if (!is_int || !fits) t = V_OTHER;
    else if (!neg || mag == 0) { t = V_UINT; v = mag; }      // "-0" is the int 0
    else if (mag <= (1ull << 63)) { t = V_NINT; v = 0ull - mag; }
    else t = V_OTHER;
    return q;
  }
  t = V_OTHER;
  return skip_value<ESC>(s, p, e);
}

// Endpoint object {"kind": <str>, "idx": <int>} (events.py:271-284) -> V_EP with
// payload kind code (host 0, gpu 1, net 2; 0xFF absent/invalid) | idx << 8 (idx
// 0xFFFFFFFF absent/invalid/too large); other members grammar-checked and ignored;
// duplicate keys: last wins (json.loads).
template <bool ESC>
__device__ uint64_t read_endpoint(const uint8_t* s, uint64_t p, uint64_t e, uint8_t& t, uint64_t& v, uint64_t wl) {
  p = skip_ws(s, p, e);
  if (p >= e) return 0;
  if (s[p] != '{') { t = V_OTHER; return skip_value<ESC>(s, p, e); }
  uint32_t kind = 0xFF, idx = 0xFFFFFFFFu;
  p = skip_ws(s, p + 1, e);
  if (p < e && s[p] == '}') { t = V_EP; v = kind | ((uint64_t)idx << 8); return p + 1; }
  while (true) {
    p = skip_ws(s, p, e);
    if (p >= e || s[p] != '"') return 0;
    Str k;
    p = scan_str<ESC>(s, p + 1, e, k, wl);
    if (!p) return 0;
    p = skip_ws(s, p, e);
    if (p >= e || s[p] != ':') return 0;
    p++;
    if (CT_IS(k, "kind")) {
      p = skip_ws(s, p, e);
      if (p < e && s[p] == '"') {
        Str x;
        p = scan_str<ESC>(s, p + 1, e, x, wl);
        if (!p) return 0;
        kind = CT_IS(x, "host") ? 0 : CT_IS(x, "gpu") ? 1 : CT_IS(x, "net") ? 2 : 0xFF;
      } else {
        p = skip_value<ESC>(s, p, e);
        kind = 0xFF;
      }
    } else if (CT_IS(k, "idx")) {
      uint8_t wt = V_NONE;
      uint64_t wv = 0;
      p = read_value<ESC>(s, p, e, -1, wt, wv, wl);
      idx = wt == V_UINT && wv <= 0xFFFF ? (uint32_t)wv : 0xFFFFFFFFu;
    } else {
      p = skip_value<ESC>(s, p, e);
    }
    if (!p) return 0;
    p = skip_ws(s, p, e);
    if (p >= e) return 0;
    if (s[p] == ',') { p++; continue; }
    if (s[p] == '}') { t = V_EP; v = kind | ((uint64_t)idx << 8); return p + 1; }
    return 0;
  }
}

struct LineOut {
  ct_record r;
  int64_t ts;
  uint64_t hash;
  uint64_t comm;  // name offset | length << 40
};

__device__ __forceinline__ bool byte_blank(uint8_t c) { return c == ' ' || c == '\t' || c == 0x1f; }
// bytes the device does not read itself: raw control characters (invalid in JSON strings,
// never JSON whitespace here).  Non-ASCII bytes and backslash escapes are decoded.
__device__ __forceinline__ bool byte_odd(uint8_t c) { return c < 0x20 && c != '\t'; }

// Line class before parsing: 0 blank (str.strip: the ASCII whitespace left inside a
// line is space, tab, \x1f), 1 plain (no byte the device does not decode itself:
// non-ASCII, backslash, control other than tab), 2 otherwise.  4 bytes at a time where
// the text is word-aligned.
__device__ __forceinline__ int line_class(const uint8_t* s, uint64_t b, uint64_t e, bool words) {
  bool blank = true, plain = true, bsl = false;
  uint64_t p = b;
  if (words) {
    for (; p < e && (p & 3); p++) {
      const uint8_t c = s[p];
      blank &= byte_blank(c);
      plain &= !byte_odd(c);
      bsl |= c == '\\';
    }
    for (; p + 4 <= e; p += 4) {
      const uint32_t w = *reinterpret_cast<const uint32_t*>(s + p);
      const uint32_t ctl = (w - 0x20202020u) & ~w & 0x80808080u;  // some byte < 0x20 (or >= 0x80)
      const uint32_t bs = w ^ 0x5C5C5C5Cu;
      const uint32_t has_bs = (bs - 0x01010101u) & ~bs & 0x80808080u;
      if ((w & 0x80808080u) | ctl | has_bs) {
        for (int q = 0; q < 4; q++) {
          const uint8_t c = (uint8_t)(w >> (8 * q));
          blank &= byte_blank(c);
          plain &= !byte_odd(c);
          bsl |= c == '\\';
        }
      } else if (w != 0x20202020u) {
        blank = false;
      }
    }
  }
  for (; p < e; p++) {
    const uint8_t c = s[p];
    blank &= byte_blank(c);
    plain &= !byte_odd(c);
    bsl |= c == '\\';
  }
  return blank ? 0 : !plain ? 2 : bsl ? 3 : 1;
}

// The canonical wire line -- write_trace's key order and compact separators
// (events.py:251-291), which the reference, this package and the interposer all emit:
//   {"seq":N,"ts":N,"kind":"K","comm":"S","nranks":N,"rank":N,"dev":N, then
//   collective  "coll":"E","algo":"E","count":N,"dtype":"E"[,"root":N]}
//   send / recv "peer":N,"count":N,"dtype":"E"}
//   copies      "ckind":"E","src":{"kind":"E","idx":N},"dst":{...},"bytes":N}
// matched literal by literal, values read by the generic readers.  true: every
// consulted key was read into (types, fld) exactly as the generic loop would (the key
// set is fixed, no duplicates, nothing else); false: any deviation -- the generic JSON
// parser then reads the line from the start.  This skips the per-key name lookups,
// which dominate the generic parse.
template <int N>
__device__ __forceinline__ bool lit_at(const uint8_t* s, uint64_t& p, uint64_t e, const char (&lit)[N]) {
  if (p + (N - 1) > e) return false;
  bool ok = true;
#pragma unroll
  for (int i = 0; i < N - 1; i++) ok &= s[p + i] == (uint8_t)lit[i];
  p += N - 1;
  return ok;
}

template <bool ESC>
__device__ bool parse_canonical(const uint8_t* s, uint64_t b, uint64_t e, uint64_t wl, uint64_t* fld, int stride,
                                uint64_t& types, const Side& side) {
  uint64_t p = b;
  auto val = [&](int key) -> bool {
    uint8_t t = V_NONE;
    uint64_t v = 0;
    p = (key == K_SRC || key == K_DST) ? read_endpoint<ESC>(s, p, e, t, v, wl)
                                       : read_value<ESC>(s, p, e, key, t, v, wl, &side);
    types |= (uint64_t)t << (3 * key);
    fld[key * stride] = v;
    return p != 0;
  };
  types = 0;
  if (!lit_at(s, p, e, "{\"seq\":") || !val(K_SEQ) || !lit_at(s, p, e, ",\"ts\":") || !val(K_TS) ||
      !lit_at(s, p, e, ",\"kind\":") || !val(K_KIND) || !lit_at(s, p, e, ",\"comm\":") || !val(K_COMM) ||
      !lit_at(s, p, e, ",\"nranks\":") || !val(K_NRANKS) || !lit_at(s, p, e, ",\"rank\":") || !val(K_RANK) ||
      !lit_at(s, p, e, ",\"dev\":") || !val(K_DEV))
    return false;
  if (((types >> (3 * K_KIND)) & 7) != V_ENUM) return false;
  const uint64_t kind = fld[K_KIND * stride];
  if (kind == CT_KIND_COLLECTIVE) {
    if (!lit_at(s, p, e, ",\"coll\":") || !val(K_COLL) || !lit_at(s, p, e, ",\"algo\":") || !val(K_ALGO) ||
        !lit_at(s, p, e, ",\"count\":") || !val(K_COUNT) || !lit_at(s, p, e, ",\"dtype\":") || !val(K_DTYPE))
      return false;
    if (p < e && s[p] == ',' && (!lit_at(s, p, e, ",\"root\":") || !val(K_ROOT))) return false;
  } else if (kind == CT_KIND_SEND || kind == CT_KIND_RECV) {
    if (!lit_at(s, p, e, ",\"peer\":") || !val(K_PEER) || !lit_at(s, p, e, ",\"count\":") || !val(K_COUNT) ||
        !lit_at(s, p, e, ",\"dtype\":") || !val(K_DTYPE))
      return false;
  } else {
    if (!lit_at(s, p, e, ",\"ckind\":") || !val(K_CKIND) || !lit_at(s, p, e, ",\"src\":") || !val(K_SRC) ||
        !lit_at(s, p, e, ",\"dst\":") || !val(K_DST) || !lit_at(s, p, e, ",\"bytes\":") || !val(K_BYTES))
      return false;
  }
  if (!lit_at(s, p, e, "}")) return false;
  return skip_ws(s, p, e) == e;  // "Extra data" otherwise (the generic path defers it)
}

// Parse line [b, e) of s; L_OK with `o` filled, L_BLANK, or L_DEFER.  ``fld`` is this
// thread's field slots in shared memory (key k at fld[k * stride]).
template <bool ESC>
__device__ uint8_t parse_line(const uint8_t* s, uint64_t b, uint64_t e, bool words, uint64_t wl, uint64_t* fld,
                              int stride, const Side& side, LineOut& o) {
  const int cls = line_class(s, b, e, words);
  if (cls == 0) return L_BLANK;
  if (cls == 2) return L_DEFER;
  if (cls == 3 && !ESC) return L_ESC;

  // consulted fields: types 3 bits per key (register), payloads in shared memory
  uint64_t types = 0;
  if (parse_canonical<ESC>(s, b, e, wl, fld, stride, types, side)) goto consulted;
  types = 0;
  {
  uint64_t p = skip_ws(s, b, e);
  if (p >= e || s[p] != '{') return L_DEFER;
  p = skip_ws(s, p + 1, e);
  if (p < e && s[p] == '}') return L_DEFER;  // {}: "kind" missing
  while (true) {
    p = skip_ws(s, p, e);
    if (p >= e || s[p] != '"') return L_DEFER;
    Str k;
    p = scan_str<ESC>(s, p + 1, e, k, wl);
    if (!p) return L_DEFER;
    const int key = key_of(k);
    p = skip_ws(s, p, e);
    if (p >= e || s[p] != ':') return L_DEFER;
    p++;
    if (key < 0) {
      p = skip_value<ESC>(s, p, e);
    } else {
      uint8_t t = V_NONE;
      uint64_t v = 0;
      p = (key == K_SRC || key == K_DST) ? read_endpoint<ESC>(s, p, e, t, v, wl)
                                         : read_value<ESC>(s, p, e, key, t, v, wl, &side);
      types = (types & ~(7ull << (3 * key))) | ((uint64_t)t << (3 * key));
      fld[key * stride] = v;
    }
    if (!p) return L_DEFER;
    p = skip_ws(s, p, e);
    if (p >= e) return L_DEFER;
    if (s[p] == ',') { p++; continue; }
    if (s[p] == '}') { p++; break; }
    return L_DEFER;
  }
  if (skip_ws(s, p, e) != e) return L_DEFER;  // "Extra data"
  }

consulted:
  // the reader's consulted keys and TraceEvent.validate, in effect (events.py:287-310)
  auto ty = [&](int key) -> uint32_t { return (uint32_t)(types >> (3 * key)) & 7; };
  auto fv = [&](int key) -> uint64_t { return ty(key) == V_NONE ? 0 : fld[key * stride]; };
  const uint64_t f_seq = fv(K_SEQ), f_ts = fv(K_TS), f_kind = fv(K_KIND), f_comm = fv(K_COMM),
                 f_nranks = fv(K_NRANKS), f_rank = fv(K_RANK), f_dev = fv(K_DEV), f_coll = fv(K_COLL),
                 f_algo = fv(K_ALGO), f_count = fv(K_COUNT), f_dtype = fv(K_DTYPE), f_root = fv(K_ROOT),
                 f_peer = fv(K_PEER), f_ckind = fv(K_CKIND), f_src = fv(K_SRC), f_dst = fv(K_DST),
                 f_bytes = fv(K_BYTES);
  if (ty(K_KIND) != V_ENUM) return L_DEFER;
  const int kind = (int)f_kind;
  if (ty(K_SEQ) != V_UINT || ty(K_COMM) != V_NAME || ty(K_NRANKS) != V_UINT || ty(K_RANK) != V_UINT ||
      ty(K_DEV) != V_UINT)
    return L_DEFER;
  if (ty(K_TS) == V_UINT) {
    if (f_ts >= (1ull << 63)) return L_DEFER;
  } else if (ty(K_TS) != V_NINT) {
    return L_DEFER;
  }
  const uint64_t n = f_nranks, rank = f_rank, dev = f_dev;
  if (n < 1 || n > 0xFFFF || rank >= n || dev > 0xFFFF) return L_DEFER;
  ct_record& r = o.r;
  r.seq = f_seq;
  r.comm = 0;
  r.nranks = (uint16_t)n;
  r.rank = (uint16_t)rank;
  r.dev = (uint16_t)dev;
  r.aux = 0;
  r.aux2 = 0;
  if (kind == CT_KIND_COLLECTIVE) {
    if (ty(K_COLL) != V_ENUM || ty(K_ALGO) != V_ENUM || ty(K_DTYPE) != V_ENUM || ty(K_COUNT) != V_UINT)
      return L_DEFER;
    const int coll = (int)f_coll, algo = (int)f_algo, dt = (int)f_dtype;
    const bool rooted = coll == CT_COLL_BROADCAST || coll == CT_COLL_REDUCE;
    if (ty(K_ROOT) != V_NONE || rooted) {
      if (ty(K_ROOT) != V_UINT) return L_DEFER;
      if (!rooted || f_root >= n) return L_DEFER;  // root only for bcast/reduce, in [0, N)
      r.aux = (uint16_t)f_root;
    }
    if ((algo == CT_ALGO_TREE || algo == CT_ALGO_COLLNET) && coll != CT_COLL_ALLREDUCE) return L_DEFER;
    r.count = f_count;
    r.kc = (uint8_t)(kind | (coll << 3) | (rooted ? 1 << 6 : 0));
    r.ad = (uint8_t)(algo | (dt << 2));
  } else if (kind == CT_KIND_SEND || kind == CT_KIND_RECV) {
    if (ty(K_PEER) != V_UINT || ty(K_COUNT) != V_UINT || ty(K_DTYPE) != V_ENUM) return L_DEFER;
    if (f_peer == rank || f_peer >= n) return L_DEFER;
    r.aux = (uint16_t)f_peer;
    r.count = f_count;
    r.kc = (uint8_t)kind;
    r.ad = (uint8_t)(f_dtype << 2);
  } else {
    if (ty(K_CKIND) != V_ENUM || ty(K_SRC) != V_EP || ty(K_DST) != V_EP || ty(K_BYTES) != V_UINT) return L_DEFER;
    const int ck = (int)f_ckind;
    const uint32_t sk = (uint32_t)(f_src & 0xFF), dk = (uint32_t)(f_dst & 0xFF);
    const uint32_t si = (uint32_t)(f_src >> 8), di = (uint32_t)(f_dst >> 8);
    if (si == 0xFFFFFFFFu || di == 0xFFFFFFFFu) return L_DEFER;  // absent / negative / > 65535
    const uint32_t want_s = ck == CT_CKIND_H2D ? 0 : 1, want_d = ck == CT_CKIND_D2H ? 0 : 1;  // host 0, gpu 1
    if (sk != want_s || dk != want_d) return L_DEFER;
    if ((want_s == 0 && si != 0) || (want_d == 0 && di != 0)) return L_DEFER;
    if (ck == CT_CKIND_D2D && si == di) return L_DEFER;
    r.aux = (uint16_t)si;
    r.aux2 = (uint16_t)di;
    r.count = f_bytes;
    r.kc = (uint8_t)kind;
    r.ad = (uint8_t)(ck << 6);
  }
  o.ts = (int64_t)f_ts;
  if ((f_comm >> 40) >= (1ull << 23)) return L_DEFER;  // name length field
  o.comm = f_comm;
  uint64_t h = 0xcbf29ce484222325ull;  // FNV-1a over the name bytes
  const uint8_t* name = name_ptr(s, side.buf, f_comm);
  const uint64_t clen = f_comm >> 40;
  for (uint64_t j = 0; j < clen; j++) h = (h ^ name[j]) * 0x100000001b3ull;
  o.hash = h == kNoKey ? kNoKey - 1 : h;
  return L_OK;
}

// One thread per line; a block's lines are contiguous in the text, so the block first
// copies their bytes into shared memory with 16-byte loads (when they fit) and every
// thread parses from there.
constexpr int kParseThreads = 128;
#ifndef CT_JSONL_STAGE
#define CT_JSONL_STAGE (24 * 1024)
#endif
constexpr uint32_t kStage = CT_JSONL_STAGE;
constexpr uint32_t kStageSlack = 32;  // readable bytes past the stage (word scans)

__global__ void __launch_bounds__(kParseThreads) k_parse(const uint8_t* s, uint64_t size, bool aligned,
                                                         const uint64_t* brk, uint64_t nb, uint64_t n_lines,
                                                         uint8_t* status, LineOut* out, Side side) {
  extern __shared__ __align__(16) uint8_t stage[];
  const uint64_t k0 = blockIdx.x * (uint64_t)kParseThreads;
  const uint64_t k1 = min(k0 + kParseThreads, n_lines) - 1;  // last line of the block
  auto line_begin = [&](uint64_t k) { return k == 0 ? 0 : brk[k - 1] + break_len(s, size, brk[k - 1]); };
  auto line_end = [&](uint64_t k) { return k < nb ? brk[k] : size; };
  const uint64_t span_b = line_begin(k0) & ~15ull, span_e = line_end(k1);
  const bool staged = aligned && span_e - span_b <= kStage;
  const uint8_t* src = s;
  if (staged) {
    const uint64_t nv = (span_e - span_b + 15) / 16;
    for (uint64_t v = threadIdx.x; v < nv; v += kParseThreads) {
      const uint64_t a = span_b + v * 16;
      uint4 w;
      if (a + 16 <= size) {
        w = *reinterpret_cast<const uint4*>(s + a);
      } else {
        uint8_t t[16];
        for (int q = 0; q < 16; q++) t[q] = a + q < size ? s[a + q] : 0;
        memcpy(&w, t, 16);
      }
      *reinterpret_cast<uint4*>(stage + v * 16) = w;
    }
    src = stage - span_b;  // absolute positions index the staged copy
  }
  __syncthreads();
  const uint64_t k = k0 + threadIdx.x;
  if (k >= n_lines) return;
  __shared__ uint64_t fields[K_N * kParseThreads];
  LineOut o;
  // word reads may run up to 24 bytes past a string start: the stage has that slack,
  // the global text is read wordwise only away from its end
  const uint64_t wl = !aligned ? 0 : staged ? span_b + kStage + kStageSlack : (size > 32 ? size - 8 : 0);
  const uint8_t st =
      parse_line<false>(src, line_begin(k), line_end(k), aligned, wl, fields + threadIdx.x, kParseThreads, side, o);
  status[k] = st;
  if (st == L_OK) {
    out[k] = o;
  }
}

// Lines holding escapes (L_ESC after k_parse), one thread each, straight from the text:
// the same parser with \\ / \\uXXXX decoding (comm names into the side buffer).
__global__ void __launch_bounds__(kParseThreads) k_parse_esc(const uint8_t* s, uint64_t size, bool aligned,
                                                             const uint64_t* brk, uint64_t nb, const uint64_t* lines,
                                                             const uint64_t* n_esc, uint8_t* status, LineOut* out,
                                                             Side side) {
  __shared__ uint64_t fields[K_N * kParseThreads];
  const uint64_t j = blockIdx.x * (uint64_t)kParseThreads + threadIdx.x;
  if (j >= *n_esc) return;
  const uint64_t k = lines[j];
  const uint64_t b = k == 0 ? 0 : brk[k - 1] + break_len(s, size, brk[k - 1]);
  const uint64_t e = k < nb ? brk[k] : size;
  const uint64_t wl = aligned && size > 32 ? size - 8 : 0;
  LineOut o;
  const uint8_t st = parse_line<true>(s, b, e, aligned, wl, fields + threadIdx.x, kParseThreads, side, o);
  status[k] = st;
  if (st == L_OK) out[k] = o;
}

struct IsEsc {
  const uint8_t* st;
  __device__ __forceinline__ bool operator()(uint64_t k) const { return st[k] == L_ESC; }
};

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
      coff[i] = lo[k].comm;
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
                         const uint64_t* seg_coff, const uint64_t* coff, const uint8_t* s, const uint8_t* side,
                         unsigned int* collide) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
    if (keys[i] == kNoKey) continue;
    const uint64_t a = coff[vals[i]], h = seg_coff[seg[i] - 1];
    if (a == h) continue;
    const uint32_t la = (uint32_t)(a >> 40), lh = (uint32_t)(h >> 40);
    bool same = la == lh;
    const uint8_t *na = name_ptr(s, side, a), *nh = name_ptr(s, side, h);
    for (uint32_t j = 0; same && j < la; j++) same = na[j] == nh[j];
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
                        const uint64_t* name_off, const uint8_t* s, const uint8_t* side, uint8_t* names,
                        uint64_t* rows) {
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < u; r += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t g = seg_order[r], c = seg_coff[g];
    const uint64_t len = c >> 40;
    const uint8_t* nm = name_ptr(s, side, c);
    for (uint64_t j = 0; j < len; j++) names[name_off[r] + j] = nm[j];
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


// ---------------------------------------------------------------- fused single pass
// The common case in one pass over the text.  One CTA per 32 KB tile,
// claimed in text order through a ticket.  A line belongs to the tile holding its
// terminator (the final unterminated line: the last tile); its start lies in the tile
// or in the kFM bytes before it, which are staged with the tile.  Per tile: terminator
// masks over the staged bytes -> ordered line ends; a blank test per line -> record
// slots; a decoupled look-back over earlier tiles -> the tile's first line number and
// record slot; then every line goes through the canonical-template parser (thread per
// line, from shared memory) or onto the slow list, which the generic parser (escapes
// included) reads in the next kernel.  Comm names are interned through a per-CTA cache
// into a global open-addressing table of 64-bit name keys; records carry the table slot
// until the final remap into first-seen order.  Outside these bounds (a line longer than
// the look-behind, > kFMaxLines lines in a tile, > kFMaxNames names, lists or record
// slots beyond their capacity) the fallback flag is raised and the caller reruns the
// multi-pass pipeline, which has no such bounds.
#ifndef CT_FTHREADS
#define CT_FTHREADS 256
#endif
constexpr int kFThreads = CT_FTHREADS;
constexpr uint32_t kFT = kFThreads * 128;  // terminator bytes per tile: 8 groups of 16 per thread
constexpr uint32_t kFM = 4 * 1024;    // look-behind: a line may start this far before its tile
constexpr uint32_t kFStage = kFM + kFT + 128;  // + zero padding (template reads overrun)
// stage offsets of line ends / tail starts: 16 bits while the stage allows it
using StOff = std::conditional_t<(kFM + kFT < 65536), uint16_t, uint32_t>;
constexpr int kFMaxLines = (int)kFT / 16;
constexpr int kFMaxRecs = (int)kFT / 64;  // records per tile (non-blank lines averaging >= 64 bytes)
constexpr int kFCache = 64;           // per-CTA name cache entries
constexpr uint32_t kFNameMax = 32;    // longest name the cache holds (longer: slow list)
constexpr uint32_t kFTable = 1u << 14;
constexpr uint32_t kFMaxNames = 2048;  // distinct names (k_ffinal ranks them in one CTA)
constexpr uint64_t kFNameCap = 1ull << 20;
constexpr uint64_t kFListCap = 1ull << 22;

enum : uint32_t { FB_FALLBACK = 1, FB_NONASCII = 2, FB_COLLIDE = 4 };

struct FCtl {
  unsigned long long ticket;
  unsigned long long n_lines, n_recs;
  unsigned long long n_slow, n_defer, n_verify;
  unsigned long long name_bytes;
  unsigned int flags, n_names, n_used;
  unsigned int pad;
};

static_assert(sizeof(FCtl) % 8 == 0, "k_finit clears FCtl as 64-bit words");

struct FArgs {
  const uint8_t* s;
  uint64_t size, ntiles, cap;
  FCtl* ctl;
  uint32_t* tcnt;             // per tile: lines, records
  unsigned long long* toff;    // per tile: first line, first record (k_fscan)
  ct_record* trec;             // per tile: kFMaxRecs temporary record slots
  int64_t* tts;
  ct_record* recs;             // final records / timestamps (k_fcompact)
  int64_t* ts;
  unsigned long long *gkey, *gname, *gfirst;  // name table: key, name ref, first record slot
  uint32_t* gid;                               // table slot -> comm id
  uint32_t* gused;                             // inserted table slots, in insertion order
  uint64_t *slow, *defer, *verify;             // 4, 4, 2 words per entry
  uint64_t* comm_rows;
  uint8_t* names;
  uint64_t lcap;  // entries of each list
  Side side;
};

__device__ __forceinline__ void fb(const FArgs& A, uint32_t f) { atomicOr(&A.ctl->flags, f); }

// 64-bit name key: little-endian 8-byte words (zero-padded), then the length; never 0
__device__ __forceinline__ uint64_t nk_mix(uint64_t h, uint64_t w) {
  h = (h ^ w) * 0x9E3779B97F4A7C15ull;
  return h ^ (h >> 29);
}
__device__ __forceinline__ uint64_t nk_final(uint64_t h, uint32_t len) {
  h = nk_mix(h, len);
  return h ? h : 1;
}
__device__ uint64_t name_key_bytes(const uint8_t* p, uint32_t len) {
  uint64_t h = 0x243F6A8885A308D3ull;
  for (uint32_t i = 0; i < len; i += 8) {
    uint64_t w = 0;
    for (uint32_t k = 0; k < 8 && i + k < len; k++) w |= (uint64_t)p[i + k] << (8 * k);
    h = nk_mix(h, w);
  }
  return nk_final(h, len);
}

// global name table slot of ``key`` (inserted with its name reference when new), -1: full
__device__ int table_slot(const FArgs& A, uint64_t key, uint64_t ref) {
  uint32_t i = (uint32_t)(key ^ (key >> 32)) & (kFTable - 1);
  for (uint32_t probe = 0; probe < kFTable / 2; probe++) {
    const unsigned long long old = atomicCAS(&A.gkey[i], 0ull, (unsigned long long)key);
    if (old == 0) {
      A.gname[i] = ref;
      const unsigned int u = atomicAdd(&A.ctl->n_names, 1u);
      if (u < kFMaxNames) A.gused[u] = i;
      else fb(A, FB_FALLBACK);
      return (int)i;
    }
    if (old == key) return (int)i;
    i = (i + 1) & (kFTable - 1);
  }
  fb(A, FB_FALLBACK);
  return -1;
}

__device__ __forceinline__ bool list_put(const FArgs& A, unsigned long long* cnt, uint64_t* list, int words,
                                         uint64_t a, uint64_t b, uint64_t c, uint64_t d) {
  const unsigned long long i = atomicAdd(cnt, 1ull);
  if (i >= A.lcap) { fb(A, FB_FALLBACK); return false; }
  list[words * i] = a;
  list[words * i + 1] = b;
  if (words == 4) { list[4 * i + 2] = c; list[4 * i + 3] = d; }
  return true;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// unaligned 8 bytes of the (16-byte aligned) stage at p
__device__ __forceinline__ uint64_t st8(const uint8_t* st, uint32_t p) {
  const uint32_t* W = reinterpret_cast<const uint32_t*>(st);
  const uint32_t i = p >> 2, sh = (p & 3) * 8;
  const uint32_t w0 = W[i], w1 = W[i + 1], w2 = W[i + 2];
  return (uint64_t)__funnelshift_r(w0, w1, sh) | ((uint64_t)__funnelshift_r(w1, w2, sh) << 32);
}

// terminator starts in stage bytes [q, q + 16) (absolute position st0 + q): the same
// rules as break_mask16; bytes at or past ``size`` are never terminators
__device__ uint32_t brk16s(const uint8_t* st, uint32_t q, uint64_t st0, const uint8_t* s, uint64_t size,
                           bool& non_ascii) {
  non_ascii = false;
  const uint4 v = *reinterpret_cast<const uint4*>(st + q);
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
  uint32_t cand = 0;
#pragma unroll
  for (int k = 0; k < 4; k++) {
    const uint32_t t = (((w[k] - 0x20202020u) & ~w[k]) | w[k]) & 0x80808080u;
    cand |= (((t >> 7) & 1u) | ((t >> 14) & 2u) | ((t >> 21) & 4u) | ((t >> 28) & 8u)) << (4 * k);
  }
  if (!cand) return 0;
  uint32_t m = 0;
  bool hi = false;
  while (cand) {
    const int j = __ffs(cand) - 1;
    cand &= cand - 1;
    const uint64_t i = st0 + q + j;
    if (i >= size) break;
    const uint32_t c = st[q + j];
    hi |= c >= 0x80;
    bool brk;
    if (c == '\n') brk = q + j > 0 ? st[q + j - 1] != '\r' : (i == 0 || s[i - 1] != '\r');
    else if (c == '\r' || c == 0x0b || c == 0x0c || c == 0x1c || c == 0x1d || c == 0x1e) brk = true;
    else if (c == 0xC2) brk = i + 1 < size && st[q + j + 1] == 0x85;
    else if (c == 0xE2) brk = i + 2 < size && st[q + j + 1] == 0x80 && (st[q + j + 2] == 0xA8 || st[q + j + 2] == 0xA9);
    else brk = false;
    if (brk) m |= 1u << j;
  }
  non_ascii = hi;
  return m;
}

// brk16s for the common group: its only byte below 0x20 is '\n' (not after a '\r') and
// none is >= 0x80 -- branch-free; ``rare`` asks for brk16s otherwise
__device__ __forceinline__ uint32_t brk16f(const uint8_t* st, uint32_t q, uint64_t st0, uint64_t size, bool& rare) {
  const uint4 v = *reinterpret_cast<const uint4*>(st + q);
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
  uint32_t m = 0, odd = 0;
#pragma unroll
  for (int k = 0; k < 4; k++) {
    const uint32_t x = w[k] ^ 0x0A0A0A0Au;
    const uint32_t z = ~(((x & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | x | 0x7F7F7F7Fu);  // exact: byte == '\n'
    odd |= ((((w[k] - 0x20202020u) & ~w[k]) | w[k]) & 0x80808080u) & ~z;      // other control / non-ASCII
    m |= (((z >> 7) * 0x01020408u) >> 24) << (4 * k);
  }
  rare = odd != 0 || st0 + q + 16 > size || ((m & 1u) && (q == 0 || st[q - 1] == '\r'));
  return m;
}

__device__ __forceinline__ uint32_t blen_s(const uint8_t* st, uint32_t p, uint32_t nst) {
  const uint8_t b = st[p];
  if (b == '\r') return p + 1 < nst && st[p + 1] == '\n' ? 2 : 1;
  if (b == 0xC2) return 2;
  if (b == 0xE2) return 3;
  return 1;
}

// ---- canonical-template parser over the stage (write_trace's key order, compact
// separators; see parse_canonical).  Every byte of [b, e) is consumed by a literal, a
// number, an enum value or the comm name, so acceptance implies a plain line.
struct FLine {
  ct_record r;
  int64_t ts;
  uint64_t key;       // name key
  uint32_t nb, nlen;  // name: stage offset, length
};

template <int N>
__device__ __forceinline__ bool flit(const uint8_t* st, uint32_t& p, const char (&lit)[N]) {
  constexpr int L = N - 1;
  uint64_t v0 = 0, v1 = 0;
#pragma unroll
  for (int i = 0; i < L && i < 8; i++) v0 |= (uint64_t)(uint8_t)lit[i] << (8 * i);
#pragma unroll
  for (int i = 8; i < L && i < 16; i++) v1 |= (uint64_t)(uint8_t)lit[i] << (8 * (i - 8));
  const uint64_t m0 = L >= 8 ? ~0ull : (1ull << (8 * L)) - 1;
  const uint64_t m1 = L <= 8 ? 0ull : (L >= 16 ? ~0ull : (1ull << (8 * (L - 8))) - 1);
  bool ok = (st8(st, p) & m0) == v0;
  if (L > 8) ok = ok && (st8(st, p + 8) & m1) == v1;
  if (L > 16) ok = ok && st[p + 16] == (uint8_t)lit[16];
  p += L;
  return ok;
}

__constant__ uint64_t kPow10[9] = {1ull, 10ull, 100ull, 1000ull, 10000ull, 100000ull, 1000000ull, 10000000ull,
                                   100000000ull};

// up to 8 digit values (first digit in the lowest byte) -> integer
__device__ __forceinline__ uint64_t swar8(uint64_t d, uint32_t k) {
  d <<= 8 * (8 - k);
  d = (d * 10 + (d >> 8)) & 0x00FF00FF00FF00FFull;
  d = (d * 100 + (d >> 16)) & 0x0000FFFF0000FFFFull;
  return (d * 10000 + (d >> 32)) & 0xFFFFFFFFull;
}

// JSON integer (no sign) of <= 19 digits at p: false for anything else (leading zeros,
// 20+ digits; fractions / exponents fail on the literal that follows)
__device__ __forceinline__ bool fnum_i(const uint8_t* st, uint32_t& p, uint64_t& v) {
  uint64_t x = st8(st, p) ^ 0x3030303030303030ull;
  uint64_t nd = ((x + 0x7676767676767676ull) | x) & 0x8080808080808080ull;
  uint32_t k = nd ? (uint32_t)(__ffsll((long long)nd) - 1) >> 3 : 8u;
  if (k == 0 || ((x & 0xFF) == 0 && k > 1)) return false;
  v = swar8(x, k);
  uint32_t tot = k;
  while (k == 8) {
    x = st8(st, p + tot) ^ 0x3030303030303030ull;
    nd = ((x + 0x7676767676767676ull) | x) & 0x8080808080808080ull;
    k = nd ? (uint32_t)(__ffsll((long long)nd) - 1) >> 3 : 8u;
    if (tot + k > 19) return false;
    if (k) v = v * kPow10[k] + swar8(x, k);
    tot += k;
  }
  p += tot;
  return true;
}

// string body at p (after the quote) up to 16 bytes without escapes: packed value for
// enum_of; p moves past the closing quote
__device__ __forceinline__ bool fstr16_i(const uint8_t* st, uint32_t& p, Str& out) {
  const uint64_t x = st8(st, p), y = st8(st, p + 8);
  const uint64_t qx = x ^ 0x2222222222222222ull, qy = y ^ 0x2222222222222222ull;
  const uint64_t zx = (qx - 0x0101010101010101ull) & ~qx & 0x8080808080808080ull;
  const uint64_t zy = (qy - 0x0101010101010101ull) & ~qy & 0x8080808080808080ull;
  uint32_t len;
  if (zx) len = (uint32_t)(__ffsll((long long)zx) - 1) >> 3;
  else if (zy) len = 8 + ((uint32_t)(__ffsll((long long)zy) - 1) >> 3);
  else return false;
  out.len = len;
  out.w0 = len >= 8 ? x : (x & ((1ull << (8 * len)) - 1));
  out.w1 = len <= 8 ? 0ull : (y & ((1ull << (8 * (len - 8))) - 1));
  p += len + 1;
  return true;
}

// One out-of-line copy of each value reader (CT_FNOINLINE, default on): the template
// parser calls them ~20 times per line, and inlining every call site made the kernel's
// code larger than the instruction cache; results come back by value (registers).
#ifndef CT_FNOINLINE
#define CT_FNOINLINE 1
#endif
struct NumOut {
  uint64_t v;
  uint32_t p;
  uint32_t ok;
};
__device__ __noinline__ NumOut fnum_o(const uint8_t* st, uint32_t p) {
  NumOut r;
  r.ok = fnum_i(st, p, r.v) ? 1u : 0u;
  r.p = p;
  return r;
}
struct StrOut {
  uint64_t w0, w1;
  uint32_t len, p, ok;
};
__device__ __noinline__ StrOut fstr16_o(const uint8_t* st, uint32_t p) {
  Str s;
  StrOut r;
  r.ok = fstr16_i(st, p, s) ? 1u : 0u;
  r.p = p;
  r.w0 = s.w0;
  r.w1 = s.w1;
  r.len = s.len;
  return r;
}
__device__ __forceinline__ bool fnum(const uint8_t* st, uint32_t& p, uint64_t& v) {
  if (!CT_FNOINLINE) return fnum_i(st, p, v);
  const NumOut r = fnum_o(st, p);
  p = r.p;
  v = r.v;
  return r.ok != 0;
}
__device__ __forceinline__ bool fstr16(const uint8_t* st, uint32_t& p, Str& out) {
  if (!CT_FNOINLINE) return fstr16_i(st, p, out);
  const StrOut r = fstr16_o(st, p);
  p = r.p;
  out.w0 = r.w0;
  out.w1 = r.w1;
  out.len = r.len;
  return r.ok != 0;
}

// the comm name at p (after the quote): plain printable ASCII without '"' / '\\', at most
// kFNameMax bytes; key accumulated over 8-byte words
__device__ __forceinline__ bool fname(const uint8_t* st, uint32_t& p, uint32_t& len, uint64_t& key) {
  uint64_t h = 0x243F6A8885A308D3ull;
  for (uint32_t i = 0; i <= kFNameMax; i += 8) {
    const uint64_t x = st8(st, p + i);
    const uint64_t qx = x ^ 0x2222222222222222ull, bx = x ^ 0x5C5C5C5C5C5C5C5Cull;
    const uint64_t q = (qx - 0x0101010101010101ull) & ~qx & 0x8080808080808080ull;
    const uint64_t bad = (((bx - 0x0101010101010101ull) & ~bx) | (x - 0x2020202020202020ull) | x) &
                         0x8080808080808080ull;  // backslash, control, non-ASCII (a superset past the quote)
    if (q) {
      const uint32_t j = (uint32_t)(__ffsll((long long)q) - 1) >> 3;
      if (bad & ((1ull << (8 * j)) - 1)) return false;
      len = i + j;
      if (len > kFNameMax) return false;
      if (j) h = nk_mix(h, x & ((1ull << (8 * j)) - 1));
      key = nk_final(h, len);
      p += len + 1;
      return true;
    }
    if (bad) return false;
    h = nk_mix(h, x);
  }
  return false;
}

// the common head {"seq":N,"ts":N,"kind":"K","comm":"S","nranks":N,"rank":N,"dev":N: p
// moves to the kind-specific part
__device__ bool fast_prefix(const uint8_t* st, uint32_t& p, FLine& o, int& kind) {
  uint64_t seq, tsm, n, rank, dev;
  bool neg = false;
  Str kv;
  if (!flit(st, p, "{\"seq\":") || !fnum(st, p, seq) || !flit(st, p, ",\"ts\":")) return false;
  if (st[p] == '-') { neg = true; p++; }
  if (!fnum(st, p, tsm) || !flit(st, p, ",\"kind\":\"") || !fstr16(st, p, kv)) return false;
  kind = enum_of(K_KIND, kv);
  if (kind < 0 || !flit(st, p, ",\"comm\":\"") || !fname(st, p, o.nlen, o.key)) return false;
  o.nb = p - o.nlen - 1;
  if (!flit(st, p, ",\"nranks\":") || !fnum(st, p, n) || !flit(st, p, ",\"rank\":") || !fnum(st, p, rank) ||
      !flit(st, p, ",\"dev\":") || !fnum(st, p, dev))
    return false;
  if (neg ? tsm > (1ull << 63) : tsm >= (1ull << 63)) return false;
  if (n < 1 || n > 0xFFFF || rank >= n || dev > 0xFFFF) return false;
  o.r.seq = seq;
  o.r.nranks = (uint16_t)n;
  o.r.rank = (uint16_t)rank;
  o.r.dev = (uint16_t)dev;
  o.ts = neg ? (int64_t)(0ull - tsm) : (int64_t)tsm;
  return true;
}

// the kind-specific tail from p to the end of the line e: count, aux, aux2, kc, ad
__device__ bool fast_suffix(const uint8_t* st, uint32_t p, uint32_t e, int kind, uint32_t n, uint32_t rank,
                            ct_record& r) {
  uint64_t cnt, x;
  r.aux = 0;
  r.aux2 = 0;
  if (kind == CT_KIND_COLLECTIVE) {
    Str cv, av, dv;
    if (!flit(st, p, ",\"coll\":\"") || !fstr16(st, p, cv) || !flit(st, p, ",\"algo\":\"") || !fstr16(st, p, av) ||
        !flit(st, p, ",\"count\":") || !fnum(st, p, cnt) || !flit(st, p, ",\"dtype\":\"") || !fstr16(st, p, dv))
      return false;
    const int coll = enum_of(K_COLL, cv), algo = enum_of(K_ALGO, av), dt = enum_of(K_DTYPE, dv);
    if (coll < 0 || algo < 0 || dt < 0) return false;
    const bool rooted = coll == CT_COLL_BROADCAST || coll == CT_COLL_REDUCE;
    if (st[p] == ',') {
      if (!flit(st, p, ",\"root\":") || !fnum(st, p, x) || !rooted || x >= n) return false;
      r.aux = (uint16_t)x;
    } else if (rooted) {
      return false;
    }
    if ((algo == CT_ALGO_TREE || algo == CT_ALGO_COLLNET) && coll != CT_COLL_ALLREDUCE) return false;
    r.count = cnt;
    r.kc = (uint8_t)(kind | (coll << 3) | (rooted ? 1 << 6 : 0));
    r.ad = (uint8_t)(algo | (dt << 2));
  } else if (kind == CT_KIND_SEND || kind == CT_KIND_RECV) {
    Str dv;
    if (!flit(st, p, ",\"peer\":") || !fnum(st, p, x) || !flit(st, p, ",\"count\":") || !fnum(st, p, cnt) ||
        !flit(st, p, ",\"dtype\":\"") || !fstr16(st, p, dv))
      return false;
    const int dt = enum_of(K_DTYPE, dv);
    if (dt < 0 || x == rank || x >= n) return false;
    r.aux = (uint16_t)x;
    r.count = cnt;
    r.kc = (uint8_t)kind;
    r.ad = (uint8_t)(dt << 2);
  } else {
    Str ckv, sk, dk;
    uint64_t si, di;
    if (!flit(st, p, ",\"ckind\":\"") || !fstr16(st, p, ckv) || !flit(st, p, ",\"src\":{\"kind\":\"") ||
        !fstr16(st, p, sk) || !flit(st, p, ",\"idx\":") || !fnum(st, p, si) ||
        !flit(st, p, "},\"dst\":{\"kind\":\"") || !fstr16(st, p, dk) || !flit(st, p, ",\"idx\":") ||
        !fnum(st, p, di) || !flit(st, p, "},\"bytes\":") || !fnum(st, p, cnt))
      return false;
    const int ck = enum_of(K_CKIND, ckv);
    if (ck < 0) return false;
    const uint32_t s_k = CT_IS(sk, "host") ? 0u : CT_IS(sk, "gpu") ? 1u : 0xFFu;
    const uint32_t d_k = CT_IS(dk, "host") ? 0u : CT_IS(dk, "gpu") ? 1u : 0xFFu;
    const uint32_t want_s = ck == CT_CKIND_H2D ? 0 : 1, want_d = ck == CT_CKIND_D2H ? 0 : 1;
    if (s_k != want_s || d_k != want_d || si > 0xFFFF || di > 0xFFFF) return false;
    if ((want_s == 0 && si != 0) || (want_d == 0 && di != 0)) return false;
    if (ck == CT_CKIND_D2D && si == di) return false;
    r.aux = (uint16_t)si;
    r.aux2 = (uint16_t)di;
    r.count = cnt;
    r.kc = (uint8_t)kind;
    r.ad = (uint8_t)(ck << 6);
  }
  if (!flit(st, p, "}")) return false;
  return p == e;
}

__global__ void __launch_bounds__(kFThreads) k_fused(FArgs A) {
  extern __shared__ __align__(16) uint8_t st[];  // the stage: [st0, t1) and 32 zero-padded bytes
  __shared__ uint16_t msk[(kFM + kFT) / 16];
  __shared__ StOff tp[kFMaxLines + 1];             // line ends (stage offsets)
  __shared__ uint16_t rl[kFMaxLines];              // record index within the tile (0xFFFF: blank)
  __shared__ unsigned long long ckey[kFCache];
  __shared__ unsigned long long cref[kFCache];
  __shared__ int cslot[kFCache];
  __shared__ uint32_t cfirst[kFCache];
  __shared__ uint32_t clen[kFCache];
  __shared__ __align__(16) uint8_t cname[kFCache][kFNameMax];
  __shared__ unsigned long long s_t;
  __shared__ uint32_t s_prev, s_nl, s_abort;
  using BS = cub::BlockScan<uint32_t, kFThreads>;
  using BR = cub::BlockReduce<int, kFThreads>;
  __shared__ union {
    typename BS::TempStorage scan;
    typename BR::TempStorage red;
  } tmp;
  const int tid = threadIdx.x;

  __shared__ __align__(8) unsigned long long sbar;
  if (tid == 0) {
    s_t = atomicAdd(&A.ctl->ticket, 1ull);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&sbar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid < kFCache) { ckey[tid] = 0; cslot[tid] = -1; cfirst[tid] = 0xFFFFFFFFu; }
  __syncthreads();
  const uint64_t t = s_t;
  const uint64_t t0 = t * kFT, t1 = min(t0 + kFT, A.size);
  const uint64_t st0 = t0 > kFM ? t0 - kFM : 0;
  const uint32_t nst = (uint32_t)(t1 - st0);
  // the stage: one TMA bulk copy of the 16-byte multiple, the rest (and the zero padding
  // past the text) by the threads
#ifndef CT_FSTAGE_TMA
#define CT_FSTAGE_TMA 1
#endif
  const uint32_t nbk = CT_FSTAGE_TMA ? (uint32_t)(min(A.size, st0 + nst + 128) - st0) & ~15u : 0u;
  if (!CT_FSTAGE_TMA) {
    for (uint32_t v = tid; v < (nst + 128 + 15) / 16; v += kFThreads) {
      const uint64_t a = st0 + 16ull * v;
      if (a + 16 <= A.size) *reinterpret_cast<uint4*>(st + 16 * v) = *reinterpret_cast<const uint4*>(A.s + a);
      else for (int q = 0; q < 16; q++) st[16 * v + q] = a + q < A.size ? A.s[a + q] : 0;
    }
  }
  if (tid == 0 && nbk) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&sbar)), "r"(nbk)
                 : "memory");
    for (uint32_t o = 0; o < nbk; o += 16384)
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_u32(st + o)),
          "l"(A.s + st0 + o), "r"(min(16384u, nbk - o)), "r"(smem_u32(&sbar))
          : "memory");
  }
  if (CT_FSTAGE_TMA)
    for (uint32_t q = nbk + tid; q < nst + 128; q += kFThreads) st[q] = st0 + q < A.size ? A.s[st0 + q] : 0;
  __syncthreads();
  if (nbk) {
    uint32_t done = 0;
    while (!done)
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
          : "=r"(done)
          : "r"(smem_u32(&sbar))
          : "memory");
  }

  // ---- terminator masks (look-behind and owned groups)
  const uint32_t gb = (uint32_t)(t0 - st0) / 16, ng = (nst + 15) / 16;
  bool hi = false;
  for (uint32_t g = gb + tid; g < ng; g += kFThreads) {  // owned groups
    bool rare, h = false;
    uint32_t m = brk16f(st, 16 * g, st0, A.size, rare);
    if (rare) m = brk16s(st, 16 * g, st0, A.s, A.size, h);
    msk[g] = (uint16_t)m;
    hi |= h;
  }
  // the last terminator before the tile (the first owned line starts after it): warp 0
  // walks the look-behind back from the tile, 32 groups per step
  if (tid < 32) {
    int last = -1;
    for (int top = (int)gb - 1; top >= 0 && last < 0; top -= 32) {
      const int g = top - tid;
      uint32_t m = 0;
      if (g >= 0) {
        bool rare, h;
        m = brk16f(st, 16 * g, st0, A.size, rare);
        if (rare) m = brk16s(st, 16 * g, st0, A.s, A.size, h);
      }
      const int cand = m ? 16 * g + 31 - __clz(m) : -1;
      last = __reduce_max_sync(0xFFFFFFFFu, cand);
    }
    if (tid == 0) {
      s_abort = 0;
      if (last >= 0) s_prev = (uint32_t)last + blen_s(st, (uint32_t)last, nst);
      else if (st0 == 0) s_prev = 0;
      else { s_prev = 0; s_abort = 1; }  // a line longer than the look-behind
    }
  }
  if (__syncthreads_or(hi) && tid == 0) fb(A, FB_NONASCII);
  // ---- owned terminators in text order: 8 contiguous groups per thread
  uint32_t cnt = 0;
  const uint32_t g0 = gb + 8 * tid;
#pragma unroll
  for (int k = 0; k < 8; k++) cnt += g0 + k < ng ? __popc((uint32_t)msk[g0 + k]) : 0u;
  uint32_t off, tot;
  BS(tmp.scan).ExclusiveSum(cnt, off, tot);
  if (tot > (uint32_t)kFMaxLines) {
    if (tid == 0) { fb(A, FB_FALLBACK); s_abort = 1; }
  } else {
#pragma unroll
    for (int k = 0; k < 8; k++) {
      if (g0 + k >= ng) break;
      uint32_t m = msk[g0 + k];
      while (m) {
        const int j = __ffs(m) - 1;
        m &= m - 1;
        tp[off++] = (StOff)(16 * (g0 + k) + j);
      }
    }
  }
  __syncthreads();
  if (tid == 0) {
    uint32_t L = min(tot, (uint32_t)kFMaxLines);
    if (t1 == A.size && !s_abort) {  // the final line when the text does not end with a terminator
      const uint32_t le = L ? tp[L - 1] + blen_s(st, tp[L - 1], nst) : s_prev;
      if (le < nst && L < (uint32_t)kFMaxLines) tp[L++] = (StOff)nst;
      else if (le < nst) s_abort = 1;
    }
    s_nl = L;
    if (s_abort) fb(A, FB_FALLBACK);
  }
  __syncthreads();
  const uint32_t L = s_nl;
  const bool abort_ = s_abort != 0;
  auto lbeg = [&](uint32_t k) -> uint32_t { return k == 0 ? s_prev : tp[k - 1] + blen_s(st, tp[k - 1], nst); };

  // ---- blank test, record index within the tile (rounds of kFThreads lines, text order)
  uint32_t rbase = 0;
  for (uint32_t r0 = 0; r0 < L; r0 += kFThreads) {
    const uint32_t k = r0 + tid;
    uint32_t nb = 0;
    if (k < L && !abort_) {
      const uint32_t b = lbeg(k), e = tp[k];
      nb = b < e && !byte_blank(st[b]) ? 1u : (line_class(st, b, e, true) != 0 ? 1u : 0u);
    }
    uint32_t o, rt;
    BS(tmp.scan).ExclusiveSum(nb, o, rt);
    if (k < L) rl[k] = nb ? (uint16_t)(rbase + o) : (uint16_t)0xFFFF;
    rbase += rt;
    __syncthreads();
  }
  const uint32_t R = rbase;
  // per-tile counts; the tile's records go to its own block of kFMaxRecs temporary slots
  // (k_fscan / k_fcompact place them), so no tile waits for another
  if (tid == 0) {
    A.tcnt[2 * t] = L;
    A.tcnt[2 * t + 1] = R;
    if (R > (uint32_t)kFMaxRecs) { fb(A, FB_FALLBACK); s_abort = 1; }
  }
  __syncthreads();
  if (s_abort) return;

  // ---- parse: canonical lines here, the rest onto the slow list.  Per round of
  // kFThreads lines: the common head (thread = line), the name through the cache, then
  // the kind-specific tail with the lines regrouped by kind so that warps stay uniform.
  // The mask array is free now: per-line state between the two halves lives there.
  StOff* s_p = reinterpret_cast<StOff*>(msk);         // tail start
  uint16_t* s_n = reinterpret_cast<uint16_t*>(s_p + kFThreads);  // nranks, rank, dev, comm slot
  uint16_t* s_rank = s_n + kFThreads;
  uint16_t* s_dev = s_rank + kFThreads;
  uint16_t* s_cs = s_dev + kFThreads;
  uint8_t* s_kind = reinterpret_cast<uint8_t*>(s_cs + kFThreads);
  uint8_t* s_ce = s_kind + kFThreads;
  uint16_t* s_ord = reinterpret_cast<uint16_t*>(s_ce + kFThreads);  // regrouped position -> line of the round
  static_assert(kFThreads * (12 + (int)sizeof(StOff)) <= (int)sizeof(msk), "per-line state must fit the mask array");
  __shared__ uint32_t s_wcnt[3][kFThreads / 32];
  const int warp = tid >> 5, lane = tid & 31;
  for (uint32_t r0 = 0; r0 < L; r0 += kFThreads) {
    const uint32_t k = r0 + tid;
    FLine o;
    int kind = -1;
    bool ok = false;
    int ce = -1;       // cache entry
    bool mine = false; // this thread inserted the entry
    uint32_t p = 0;
    const bool line_here = k < L && rl[k] != 0xFFFF;
    if (line_here) {
      p = lbeg(k);
      ok = fast_prefix(st, p, o, kind);
      if (ok) {  // cache entry of the name (inserted by the first thread to see it)
        uint32_t i = (uint32_t)o.key & (kFCache - 1);
        for (int probe = 0; probe < kFCache; probe++, i = (i + 1) & (kFCache - 1)) {
          const unsigned long long old = atomicCAS(&ckey[i], 0ull, (unsigned long long)o.key);
          if (old == 0) { ce = (int)i; mine = true; break; }
          if (old == o.key) { ce = (int)i; break; }
        }
        if (ce < 0) ok = false;  // cache full: the slow list interns it
      }
    }
    __syncthreads();
    if (mine) {
      clen[ce] = o.nlen;
#pragma unroll
      for (int w = 0; w < (int)kFNameMax / 8; w++) {
        const uint32_t q = 8 * w;
        const uint64_t x = q < o.nlen ? st8(st, o.nb + q) : 0ull;
        const uint64_t mk = q + 8 <= o.nlen ? ~0ull : (q < o.nlen ? (1ull << (8 * (o.nlen - q))) - 1 : 0ull);
        *reinterpret_cast<uint64_t*>(&cname[ce][q]) = x & mk;
      }
      const uint64_t ref = (st0 + o.nb) | ((uint64_t)o.nlen << 40);
      cref[ce] = ref;
      cslot[ce] = table_slot(A, o.key, ref);
    }
    __syncthreads();
    if (ok) {  // the name must equal the entry's (a 64-bit key collision fails the load)
      bool same = clen[ce] == o.nlen && cslot[ce] >= 0;
#pragma unroll
      for (int w = 0; w < (int)kFNameMax / 8; w++) {
        const uint32_t q = 8 * w;
        const uint64_t x = q < o.nlen ? st8(st, o.nb + q) : 0ull;
        const uint64_t mk = q + 8 <= o.nlen ? ~0ull : (q < o.nlen ? (1ull << (8 * (o.nlen - q))) - 1 : 0ull);
        same = same && *reinterpret_cast<const uint64_t*>(&cname[ce][q]) == (x & mk);
      }
      if (!same) {
        if (cslot[ce] >= 0) fb(A, FB_COLLIDE);
        ok = false;
      }
    }
    if (line_here) {
      if (ok) {  // the head's fields; the tail comes below
        const uint64_t slot = t * kFMaxRecs + rl[k];
        reinterpret_cast<unsigned long long*>(A.trec + slot)[1] = o.r.seq;
        A.tts[slot] = o.ts;
        s_p[tid] = (StOff)p;
        s_n[tid] = o.r.nranks;
        s_rank[tid] = o.r.rank;
        s_dev[tid] = o.r.dev;
        s_cs[tid] = (uint16_t)cslot[ce];
        s_kind[tid] = (uint8_t)kind;
        s_ce[tid] = (uint8_t)ce;
      } else {  // (tile, line in tile, record in tile), byte range
        list_put(A, &A.ctl->n_slow, A.slow, 4, t << 32 | (uint64_t)k << 16 | rl[k], 0, st0 + lbeg(k), st0 + tp[k]);
      }
    }
    // regroup the lines with a valid head by kind class (collective, send/recv, copy)
    const int cls = ok ? (kind == CT_KIND_COLLECTIVE ? 0 : (kind <= CT_KIND_RECV ? 1 : 2)) : 3;
    unsigned bm[3];
#pragma unroll
    for (int c = 0; c < 3; c++) {
      bm[c] = __ballot_sync(0xFFFFFFFFu, cls == c);
      if (lane == 0) s_wcnt[c][warp] = __popc(bm[c]);
    }
    __syncthreads();
    uint32_t nsorted = 0, pos = 0;
#pragma unroll
    for (int c = 0; c < 3; c++)
      for (int w = 0; w < kFThreads / 32; w++) {
        const uint32_t v = s_wcnt[c][w];
        if (c < cls || (c == cls && w < warp)) pos += v;
        nsorted += v;
      }
    if (cls < 3) s_ord[pos + __popc(bm[cls] & ((1u << lane) - 1))] = (uint16_t)tid;
    __syncthreads();
    if ((uint32_t)tid < nsorted) {
      const uint32_t i = s_ord[tid], kk = r0 + i;
      ct_record rec;
      const int kd = s_kind[i];
      if (fast_suffix(st, s_p[i], tp[kk], kd, s_n[i], s_rank[i], rec)) {
        const uint64_t slot = t * kFMaxRecs + rl[kk];
        atomicMin(&cfirst[s_ce[i]], (uint32_t)rl[kk]);
        reinterpret_cast<unsigned long long*>(A.trec + slot)[0] = rec.count;
        uint4 w;
        w.x = s_cs[i];
        w.y = (uint32_t)s_n[i] | ((uint32_t)s_rank[i] << 16);
        w.z = (uint32_t)s_dev[i] | ((uint32_t)rec.aux << 16);
        w.w = (uint32_t)rec.aux2 | ((uint32_t)rec.kc << 16) | ((uint32_t)rec.ad << 24);
        reinterpret_cast<uint4*>(A.trec + slot)[1] = w;
      } else {
        list_put(A, &A.ctl->n_slow, A.slow, 4, t << 32 | (uint64_t)kk << 16 | rl[kk], 0, st0 + lbeg(kk), st0 + tp[kk]);
      }
    }
    __syncthreads();
  }
  __syncthreads();
  if (tid < kFCache && ckey[tid] && cslot[tid] >= 0 && cfirst[tid] != 0xFFFFFFFFu) {
    atomicMin(&A.gfirst[cslot[tid]], t << 16 | cfirst[tid]);  // (tile, record in tile): text order
    list_put(A, &A.ctl->n_verify, A.verify, 2, (uint64_t)cslot[tid], cref[tid], 0, 0);
  }
}

// tiles in text order: first line number and first record slot of every tile
constexpr int kScanThreads = 512;
__global__ void __launch_bounds__(kScanThreads) k_fscan(FArgs A) {
  constexpr int kI = 8;
  using Scan = cub::BlockScan<unsigned long long, kScanThreads>;
  __shared__ typename Scan::TempStorage tmp;
  if (A.ctl->flags & FB_FALLBACK) return;
  unsigned long long bl = 0, br = 0;
  for (uint64_t c0 = 0; c0 < A.ntiles; c0 += kScanThreads * kI) {
    const uint64_t t0 = c0 + (uint64_t)threadIdx.x * kI;
    unsigned long long l[kI], r[kI], ol[kI], orr[kI], sl, sr;
#pragma unroll
    for (int q = 0; q < kI; q++) {
      const bool in = t0 + q < A.ntiles;
      const uint2 c = in ? reinterpret_cast<const uint2*>(A.tcnt)[t0 + q] : make_uint2(0, 0);
      l[q] = c.x;
      r[q] = c.y;
    }
    Scan(tmp).ExclusiveSum(l, ol, sl);
    __syncthreads();
    Scan(tmp).ExclusiveSum(r, orr, sr);
    __syncthreads();
#pragma unroll
    for (int q = 0; q < kI; q++)
      if (t0 + q < A.ntiles) reinterpret_cast<ulonglong2*>(A.toff)[t0 + q] = make_ulonglong2(bl + ol[q], br + orr[q]);
    bl += sl;
    br += sr;
  }
  if (threadIdx.x == 0) {
    A.ctl->n_lines = bl;
    A.ctl->n_recs = br;
    if (br > A.cap) fb(A, FB_FALLBACK);
  }
}

// per-call state: control block, name table (keys 0, first records ~0), side buffer use
__global__ void k_finit(FArgs A) {
  const uint32_t i0 = blockIdx.x * blockDim.x + threadIdx.x;
  for (uint32_t i = i0; i < kFTable; i += gridDim.x * blockDim.x) {
    A.gkey[i] = 0;
    A.gfirst[i] = ~0ull;
  }
  if (i0 < sizeof(FCtl) / sizeof(unsigned long long)) reinterpret_cast<unsigned long long*>(A.ctl)[i0] = 0;
  if (i0 == 0) *A.side.used = 0;
}

// slow list: the generic parser (escapes decoded) straight from the text, into the
// tile's temporary slot
__global__ void __launch_bounds__(kParseThreads) k_fslow(FArgs A, bool aligned) {
  __shared__ uint64_t fields[K_N * kParseThreads];
  if (A.ctl->flags & FB_FALLBACK) return;
  const uint64_t n = min(*reinterpret_cast<volatile unsigned long long*>(&A.ctl->n_slow), (unsigned long long)A.lcap);
  const uint64_t wl = aligned && A.size > 32 ? A.size - 8 : 0;
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n; j += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t w0 = A.slow[4 * j], b = A.slow[4 * j + 2], e = A.slow[4 * j + 3];
    const uint64_t tt = w0 >> 32, k = (w0 >> 16) & 0xFFFF, lr = w0 & 0xFFFF;
    const uint64_t tmp_slot = tt * kFMaxRecs + lr;
    LineOut o;
    const uint8_t st = parse_line<true>(A.s, b, e, aligned, wl, fields + threadIdx.x, kParseThreads, A.side, o);
    if (st == L_OK) {
      const uint32_t len = (uint32_t)(o.comm >> 40);
      const uint64_t key = name_key_bytes(name_ptr(A.s, A.side.buf, o.comm), len);
      const int gs = table_slot(A, key, o.comm);
      if (gs >= 0) {
        atomicMin(&A.gfirst[gs], (unsigned long long)(tt << 16 | lr));
        list_put(A, &A.ctl->n_verify, A.verify, 2, (uint64_t)gs, o.comm, 0, 0);
      }
      o.r.comm = gs >= 0 ? (uint32_t)gs : 0u;
      A.trec[tmp_slot] = o.r;
      A.tts[tmp_slot] = o.ts;
    } else {  // the caller reads it (a blank one is dropped there)
      A.trec[tmp_slot] = ct_record{};
      A.tts[tmp_slot] = 0;
      list_put(A, &A.ctl->n_defer, A.defer, 4, A.toff[2 * tt] + k + 1, A.toff[2 * tt + 1] + lr, b, e - b);
    }
  }
}

// every (table slot, name) pair seen: byte-equal to the slot's name
__global__ void k_fverify(FArgs A) {
  const uint64_t n = min(*reinterpret_cast<volatile unsigned long long*>(&A.ctl->n_verify), (unsigned long long)A.lcap);
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n; j += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t gs = A.verify[2 * j], a = A.verify[2 * j + 1], h = A.gname[gs];
    if (a == h) continue;
    const uint32_t la = (uint32_t)(a >> 40), lh = (uint32_t)(h >> 40);
    bool same = la == lh;
    const uint8_t *na = name_ptr(A.s, A.side.buf, a), *nh = name_ptr(A.s, A.side.buf, h);
    for (uint32_t q = 0; same && q < la; q++) same = na[q] == nh[q];
    if (!same) fb(A, FB_COLLIDE);
  }
}

// one CTA: table slots in first-seen order -> comm ids, comm rows and names
constexpr int kFinThreads = 1024;
__global__ void __launch_bounds__(kFinThreads) k_ffinal(FArgs A) {
  using Scan = cub::BlockScan<unsigned long long, kFinThreads>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ unsigned long long ufirst[kFMaxNames];
  __shared__ uint32_t uslot[kFMaxNames];
  __shared__ uint32_t uorder[kFMaxNames];  // rank -> entry
  __shared__ unsigned int n_used;
  const int tid = threadIdx.x;
  if (tid == 0) n_used = 0;
  __syncthreads();
  if (A.ctl->flags & FB_FALLBACK) return;
  const uint32_t nins = min(A.ctl->n_names, kFMaxNames);
  for (uint32_t q = tid; q < nins; q += kFinThreads) {
    const uint32_t i = A.gused[q];
    // a name whose lines all left the template path and were deferred has no first record
    if (A.gfirst[i] == ~0ull) continue;
    const unsigned int u = atomicAdd(&n_used, 1u);
    if (u < kFMaxNames) { ufirst[u] = A.gfirst[i]; uslot[u] = i; }
  }
  __syncthreads();
  const uint32_t nu = n_used;
  if (nu > kFMaxNames) {
    if (tid == 0) fb(A, FB_FALLBACK);
    return;
  }
  // first-seen order: the rank of each (tile, record in tile) key among the (distinct) keys
  for (uint32_t i = tid; i < nu; i += kFinThreads) {
    const unsigned long long k = ufirst[i];
    uint32_t r = 0;
    for (uint32_t q = 0; q < nu; q++) r += ufirst[q] < k ? 1u : 0u;
    uorder[r] = i;
  }
  __syncthreads();
  constexpr int kI = kFMaxNames / kFinThreads;
  unsigned long long len[kI], off[kI];
#pragma unroll
  for (int q = 0; q < kI; q++) {
    const uint32_t r = kI * tid + q;
    len[q] = r < nu ? (A.gname[uslot[uorder[r]]] >> 40) : 0ull;
  }
  unsigned long long tot;
  Scan(tmp).ExclusiveSum(len, off, tot);
  if (tid == 0) { A.ctl->name_bytes = tot; A.ctl->n_used = nu; }
  if (tot > kFNameCap) {
    if (tid == 0) fb(A, FB_FALLBACK);
    return;
  }
#pragma unroll
  for (int q = 0; q < kI; q++) {
    const uint32_t r = kI * tid + q;
    if (r >= nu) continue;
    const uint32_t e = uorder[r], gs = uslot[e];
    const unsigned long long k = ufirst[e];
    A.gid[gs] = r;
    A.comm_rows[3 * r] = A.toff[2 * (k >> 16) + 1] + (k & 0xFFFF);
    A.comm_rows[3 * r + 1] = off[q];
    A.comm_rows[3 * r + 2] = len[q];
    const uint8_t* nm = name_ptr(A.s, A.side.buf, A.gname[gs]);
    for (uint64_t b = 0; b < len[q]; b++) A.names[off[q] + b] = nm[b];
  }
}

// tiles' temporary records -> final positions, comm field: table slot -> comm id
__global__ void __launch_bounds__(256) k_fcompact(FArgs A) {
  if (A.ctl->flags & FB_FALLBACK) return;
  for (uint64_t tt = blockIdx.x; tt < A.ntiles; tt += gridDim.x) {
    const uint32_t R = A.tcnt[2 * tt + 1];
    const uint64_t dst = A.toff[2 * tt + 1], src = tt * kFMaxRecs;
    for (uint32_t i = threadIdx.x; i < R; i += blockDim.x) {
      ct_record r = A.trec[src + i];
      r.comm = A.gid[r.comm & (kFTable - 1)];
      A.recs[dst + i] = r;
      A.ts[dst + i] = A.tts[src + i];
    }
  }
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

// The fused single pass (k_fused + slow list + name table finalisation): 0 done, 1 the
// text needs the multi-pass pipeline, else an error status.
int run_fused(ct_jsonl* j, const uint8_t* s, uint64_t size, Pool& pool, cudaEvent_t done) {
  const uint64_t ntiles = (size + kFT - 1) / kFT;
  // record slots: a valid trace line is > 90 bytes; texts whose non-blank lines average
  // fewer than 64 bytes overflow and take the multi-pass pipeline
  const uint64_t cap = size / 64 + 64;
  if (cap >= (1ull << 32)) return 1;
  FArgs A{};
  A.s = s;
  A.size = size;
  A.ntiles = ntiles;
  A.cap = cap;
  A.lcap = std::min<uint64_t>(cap, kFListCap);
  // one stream-ordered allocation carved into every array (a single pool call per text)
  const uint64_t side_cap = std::min<uint64_t>(16ull << 20, std::max<uint64_t>(size, 1024));
  uint8_t* side = nullptr;
  unsigned long long* side_used = nullptr;
  uint8_t* base = nullptr;
  uint64_t used = 0;
  auto carve = [&](auto*& ptr, uint64_t n) {
    used = (used + 255) & ~255ull;
    ptr = reinterpret_cast<std::remove_reference_t<decltype(ptr)>>(base + used);
    used += n * sizeof(*ptr);
  };
  for (int pass = 0; pass < 2; pass++) {
    used = 0;
    carve(A.ctl, 1);
    carve(A.tcnt, 2 * ntiles);
    carve(A.toff, 2 * ntiles);
    carve(A.trec, ntiles * kFMaxRecs);
    carve(A.tts, ntiles * kFMaxRecs);
    carve(A.recs, cap);
    carve(A.ts, cap);
    carve(A.gkey, kFTable);
    carve(A.gname, kFTable);
    carve(A.gfirst, kFTable);
    carve(A.gid, kFTable);
    carve(A.gused, kFMaxNames);
    carve(A.slow, 4 * A.lcap);
    carve(A.defer, 4 * A.lcap);
    carve(A.verify, 2 * A.lcap);
    carve(A.comm_rows, 3 * kFMaxNames);
    carve(A.names, kFNameCap);
    carve(side, side_cap);
    carve(side_used, 1);
    if (pass == 0) {
      base = pool.alloc<uint8_t>(used);
      JL_NN(base);
    }
  }
  A.side = Side{side, side_used, side_cap};
  k_finit<<<16, 256, 0, j->st>>>(A);
  static bool attr_set[64] = {};  // the attribute lives in each device's context
  if (j->device < 0 || j->device >= 64 || !attr_set[j->device]) {
    JL_TRY(cudaFuncSetAttribute(k_fused, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kFStage));
    if (j->device >= 0 && j->device < 64) attr_set[j->device] = true;
  }
  const bool dbg = getenv("CT_JSONL_DEBUG") != nullptr;
  cudaEvent_t ev[6];
  if (dbg)
    for (auto& x : ev) cudaEventCreate(&x);
  if (dbg) cudaEventRecord(ev[0], j->st);
  k_fused<<<(unsigned)ntiles, kFThreads, kFStage, j->st>>>(A);
  k_fscan<<<1, kScanThreads, 0, j->st>>>(A);
  if (dbg) cudaEventRecord(ev[1], j->st);
  k_fslow<<<148 * 4, kParseThreads, 0, j->st>>>(A, true);
  if (dbg) cudaEventRecord(ev[2], j->st);
  k_fverify<<<148, 256, 0, j->st>>>(A);
  if (dbg) cudaEventRecord(ev[3], j->st);
  k_ffinal<<<1, kFinThreads, 0, j->st>>>(A);
  if (dbg) cudaEventRecord(ev[4], j->st);
  k_fcompact<<<(unsigned)std::min<uint64_t>(ntiles, 148 * 16), 256, 0, j->st>>>(A);
  if (dbg) cudaEventRecord(ev[5], j->st);
  JL_TRY(cudaGetLastError());
  JL_TRY(cudaEventRecord(done, j->st));  // end of the device work (the status read below is host I/O)
  if (dbg) {
    cudaEventSynchronize(ev[5]);
    float f[5];
    for (int q = 0; q < 5; q++) cudaEventElapsedTime(&f[q], ev[q], ev[q + 1]);
    fprintf(stderr, "ct_jsonl fused ms: fused+scan %.3f slow %.3f verify %.3f final %.3f compact %.3f\n", f[0], f[1], f[2],
            f[3], f[4]);
    for (auto& x : ev) cudaEventDestroy(x);
  }
  FCtl c{};
  JL_TRY(cudaMemcpyAsync(&c, A.ctl, sizeof(FCtl), cudaMemcpyDeviceToHost, j->st));
  JL_TRY(cudaStreamSynchronize(j->st));
  if (c.flags & FB_FALLBACK) return 1;
  if (c.flags & FB_COLLIDE) {
    j->err = "comm name hash collision (64-bit name key): two different names share a key";
    return CT_ERR_CAPACITY;
  }
  if (c.n_recs >= (1ull << 32)) { j->err = "more than 2^32 - 1 records in one text"; return CT_ERR_CAPACITY; }
  j->info.n_lines = c.n_lines;
  j->info.n_records = c.n_recs;
  j->info.n_deferred = c.n_defer;
  j->info.n_comms = c.n_used;
  j->info.comm_bytes = c.name_bytes;
  j->info.non_ascii = (c.flags & FB_NONASCII) ? 1 : 0;
  j->info.n_slow = c.n_slow;
  if (getenv("CT_JSONL_DEBUG") && c.n_slow) {  // the first slow lines (1-based numbers) on stderr
    uint64_t rows[4 * 8];
    const uint64_t k = std::min<uint64_t>(c.n_slow, 8);
    JL_TRY(cudaMemcpy(rows, A.slow, 4 * k * sizeof(uint64_t), cudaMemcpyDeviceToHost));
    for (uint64_t i = 0; i < k; i++)
      fprintf(stderr, "ct_jsonl slow line %llu (bytes %llu..%llu)\n", (unsigned long long)rows[4 * i],
              (unsigned long long)rows[4 * i + 2], (unsigned long long)rows[4 * i + 3]);
  }
  j->recs = A.recs;
  j->ts = A.ts;
  j->deferred_rows = A.defer;
  j->comm_rows = A.comm_rows;
  j->names = A.names;
  return 0;
}

// Host <-> device through pinned staging.  A pageable cudaMemcpy goes through the
// driver's bounce buffers at a fraction of the link rate; large transfers instead stream
// through two pinned 16 MB slots per device: host threads copy chunk k + 1 into (or out
// of) one slot while the DMA engine moves chunk k through the other.
constexpr uint64_t kStageChunk = 16ull << 20;

struct Staging {  // per device, created on first use and reused across calls
  uint8_t* pinned = nullptr;
  cudaEvent_t ev[2];
  std::mutex mu;
};

Staging* staging_for(int device) {
  constexpr int kDevs = 64;
  static Staging st_of[kDevs];
  static std::mutex init_mu;
  if (device < 0 || device >= kDevs) return nullptr;
  Staging& S = st_of[device];
  std::lock_guard<std::mutex> lock(init_mu);
  if (!S.pinned) {
    uint8_t* p = nullptr;
    if (cudaHostAlloc(&p, 2 * kStageChunk, cudaHostAllocPortable) != cudaSuccess) return nullptr;
    if (cudaEventCreateWithFlags(&S.ev[0], cudaEventDisableTiming) != cudaSuccess ||  // on `device` (the caller's)
        cudaEventCreateWithFlags(&S.ev[1], cudaEventDisableTiming) != cudaSuccess) {
      cudaFreeHost(p);
      return nullptr;
    }
    S.pinned = p;
  }
  return &S;
}

int stage_threads() {
  static const int env = getenv("CT_JSONL_UPLOAD_THREADS") ? atoi(getenv("CT_JSONL_UPLOAD_THREADS")) : 8;
  return std::max(1, std::min(env, omp_get_max_threads()));
}

void par_copy(uint8_t* dst, const uint8_t* src, uint64_t len, int nthr) {
  const uint64_t part = (len + nthr - 1) / nthr;
#pragma omp parallel for num_threads(nthr) schedule(static)
  for (int q = 0; q < nthr; q++) {
    const uint64_t a = (uint64_t)q * part;
    if (a < len) memcpy(dst + a, src + a, std::min(part, len - a));
  }
}

bool staged(uint64_t size, uint64_t min_size) {
  return size >= min_size && !getenv("CT_JSONL_PAGEABLE");
}

int upload_text(ct_jsonl* j, uint8_t* d, const uint8_t* text, uint64_t size) {
  Staging* S = staged(size, 4 * kStageChunk) ? staging_for(j->device) : nullptr;
  if (!S) {
    JL_TRY(cudaMemcpyAsync(d, text, size, cudaMemcpyHostToDevice, j->st));
    return 0;
  }
  std::lock_guard<std::mutex> lock(S->mu);
  const int nthr = stage_threads();
  uint64_t k = 0;
  for (uint64_t off = 0; off < size; off += kStageChunk, k++) {
    const int slot = (int)(k & 1);
    if (k >= 2) JL_TRY(cudaEventSynchronize(S->ev[slot]));  // the slot's previous DMA is done
    const uint64_t len = std::min(kStageChunk, size - off);
    uint8_t* stg = S->pinned + slot * kStageChunk;
    par_copy(stg, text + off, len, nthr);
    JL_TRY(cudaMemcpyAsync(d + off, stg, len, cudaMemcpyHostToDevice, j->st));
    JL_TRY(cudaEventRecord(S->ev[slot], j->st));
  }
  // the staging slots are reused by the next call: their last DMAs must finish first
  JL_TRY(cudaEventSynchronize(S->ev[(k - 1) & 1]));
  return 0;
}

// Device -> pageable host (the timestamps): DMA chunk k + 1 into one slot while host
// threads copy chunk k out of the other.
int download(ct_jsonl* j, uint8_t* host, const uint8_t* d, uint64_t size) {
  Staging* S = staged(size, kStageChunk) ? staging_for(j->device) : nullptr;
  if (!S) {
    JL_TRY(cudaMemcpyAsync(host, d, size, cudaMemcpyDeviceToHost, j->st));
    JL_TRY(cudaStreamSynchronize(j->st));
    return 0;
  }
  std::lock_guard<std::mutex> lock(S->mu);
  const int nthr = stage_threads();
  const uint64_t nk = (size + kStageChunk - 1) / kStageChunk;
  auto issue = [&](uint64_t k) -> cudaError_t {
    const uint64_t off = k * kStageChunk, len = std::min(kStageChunk, size - off);
    cudaError_t e = cudaMemcpyAsync(S->pinned + (k & 1) * kStageChunk, d + off, len, cudaMemcpyDeviceToHost, j->st);
    return e == cudaSuccess ? cudaEventRecord(S->ev[k & 1], j->st) : e;
  };
  JL_TRY(issue(0));
  for (uint64_t k = 0; k < nk; k++) {
    if (k + 1 < nk) JL_TRY(issue(k + 1));  // the other slot: its copy-out (chunk k - 1) is done
    JL_TRY(cudaEventSynchronize(S->ev[k & 1]));
    const uint64_t off = k * kStageChunk;
    par_copy(host + off, S->pinned + (k & 1) * kStageChunk, std::min(kStageChunk, size - off), nthr);
  }
  return 0;
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
    if (int e = upload_text(j, d, text, size)) return e;
    s = d;
  }
  JL_TRY(cudaEventRecord(e0, j->st));
  if (getenv("CT_JSONL_DEBUG")) {
    cudaEventSynchronize(e0);
    fprintf(stderr, "ct_jsonl: text on the device\n");
  }
  const bool multipass = getenv("CT_JSONL_MULTIPASS") != nullptr;  // A/B and tests
  if (size > 0 && (reinterpret_cast<uintptr_t>(s) & 15) == 0 && !multipass) {
    const int rc = run_fused(j, s, size, pool, e1);
    if (rc != 1) {
      JL_TRY(cudaEventSynchronize(e1));
      float ms = 0;
      JL_TRY(cudaEventElapsedTime(&ms, e0, e1));
      j->info.ms_device = ms;
      j->info.fused = 1;
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
      return rc;
    }
    j->info = ct_jsonl_info{};  // the multi-pass pipeline from the start
  }
  uint64_t* scal = pool.alloc<uint64_t>(8);  // device scalars
  JL_NN(scal);
  JL_TRY(cudaMemsetAsync(scal, 0, 8 * sizeof(uint64_t), j->st));
  unsigned int* flags = reinterpret_cast<unsigned int*>(scal + 6);

  // 1. terminators: per-tile counts, tile offsets, ordered positions
  thrust::counting_iterator<uint64_t> idx(0);
  const bool aligned = (reinterpret_cast<uintptr_t>(s) & 15) == 0;
  const uint64_t n_tiles = (size + kTileBytes - 1) / kTileBytes;
  uint32_t* tile_cnt = pool.alloc<uint32_t>(n_tiles + 1);
  uint64_t* tile_off = pool.alloc<uint64_t>(n_tiles + 1);
  JL_NN(tile_cnt); JL_NN(tile_off);
  JL_TRY(cudaMemsetAsync(tile_cnt + n_tiles, 0, sizeof(uint32_t), j->st));
  if (n_tiles) k_brk_count<<<(unsigned)n_tiles, kTileThreads, 0, j->st>>>(s, size, aligned, tile_cnt, flags);
  JL_TRY(cudaGetLastError());
  size_t tb = 0;
  JL_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tb, tile_cnt, tile_off, (int64_t)n_tiles + 1, j->st));
  void* t = pool.temp(tb);
  JL_NN(t);
  JL_TRY(cub::DeviceScan::ExclusiveSum(t, tb, tile_cnt, tile_off, (int64_t)n_tiles + 1, j->st));
  uint64_t nb = 0;
  JL_TRY(cudaMemcpyAsync(&nb, tile_off + n_tiles, sizeof(uint64_t), cudaMemcpyDeviceToHost, j->st));
  JL_TRY(cudaStreamSynchronize(j->st));
  uint64_t* brk = pool.alloc<uint64_t>(nb);
  JL_NN(brk);
  if (nb) k_brk_write<<<(unsigned)n_tiles, kTileThreads, 0, j->st>>>(s, size, aligned, tile_off, brk);
  JL_TRY(cudaGetLastError());
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

  // 2. parse, one thread per line
  uint8_t* status = pool.alloc<uint8_t>(n_lines + 1);  // + a blank terminator for the scan
  LineOut* lo = pool.alloc<LineOut>(n_lines);
  uint64_t* ridx = pool.alloc<uint64_t>(n_lines + 1);
  JL_NN(status); JL_NN(lo); JL_NN(ridx);
  JL_TRY(cudaMemsetAsync(status + n_lines, L_BLANK, 1, j->st));
  // decoded (escaped) comm names: up to 16 MB, the rest of such lines are read on the host
  const uint64_t side_cap = std::min<uint64_t>(16ull << 20, std::max<uint64_t>(size, 1024));
  uint8_t* side = pool.alloc<uint8_t>(side_cap);
  JL_NN(side);
  if (n_lines) {
    JL_TRY(cudaFuncSetAttribute(k_parse, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(kStage + kStageSlack)));
    k_parse<<<(unsigned)((n_lines + kParseThreads - 1) / kParseThreads), kParseThreads, kStage + kStageSlack, j->st>>>(
        s, size, aligned, brk, nb, n_lines, status, lo, Side{side, reinterpret_cast<unsigned long long*>(scal + 4),
                                                             side_cap});
  }
  JL_TRY(cudaGetLastError());
  if (n_lines) {  // lines with escapes: compacted, parsed by the escape-decoding instantiation
    uint64_t* elines = pool.alloc<uint64_t>(n_lines);
    JL_NN(elines);
    tb = 0;
    IsEsc ise{status};
    JL_TRY(cub::DeviceSelect::If(nullptr, tb, idx, elines, scal + 3, (int64_t)n_lines, ise, j->st));
    t = pool.temp(tb);
    JL_NN(t);
    JL_TRY(cub::DeviceSelect::If(t, tb, idx, elines, scal + 3, (int64_t)n_lines, ise, j->st));
    uint64_t ne = 0;
    JL_TRY(cudaMemcpyAsync(&ne, scal + 3, sizeof(uint64_t), cudaMemcpyDeviceToHost, j->st));
    JL_TRY(cudaStreamSynchronize(j->st));
    if (ne)
      k_parse_esc<<<(unsigned)((ne + kParseThreads - 1) / kParseThreads), kParseThreads, 0, j->st>>>(
          s, size, aligned, brk, nb, elines, scal + 3, status, lo,
          Side{side, reinterpret_cast<unsigned long long*>(scal + 4), side_cap});
    JL_TRY(cudaGetLastError());
  }
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
    k_verify<<<g, 256, 0, j->st>>>(n_rec, keys2, vals2, seg, seg_coff, coff, s, side, flags);
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
    k_names<<<grid_for(u), 256, 0, j->st>>>(u, seg_order, seg_first, seg_coff, name_off, s, side, j->names,
                                            j->comm_rows);
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
  if (size >= (1ull << 39)) { j->err = "text larger than 2^39 bytes"; return CT_ERR_ARGUMENT; }
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) {  // keep freed blocks in the stream-ordered pool between calls
    cudaMemPool_t mp;
    if (cudaDeviceGetDefaultMemPool(&mp, device) == cudaSuccess) {
      uint64_t keep = ~0ull;
      cudaMemPoolSetAttribute(mp, cudaMemPoolAttrReleaseThreshold, &keep);
    }
  }
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&j->st, cudaStreamNonBlocking);
  if (e != cudaSuccess) { j->err = cudaGetErrorString(e); return CT_ERR_CUDA; }
  const int rc = run(j, reinterpret_cast<const uint8_t*>(text), size, on_device);
  if (info) *info = j->info;
  return rc;
}

int ct_jsonl_records(ct_jsonl* j, ct_record* dev_out, int64_t* host_ts) {
  if (!j) return CT_ERR_ARGUMENT;
  const uint64_t n = j->info.n_records;
  cudaError_t e = cudaSetDevice(j->device);  // the staging events belong to the device
  if (e == cudaSuccess && n && dev_out) e = cudaMemcpyAsync(dev_out, j->recs, n * sizeof(ct_record), cudaMemcpyDeviceToDevice, j->st);
  if (e != cudaSuccess) { j->err = cudaGetErrorString(e); return CT_ERR_CUDA; }
  if (n && host_ts) {
    if (download(j, reinterpret_cast<uint8_t*>(host_ts), reinterpret_cast<const uint8_t*>(j->ts),
                 n * sizeof(int64_t)))
      return CT_ERR_CUDA;
  }
  e = cudaStreamSynchronize(j->st);
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
  if (j->info.fused && n > 1) {  // appended in completion order: line order for the caller
    std::vector<std::array<uint64_t, 4>> v(n);
    memcpy(v.data(), rows, 4 * n * sizeof(uint64_t));
    std::sort(v.begin(), v.end(), [](const auto& a, const auto& b) { return a[0] < b[0]; });
    memcpy(rows, v.data(), 4 * n * sizeof(uint64_t));
  }
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
