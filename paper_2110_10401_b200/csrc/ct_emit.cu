// Emit mode: per-record transfer lists for the decompose_* API (decompose.py:130-406).
//
// Two passes over canonical instance blocks: pass 0 counts each record's transfers,
// an exclusive prefix sum (CUB) assigns every record its output slots, pass 1 writes
// rows {instance/record index, src, dst, bytes_lo, bytes_hi, src rank, sub} (endpoint:
// gpu id, -1 net, -2 host; sub = destination rank for collective edges, 0/1 for the
// collnet dev->net / net->dev transfers).  The expansion is the same rank-attributed code the accumulate
// kernel runs (ct_expand.cuh), so the acceptance-grid parity tests exercise it.
#include "ct_expand.cuh"

namespace ct {

namespace {

constexpr int kEmitCols = 7;

struct GDev {
  const ct_record* g;
  __device__ __forceinline__ uint32_t dev_of(uint64_t i) const { return g[i].dev; }
};

struct EmitSink {
  uint32_t flags;
  uint32_t count;
  int64_t* rows;      // pass 1 output (already offset to this record's slots)
  int64_t id;
  int64_t rank;
  __device__ __forceinline__ void stat(int, unsigned __int128) {}
  __device__ __forceinline__ void edge(int, int src, int dst, unsigned __int128 bytes, int sub = 0) {
    if (rows) {
      int64_t* o = rows + kEmitCols * (int64_t)count;
      o[0] = id;
      o[5] = rank;
      o[6] = sub;
      o[1] = src == -2 ? -1 : (src == -1 ? -2 : src);
      o[2] = dst == -2 ? -1 : (dst == -1 ? -2 : dst);
      o[3] = (int64_t)(uint64_t)bytes;
      o[4] = (int64_t)(uint64_t)(bytes >> 64);
    }
    count++;
  }
};

__global__ void k_emit(const ct_record* recs, uint64_t n, ExpandParams ex, uint32_t* counts,
                       const uint64_t* offsets, int64_t* rows, unsigned int* flags) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const Rec rc = load_global(recs + i);
    const Rec rc0 = load_global(recs + i);
    EmitSink sink{0, 0, rows ? rows + kEmitCols * offsets[i] : nullptr, (int64_t)i, (int64_t)rc0.rank};
    const int kind = rc.kind();
    if (kind == CT_KIND_COLLECTIVE) {
      const uint64_t head = i - rc.rank;
      sink.id = (int64_t)head;
      GDev v{recs};
      if ((rc.count >> 40) == 0) expand_collective<uint64_t>(ex, v, sink, rc, head);
      else expand_collective<unsigned __int128>(ex, v, sink, rc, head);
    } else if (kind == CT_KIND_SEND) {
      if (i + 1 < n) {
        const Rec q = load_global(recs + i + 1);
        const unsigned __int128 nb = (unsigned __int128)rc.count * (unsigned)dtype_width(rc.dtype());
        if (q.dev != rc.dev) sink.edge(CT_T_SENDRECV, (int)rc.dev, (int)q.dev, nb);
      }
    } else if (kind >= CT_KIND_MEMCPY) {
      const int ck = rc.ckind();
      sink.edge(0, ck == CT_CKIND_H2D ? -1 : (int)rc.aux, ck == CT_CKIND_D2H ? -1 : (int)rc.aux2,
                (unsigned __int128)rc.count);
    }
    if (!rows) counts[i] = sink.count;
    if (sink.flags) atomicOr(flags, sink.flags);
  }
}

}  // namespace

void launch_emit(const ct_record* recs, uint64_t n, const ExpandParams& ex, uint32_t* counts,
                 const uint64_t* offsets, int64_t* rows, int pass, unsigned int* flags, cudaStream_t st) {
  if (!n) return;
  uint64_t g = (n + 255) / 256;
  if (g > 8192) g = 8192;
  k_emit<<<(unsigned)g, 256, 0, st>>>(recs, n, ex, counts, pass ? offsets : nullptr, pass ? rows : nullptr, flags);
}

}  // namespace ct
