// Counting canonicaliser for capture-layout (rank-interleaved) traces; see ct_canon.cu.
#pragma once
#include "ct_exact.cuh"

namespace ct {

// count_canonicalize's return value when the trace is outside its scope (too many keys,
// nranks disagreement, malformed records): the caller takes the exact path instead
constexpr int kCanonUnsupported = 0x7FFF0002;

// Fills res->canon / m / n_incomplete / n_unmatched_* / launches and *max_dev (over ALL
// records) like exact_canonicalize; returns 0, kCanonUnsupported or a cudaError_t.
int count_canonicalize(const ct_record* recs, uint64_t n, uint32_t n_comms, int num_sms, cudaStream_t st,
                       ExactResult* res, int* max_dev);

// ---- multi-GPU: canonicalise globally, then shard (ct_canon.cu)
struct ShardState {
  // per-tile key counts of the local shard (kept between shard_count and shard_route)
  uint32_t* counts = nullptr;
  uint64_t* offs = nullptr;
  uint64_t* kbase = nullptr;
  const ct_record* recs = nullptr;
  uint64_t n = 0, chunk = 0, T = 0, kc = 0, kh = 0;
  uint32_t K = 0, nmax = 0;
  // the routed part and what its partial must add (set by shard_route / shard_assemble)
  uint64_t part_lo = 0, part_len = 0;
  const ct_record* part = nullptr;
  uint64_t extra_diag[3] = {0, 0, 0};  // incomplete, unmatched send, unmatched recv (rank 0)
  int global_max_dev = -1;
  int rank = 0;
  bool valid = false;
  void release(cudaStream_t st);
};

uint64_t shard_meta_words(uint32_t n_comms);
uint64_t shard_count_words();
int shard_meta(const ct_record* recs, uint64_t n, uint32_t n_comms, int num_sms, cudaStream_t st, uint64_t* dev_out);
int shard_count(ShardState* S, const ct_record* recs, uint64_t n, uint32_t n_comms, const uint64_t* dev_metas,
                int world, int num_sms, cudaStream_t st, uint64_t* dev_out);
int shard_route(ShardState* S, uint32_t n_comms, const uint64_t* dev_metas, const uint64_t* dev_counts, int world,
                int rank, int num_sms, cudaStream_t st, uint64_t* out_pos, ct_record* out_rec, uint64_t* send_counts,
                uint64_t* recv_counts, uint64_t* part_len);
int shard_assemble(ShardState* S, const uint64_t* in_pos, const ct_record* in_rec, uint64_t n_in, ct_record* part,
                   cudaStream_t st);

}  // namespace ct
