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

}  // namespace ct
