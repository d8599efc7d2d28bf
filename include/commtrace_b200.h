/*
 * commtrace_b200 — C ABI of the B200-native trace → communication-matrix path.
 *
 * This is the drop-in boundary for the reference's analysis entry point
 *   analyze_events(events, d=None, config=ModelConfig())   pkg/src/commtrace/matrix.py:316-347
 * and its siblings split_by_primitive (matrix.py:261), summarize (matrix.py:279),
 * group_collectives (grouping.py:82) and match_p2p (decompose.py:342).  The
 * reference has no FFI of its own (it is pure Python); INTEGRATION.md shows the
 * ctypes stub a maintainer adds to matrix.py to call this library instead.
 *
 * Plain C types only: no torch, no CUDA types in signatures (streams are void*).
 * Every entry point returns a ct_status; CT_ERR_* codes map 1:1 onto the
 * reference's exception classes (errors.py:9-56 plus OverflowError).
 */
#ifndef COMMTRACE_B200_H
#define COMMTRACE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CT_ABI_VERSION 1

/* ---------------------------------------------------------------- records
 * One trace record (one JSONL line of the reference wire format,
 * events.py:8-24), packed to 32 bytes.  The record size is the roofline unit.
 */
typedef struct ct_record {
  uint64_t count;   /* collective/p2p element count; copy byte count          */
  uint64_t seq;     /* per-(comm, rank) sequence counter                       */
  uint32_t comm;    /* interned communicator id                                */
  uint16_t nranks;  /* communicator size N                                     */
  uint16_t rank;    /* caller rank                                             */
  uint16_t dev;     /* caller GPU                                              */
  uint16_t aux;     /* root (bcast/reduce) | peer (send/recv) | copy src GPU    */
  uint16_t aux2;    /* copy dst GPU                                            */
  uint8_t kc;       /* kind[0:3] | coll[3:6] | has_root[6]                     */
  uint8_t ad;       /* algo[0:2] | dtype[2:6] | ckind[6:8]                     */
} ct_record;

enum { CT_KIND_COLLECTIVE = 0, CT_KIND_SEND = 1, CT_KIND_RECV = 2,
       CT_KIND_MEMCPY = 3, CT_KIND_UM = 4, CT_KIND_ZEROCOPY = 5 };
enum { CT_COLL_ALLREDUCE = 0, CT_COLL_BROADCAST = 1, CT_COLL_REDUCE = 2,
       CT_COLL_REDUCESCATTER = 3, CT_COLL_ALLGATHER = 4 };
enum { CT_ALGO_RING = 0, CT_ALGO_TREE = 1, CT_ALGO_COLLNET = 2, CT_ALGO_AUTO = 3 };
enum { CT_CKIND_H2D = 0, CT_CKIND_D2H = 1, CT_CKIND_D2D = 2 };

/* matrix/statistics type keys, in the reference's ALL_TYPES order (matrix.py:39-44) */
enum { CT_T_ALLREDUCE = 0, CT_T_BROADCAST, CT_T_REDUCE, CT_T_REDUCESCATTER, CT_T_ALLGATHER,
       CT_T_SENDRECV, CT_T_EXPLICIT, CT_T_UNIFIED, CT_T_ZEROCOPY, CT_NTYPES };

/* diagnostic reasons (grouping.py:64-65) */
enum { CT_DIAG_INCOMPLETE = 0, CT_DIAG_INCOMPATIBLE, CT_DIAG_DUPLICATE_DEVICE,
       CT_DIAG_UNMATCHED_SEND, CT_DIAG_UNMATCHED_RECV, CT_DIAG_MISMATCHED_P2P, CT_NDIAG };

/* ---------------------------------------------------------------- status */
typedef enum ct_status {
  CT_OK = 0,
  CT_ERR_INVARIANT = 1,       /* InvariantViolation: nranks disagreement / duplicate seq */
  CT_ERR_INVALID_CONFIG = 2,  /* InvalidConfig: ring order is not a permutation          */
  CT_ERR_ENDPOINT_RANGE = 3,  /* EndpointOutOfRange: transfer GPU >= d                    */
  CT_ERR_OVERFLOW = 4,        /* OverflowError: a matrix cell exceeds 2^63-1              */
  CT_ERR_WRONG_ALGORITHM = 5, /* WrongAlgorithm                                           */
  CT_ERR_MISSING_ROOT = 6,    /* MissingRoot                                              */
  CT_ERR_ARGUMENT = 20,       /* bad argument to this API                                 */
  CT_ERR_CUDA = 21,           /* CUDA runtime failure (message via ct_last_error)         */
  CT_ERR_NOT_CANONICAL = 22,  /* force_path=FAST on a trace the fast path cannot take      */
  CT_ERR_CAPACITY = 23        /* a fixed-capacity table overflowed (see ct_last_error)     */
} ct_status;

/* ---------------------------------------------------------------- config
 * Mirrors ModelConfig (matrix.py:207-222) plus the analyze_events ``d`` argument.
 */
typedef struct ct_config {
  int64_t d;                  /* matrix GPU count; -1 = infer (matrix.py:250-258)      */
  uint64_t tree_threshold;    /* AUTO allreduce: tree below, ring at/above (decompose.py:44) */
  int32_t ring_len;           /* 0 = identity rings; else ring applies where N == ring_len */
  int32_t force_path;         /* 0 auto, 1 fast (canonical layout only), 2 exact,      
                                 3 counting canonicaliser (capture layout) + fast        */
  const uint16_t *ring_order; /* host pointer, ring_len entries (need not be a permutation:
                                 an invalid order raises InvalidConfig only when used)  */
  int32_t dev_hint;           /* >0: caller's bound on (max GPU id + 1); sizes histograms */
  int32_t n_comms;            /* number of interned communicator ids (max comm + 1)     */
} ct_config;

/* ---------------------------------------------------------------- summary
 * Everything except the cells.  Cells are fetched with ct_result_cells in the
 * internal index layout: [type][src][dst] with g2 = g_cap + 2 and endpoint index
 * host = 0, net = 1, gpu g = g + 2 (the host-side wrapper remaps to the reference's
 * host = 0, gpu g = g + 1, net = d + 1 layout, matrix.py:82-102).
 */
typedef struct ct_summary {
  int32_t status;
  int32_t path;               /* 1 = fast (canonical), 2 = exact (sort-based join),     
                                 3 = counting canonicaliser (capture layout) + fast     */
  int64_t d;
  int32_t g_cap;              /* GPUs covered by the cell arrays                        */
  int32_t net_used;           /* bit t set: type t received a collnet transfer          */
  uint64_t calls[CT_NTYPES];
  uint64_t payload_lo[CT_NTYPES];
  uint64_t payload_hi[CT_NTYPES];
  uint64_t diag[CT_NDIAG];
  uint64_t type_first[CT_NTYPES]; /* position of type t in the per_primitive dict order
                                     (matrix.py:334-335); ~0 when the type is absent */
  uint64_t n_records;
  /* error detail (valid when status != CT_OK) */
  uint64_t err_index;         /* record index involved (global numbering)               */
  uint64_t err_aux[4];
  /* timing of the last call, device-measured */
  float ms_total;
  float ms_kernel;            /* the fused expand+accumulate kernel alone               */
  uint32_t n_launches;        /* kernels launched by this call                          */
  uint32_t reserved;
} ct_summary;

typedef struct ct_context ct_context;

/* Create a context bound to CUDA device ``device``; owns scratch and the stream. */
int ct_context_create(int device, ct_context **out);
int ct_context_destroy(ct_context *ctx);
const char *ct_last_error(ct_context *ctx);

/* Analyze n records.  ``recs`` is device memory when on_device != 0, else host
 * memory (copied in inside the call).  ``stream`` may be NULL (context stream).
 * Synchronous: returns when the summary is filled.
 * Replaces analyze_events (matrix.py:316-347) on a packed trace. */
int ct_analyze(ct_context *ctx, const ct_record *recs, uint64_t n, int on_device,
               const ct_config *cfg, ct_summary *out, void *stream);

/* Copy the last result's cells: bytes and freq, each CT_NTYPES*g2*g2 uint64
 * (g2 = out->g_cap + 2).  Host pointers. */
int ct_result_cells(ct_context *ctx, uint64_t *bytes, uint64_t *freq, uint64_t n_cells);

/* Materialise the grouping of the last analyzed trace for the Python-object lists
 * AnalysisResult.instances / .diagnostics (group_collectives, grouping.py:82-183, and
 * match_p2p, decompose.py:342-394), computed by the exact join on the device.
 * ct_result_groups: rows of 5 uint64 {comm, ordinal, status, n_members, member_off} in
 *   reference order (comm first-seen, ordinal); status 0 = instance, else CT_DIAG_*+1;
 *   members = original record indices (rank order), rows concatenated.
 * ct_result_p2p_diags: rows of 7 uint64 {reason, comm, src, dst, k, send_idx, recv_idx}
 *   (~0 for a missing side), per channel in (comm id, src, dst) order.
 * Call with null buffers to query the sizes. */
int ct_result_groups(ct_context *ctx, uint64_t *rows, uint64_t row_cap, uint64_t *members,
                     uint64_t member_cap, uint64_t *n_rows, uint64_t *n_members);
int ct_result_p2p_diags(ct_context *ctx, uint64_t *rows, uint64_t row_cap, uint64_t *n_rows);
/* Run the materialising join on ``recs`` (instead of the last analyzed trace).  Fatal
 * grouping errors (duplicate seq, nranks disagreement) are reported in ``out`` exactly
 * as ct_analyze reports them. */
int ct_materialize(ct_context *ctx, const ct_record *recs, uint64_t n, int on_device, int32_t n_comms,
                   ct_summary *out);

/* infer_device_count (matrix.py:250-258): max(dev, copy GPU endpoint) + 1 over all records. */
int ct_infer_device_count(ct_context *ctx, const ct_record *recs, uint64_t n, int on_device, int64_t *d);

/* Emit mode: per-record transfers of canonical instance blocks (decompose_instance,
 * decompose.py:292-406).  Records must form canonical blocks (ranks 0..n-1
 * consecutive; a send directly followed by its recv).  Output rows of 7 int64
 * {block/record index, src endpoint, dst endpoint, bytes_lo, bytes_hi, src rank, sub}
 * (endpoint: gpu id, -1 = net, -2 = host; sub = destination rank of a collective
 * edge, 0/1 for collnet dev->net / net->dev).  Rows are grouped per record; callers
 * order them per instance. */
int ct_emit_transfers(ct_context *ctx, const ct_record *recs, uint64_t n, int on_device,
                      const ct_config *cfg, int64_t *rows, uint64_t row_cap, uint64_t *n_rows);

/* Synthetic workload generators writing packed records on the
 * device: kind 2 = C2 mixed collectives, 3 = C3 mixed with p2p/copies,
 * 4 = C4 bucketed gradient allreduce, 5 = C5 ring/tree sweep, 6 = C4 in the capture
 * layout of an LD_PRELOAD interposer (ranks interleaved, per-rank order kept).  Records
 * [first, first + n) of the infinite seeded stream are written to dev_out. */
int ct_generate(ct_context *ctx, int kind, uint64_t seed, uint64_t first, uint64_t n,
                ct_record *dev_out, void *stream);
/* Shape of the C4 (ResNet-50, 25 MiB buckets) generator: tensor and bucket counts and
 * the bucket byte sizes (bucket_bytes may be NULL; else room for 64 entries). */
void ct_c4_shape(uint64_t *n_tensors, uint64_t *n_buckets, uint64_t *bucket_bytes);
/* Record index of the first element boundary (block head / send / copy) at or
 * after ``at`` for generator ``kind`` — shard cut points for multi-GPU runs. */
uint64_t ct_generate_boundary(int kind, uint64_t at);

/* Multi-GPU (one process per GPU): each rank analyzes its shard,
 * exports a fixed-size uint64 partial (device memory) that the host all-gathers
 * over NCCL, then merges the ``world`` gathered partials (rank order == shard
 * order) into the final result.  Sums are exact: cells are < 2^63 per shard and
 * are re-checked against the 63-bit bound after merging (matrix.py:164-178);
 * shard-boundary chains (seq order across shards) are re-validated from the
 * boundary records carried in each partial.  All ranks must use the same g_cap
 * (set ct_config.d or dev_hint). */
int ct_partial_size(ct_context *ctx, uint64_t *words);
int ct_partial_export(ct_context *ctx, uint64_t *dev_out, uint64_t words, void *stream);
int ct_partial_merge(ct_context *ctx, const uint64_t *dev_in, int world, uint64_t words,
                     ct_summary *out, void *stream);

/* Multi-GPU for traces in ANY layout (capture layouts included): canonicalise globally,
 * then shard.  Each rank holds a record range (shard) of the trace, in rank order.
 *   1. ct_shard_meta    -> meta_words uint64 (device); all-gather them (rank order)
 *   2. ct_shard_count   (gathered metas) -> count_words uint64; all-gather them
 *   3. ct_shard_route   (both gathered lists): the global canonical layout (what
 *      ct_analyze's counting canonicaliser would build for the whole trace), this
 *      shard's records sorted by global canonical position into dev_out_pos /
 *      dev_out_rec (room for n), grouped by destination rank: send_counts[world],
 *      recv_counts[world] (host) and this rank's part length
 *   4. all-to-all of positions and records with those counts (NCCL)
 *   5. ct_shard_assemble -> the part (a slice of the global canonical stream)
 *   6. ct_analyze(part, force_path = 1), ct_partial_export, all-gather, ct_partial_merge
 *      (the export adds the diagnostics of records no part holds, on rank 0).
 * Scope as the counting canonicaliser (ct_analyze force_path 3); outside it the calls
 * return CT_ERR_NOT_CANONICAL.  Replaces group_collectives / match_p2p over the whole
 * trace (grouping.py:82-183, decompose.py:342-394) before the per-rank merge
 * (matrix.py:164-178). */
int ct_shard_words(int32_t n_comms, uint64_t *meta_words, uint64_t *count_words);
int ct_shard_meta(ct_context *ctx, const ct_record *recs, uint64_t n, int32_t n_comms, uint64_t *dev_out,
                  void *stream);
int ct_shard_count(ct_context *ctx, const ct_record *recs, uint64_t n, int32_t n_comms, const uint64_t *dev_metas,
                   int world, uint64_t *dev_out, void *stream);
int ct_shard_route(ct_context *ctx, int32_t n_comms, const uint64_t *dev_metas, const uint64_t *dev_counts,
                   int world, int rank, uint64_t *dev_out_pos, ct_record *dev_out_rec, uint64_t *send_counts,
                   uint64_t *recv_counts, uint64_t *part_len, void *stream);
int ct_shard_assemble(ct_context *ctx, const uint64_t *dev_in_pos, const ct_record *dev_in_rec, uint64_t n_in,
                      ct_record *dev_part, void *stream);
/* First element start (collective rank-0 record, send, copy) at or after record ``at``
 * of a canonical-layout trace (n when none follows): element-aligned cut points for
 * record-range shards of any canonical trace.  CT_ERR_NOT_CANONICAL when no element
 * starts within the next 64 records. */
int ct_element_boundary(ct_context *ctx, const ct_record *recs, uint64_t n, int on_device, uint64_t at,
                        uint64_t *out);

/* ---------------------------------------------------------------- JSONL loader
 * Device loader for the reference wire format, replacing
 *   parse_trace(source)            pkg/src/commtrace/events.py:352-384
 * (field readers events.py:294-349, TraceEvent.validate events.py:166-236) plus the
 * packing of the events into ct_record (comm ids in first-seen order).  Lines follow
 * str.splitlines(); blank lines are skipped.  A line the device cannot prove the
 * reference accepts unchanged (non-ASCII, escapes, floats/bools/null/huge ints in
 * consulted keys, grammar or validation failures) is "deferred": its record slot is
 * zero and the caller must parse that line with the reference reader, which raises
 * the reference's error for the first bad line (device-accepted lines never raise).
 * A deferred line that turns out blank must be dropped by the caller. */
typedef struct ct_jsonl ct_jsonl;
typedef struct ct_jsonl_info {
  uint64_t n_lines;     /* lines per str.splitlines()                               */
  uint64_t n_records;   /* non-blank lines = record slots (deferred ones included)   */
  uint64_t n_deferred;  /* lines left to the caller (ct_jsonl_deferred)              */
  uint64_t n_comms;     /* distinct comm names among device-parsed lines            */
  uint64_t comm_bytes;  /* total bytes of those names                               */
  uint32_t non_ascii;   /* 1: the text holds bytes >= 0x80 (UTF-8 check is the caller's) */
  float ms_device;      /* device time of the parse (CUDA events)                   */
  uint32_t fused;       /* 1: the single-pass loader took the text, 0: the multi-pass one */
  uint64_t n_slow;      /* single pass: lines read by the generic parser (not the template) */
} ct_jsonl_info;
/* Parse ``size`` bytes (host or device memory).  *out is always set (free it with
 * ct_jsonl_free, also on error; message via ct_jsonl_error). */
int ct_jsonl_parse(int device, const char *text, uint64_t size, int on_device, ct_jsonl **out,
                   ct_jsonl_info *info);
/* n_records records to device memory (comm ids final for device lines); optional
 * n_records int64 timestamps to host memory. */
int ct_jsonl_records(ct_jsonl *j, ct_record *dev_out, int64_t *host_ts);
/* n_deferred rows of 4 uint64: {1-based line number, record slot, byte offset, byte length}. */
int ct_jsonl_deferred(ct_jsonl *j, uint64_t *rows);
/* n_comms rows of 3 uint64 {first record slot, offset into names, length} in comm-id
 * order, and comm_bytes of names. */
int ct_jsonl_comms(ct_jsonl *j, uint64_t *rows, char *names);
const char *ct_jsonl_error(const ct_jsonl *j);
void ct_jsonl_free(ct_jsonl *j);

#ifdef __cplusplus
}
#endif
#endif
