/*
 * LD_PRELOAD NCCL interposer (reference spec SPEC.md:453-491, TS model
 * shim.ts:54-163): one trace line per intercepted call per rank in the reference wire
 * format (events.py:251-291 canonical key order, compact separators), then the call
 * is forwarded unchanged and its status returned verbatim.
 *
 *   LD_PRELOAD=libcomscribe_shim.so COMSCRIBE_OUT=trace.jsonl <app>
 *
 * Intercepted: ncclAllReduce, ncclBroadcast, ncclReduce, ncclAllGather,
 * ncclReduceScatter, ncclSend, ncclRecv (+ communicator creation, for ids).
 * Env: COMSCRIBE_OUT (sink, default comscribe_trace.jsonl; opened O_APPEND so the
 * processes of one job can share it, one write(2) per line), COMSCRIBE_DISABLE=1.
 * An unwritable sink disables logging with one warning; calls still forward.
 * COMSCRIBE_NCCL_LIB names the real library when it is not in the global scope.
 *
 * Communicator ids: the spec derives them from the handle address + a process nonce,
 * which only groups ranks living in one process.  Here a communicator created by
 * ncclCommInitRank[Config] is named after a hash of its ncclUniqueId (identical on
 * every rank of the communicator, so one-process-per-GPU jobs group correctly), a
 * ncclCommSplit child after (parent id, color, k) with k the parent's split counter
 * (splits are collective over the parent, so k agrees on every rank and repeated
 * splits with one color get distinct ids), ncclCommInitAll after the nonce + the
 * first handle; a communicator the shim never saw created falls back to address +
 * nonce.  Communicators are named when creation returns ncclSuccess or
 * ncclInProgress (non-blocking init); ncclCommDestroy / ncclCommAbort free their
 * table entry (a full table warns once and leaves new communicators unlogged).  "algo" is "auto" (not observable at the API; the analyzer selects it).
 * Thread safety: per-call formatting in a stack buffer, a mutex around the
 * communicator table, atomic per-communicator sequence counters.
 */
#define _GNU_SOURCE
#include <dlfcn.h>
#include <fcntl.h>
#include <pthread.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
#include <unistd.h>

/* NCCL ABI subset (nccl.h): opaque handles, enums as int, 128-byte unique id */
typedef struct ncclComm* ncclComm_t;
typedef int ncclResult_t;
typedef int ncclDataType_t;
typedef int ncclRedOp_t;
typedef void* cudaStream_t;
typedef struct { char internal[128]; } ncclUniqueId;
typedef struct ncclConfig ncclConfig_t;

#define SHIM_EXPORT __attribute__((visibility("default")))

/* ------------------------------------------------------------------ sink */

static pthread_once_t g_once = PTHREAD_ONCE_INIT;
static int g_fd = -1;
static int g_enabled = 0;
static unsigned long long g_nonce = 0;

static void shim_init(void) {
  const char* dis = getenv("COMSCRIBE_DISABLE");
  if (dis && strcmp(dis, "1") == 0) return;
  const char* path = getenv("COMSCRIBE_OUT");
  if (!path || !*path) path = "comscribe_trace.jsonl";
  g_fd = open(path, O_WRONLY | O_CREAT | O_APPEND | O_CLOEXEC, 0644);
  if (g_fd < 0) {
    fprintf(stderr, "comscribe: cannot open trace sink '%s'; logging disabled\n", path);
    return;
  }
  struct timespec t;
  clock_gettime(CLOCK_REALTIME, &t);
  g_nonce = ((unsigned long long)getpid() << 32) ^ (unsigned long long)t.tv_nsec ^ ((unsigned long long)t.tv_sec << 20);
  g_enabled = 1;
}

static void emit(const char* line, size_t len) {
  size_t off = 0;
  while (off < len) {
    ssize_t w = write(g_fd, line + off, len - off);
    if (w <= 0) {
      g_enabled = 0;
      fprintf(stderr, "comscribe: trace sink write failed; logging disabled\n");
      return;
    }
    off += (size_t)w;
  }
}

/* ------------------------------------------------------- real symbols */

/* The real symbol: the next definition in the global scope, else the already-loaded
 * libnccl.so.2 (frameworks such as torch load it in a RTLD_LOCAL scope that RTLD_NEXT
 * does not search), else COMSCRIBE_NCCL_LIB. */
static void* real(const char* name) {
  void* f = dlsym(RTLD_NEXT, name);
  if (f) return f;
  static void* h = NULL;
  if (!h) {
    const char* lib = getenv("COMSCRIBE_NCCL_LIB");
    h = dlopen(lib && *lib ? lib : "libnccl.so.2", RTLD_NOLOAD | RTLD_LAZY);
    if (!h && lib && *lib) h = dlopen(lib, RTLD_LAZY);
  }
  if (h) f = dlsym(h, name);
  if (!f) fprintf(stderr, "comscribe: %s not found (set COMSCRIBE_NCCL_LIB)\n", name);
  return f;
}

/* the next library's definition of ``name`` (same signature as the interposer) */
#define REAL(name)                                 \
  static __typeof__(name)* p_##name = NULL;        \
  if (!p_##name) p_##name = (__typeof__(name)*)real(#name);

typedef ncclResult_t (*fn_rank)(const ncclComm_t, int*);

static int comm_int(const char* name, ncclComm_t comm) {
  static fn_rank f[3];
  static const char* names[3] = {"ncclCommUserRank", "ncclCommCount", "ncclCommCuDevice"};
  int k = strcmp(name, names[0]) == 0 ? 0 : strcmp(name, names[1]) == 0 ? 1 : 2;
  if (!f[k]) f[k] = (fn_rank)real(names[k]);
  int v = -1;
  if (f[k] && f[k](comm, &v) != 0) v = -1;
  return v;
}

/* ------------------------------------------------------- communicator table */

#define TABLE_SIZE 4096
#define NCCL_IN_PROGRESS 7 /* ncclInProgress: non-blocking creation still running */
#define TOMBSTONE ((ncclComm_t)(uintptr_t)1)
typedef struct {
  ncclComm_t comm;              /* NULL: never used; TOMBSTONE: freed */
  unsigned long long id;
  unsigned long long seq;
  unsigned long long splits;    /* ncclCommSplit calls on this communicator */
} Entry;
static Entry g_table[TABLE_SIZE];
static pthread_mutex_t g_mu = PTHREAD_MUTEX_INITIALIZER;
static int g_full_warned = 0;

static int created(ncclResult_t r) { return r == 0 || r == NCCL_IN_PROGRESS; }

static unsigned long long mix(unsigned long long h, const void* p, size_t n) {
  const unsigned char* b = (const unsigned char*)p;
  for (size_t i = 0; i < n; i++) h = (h ^ b[i]) * 0x100000001b3ull;
  return h;
}

/* open addressing with tombstones (entries of destroyed communicators); g_mu held */
static Entry* slot(ncclComm_t comm, int create) {
  size_t h = (size_t)(((uintptr_t)comm >> 4) * 0x9E3779B97F4A7C15ull) % TABLE_SIZE;
  Entry* reuse = NULL;
  for (size_t i = 0; i < TABLE_SIZE; i++) {
    Entry* e = &g_table[(h + i) % TABLE_SIZE];
    if (e->comm == comm) return e;
    if (e->comm == TOMBSTONE) {
      if (!reuse) reuse = e;
      continue;
    }
    if (!e->comm) {
      if (!reuse) reuse = e;
      break;
    }
  }
  if (!create) return NULL;
  if (!reuse) {
    if (!g_full_warned) {
      g_full_warned = 1;
      fprintf(stderr, "comscribe: communicator table full (%d live); calls on new communicators are not logged\n",
              TABLE_SIZE);
    }
    return NULL;
  }
  reuse->comm = comm;
  reuse->id = mix(0xcbf29ce484222325ull ^ g_nonce, &comm, sizeof(comm));  /* fallback name */
  reuse->seq = 0;
  reuse->splits = 0;
  return reuse;
}

static void forget_comm(ncclComm_t comm) {
  pthread_mutex_lock(&g_mu);
  Entry* e = slot(comm, 0);
  if (e) e->comm = TOMBSTONE;
  pthread_mutex_unlock(&g_mu);
}

static void name_comm(ncclComm_t comm, unsigned long long id) {
  pthread_mutex_lock(&g_mu);
  Entry* e = slot(comm, 1);
  if (e) { e->id = id; e->seq = 0; e->splits = 0; }
  pthread_mutex_unlock(&g_mu);
}

/* id and next sequence number of comm */
static int next_seq(ncclComm_t comm, unsigned long long* id, unsigned long long* seq) {
  pthread_mutex_lock(&g_mu);
  Entry* e = slot(comm, 1);
  if (e) { *id = e->id; *seq = e->seq++; }
  pthread_mutex_unlock(&g_mu);
  return e != NULL;
}

/* ------------------------------------------------------------ formatting */

static const char* dtype_name(ncclDataType_t t) {
  /* ncclInt8 0, ncclUint8 1, ncclInt32 2, ncclUint32 3, ncclInt64 4, ncclUint64 5,
   * ncclFloat16 6, ncclFloat32 7, ncclFloat64 8, ncclBfloat16 9; the fp8 types (10, 11)
   * have no trace dtype and are logged as uint8 (same element width) */
  static const char* names[] = {"int8", "uint8", "int32", "uint32", "int64", "uint64",
                                "float16", "float32", "float64", "bfloat16"};
  if (t >= 0 && t < 10) return names[t];
  return "uint8";
}

static void log_call(ncclComm_t comm, const char* kind, const char* coll, size_t count, ncclDataType_t dt,
                     int root, int peer) {
  pthread_once(&g_once, shim_init);
  if (!g_enabled) return;
  unsigned long long id, seq;
  if (!next_seq(comm, &id, &seq)) return;
  const int rank = comm_int("ncclCommUserRank", comm), nranks = comm_int("ncclCommCount", comm);
  const int dev = comm_int("ncclCommCuDevice", comm);
  struct timespec t;
  clock_gettime(CLOCK_REALTIME, &t);
  const long long ts = (long long)t.tv_sec * 1000000000ll + t.tv_nsec;
  char line[512];
  int n = snprintf(line, sizeof line,
                   "{\"seq\":%llu,\"ts\":%lld,\"kind\":\"%s\",\"comm\":\"%016llx\",\"nranks\":%d,\"rank\":%d,\"dev\":%d",
                   seq, ts, kind, id, nranks, rank, dev);
  if (coll)
    n += snprintf(line + n, sizeof line - n, ",\"coll\":\"%s\",\"algo\":\"auto\",\"count\":%zu,\"dtype\":\"%s\"", coll,
                  count, dtype_name(dt));
  else
    n += snprintf(line + n, sizeof line - n, ",\"peer\":%d,\"count\":%zu,\"dtype\":\"%s\"", peer, count, dtype_name(dt));
  if (root >= 0) n += snprintf(line + n, sizeof line - n, ",\"root\":%d", root);
  n += snprintf(line + n, sizeof line - n, "}\n");
  emit(line, (size_t)n);
}

/* -------------------------------------------------------- creation (ids) */

SHIM_EXPORT ncclResult_t ncclCommInitRank(ncclComm_t* comm, int nranks, ncclUniqueId id, int rank) {
  REAL(ncclCommInitRank);
  if (!p_ncclCommInitRank) return 1;
  ncclResult_t r = p_ncclCommInitRank(comm, nranks, id, rank);
  if (created(r) && comm && *comm) name_comm(*comm, mix(0xcbf29ce484222325ull, id.internal, sizeof id.internal));
  return r;
}

SHIM_EXPORT ncclResult_t ncclCommInitRankConfig(ncclComm_t* comm, int nranks, ncclUniqueId id, int rank,
                                                ncclConfig_t* config) {
  REAL(ncclCommInitRankConfig);
  if (!p_ncclCommInitRankConfig) return 1;
  ncclResult_t r = p_ncclCommInitRankConfig(comm, nranks, id, rank, config);
  if (created(r) && comm && *comm) name_comm(*comm, mix(0xcbf29ce484222325ull, id.internal, sizeof id.internal));
  return r;
}

SHIM_EXPORT ncclResult_t ncclCommInitAll(ncclComm_t* comms, int ndev, const int* devlist) {
  REAL(ncclCommInitAll);
  if (!p_ncclCommInitAll) return 1;
  ncclResult_t r = p_ncclCommInitAll(comms, ndev, devlist);
  if (created(r) && ndev > 0) {
    pthread_once(&g_once, shim_init);
    const unsigned long long id = mix(0xcbf29ce484222325ull ^ g_nonce, &comms[0], sizeof comms[0]);
    for (int i = 0; i < ndev; i++) name_comm(comms[i], id);
  }
  return r;
}

SHIM_EXPORT ncclResult_t ncclCommSplit(ncclComm_t comm, int color, int key, ncclComm_t* newcomm,
                                       ncclConfig_t* config) {
  REAL(ncclCommSplit);
  if (!p_ncclCommSplit) return 1;
  unsigned long long parent = 0, k = 0;
  pthread_mutex_lock(&g_mu);
  Entry* e = slot(comm, 1);
  if (e) { parent = e->id; k = e->splits++; }
  pthread_mutex_unlock(&g_mu);
  ncclResult_t r = p_ncclCommSplit(comm, color, key, newcomm, config);
  if (created(r) && newcomm && *newcomm) name_comm(*newcomm, mix(mix(parent, &color, sizeof color), &k, sizeof k));
  return r;
}

SHIM_EXPORT ncclResult_t ncclCommDestroy(ncclComm_t comm) {
  REAL(ncclCommDestroy);
  forget_comm(comm);
  return p_ncclCommDestroy ? p_ncclCommDestroy(comm) : 1;
}

SHIM_EXPORT ncclResult_t ncclCommAbort(ncclComm_t comm) {
  REAL(ncclCommAbort);
  forget_comm(comm);
  return p_ncclCommAbort ? p_ncclCommAbort(comm) : 1;
}

/* ----------------------------------------------------------- collectives */

SHIM_EXPORT ncclResult_t ncclAllReduce(const void* sendbuff, void* recvbuff, size_t count, ncclDataType_t datatype,
                                       ncclRedOp_t op, ncclComm_t comm, cudaStream_t stream) {
  REAL(ncclAllReduce);
  log_call(comm, "collective", "allreduce", count, datatype, -1, -1);
  return p_ncclAllReduce ? p_ncclAllReduce(sendbuff, recvbuff, count, datatype, op, comm, stream) : 1;
}

SHIM_EXPORT ncclResult_t ncclBroadcast(const void* sendbuff, void* recvbuff, size_t count, ncclDataType_t datatype,
                                       int root, ncclComm_t comm, cudaStream_t stream) {
  REAL(ncclBroadcast);
  log_call(comm, "collective", "broadcast", count, datatype, root, -1);
  return p_ncclBroadcast ? p_ncclBroadcast(sendbuff, recvbuff, count, datatype, root, comm, stream) : 1;
}

SHIM_EXPORT ncclResult_t ncclReduce(const void* sendbuff, void* recvbuff, size_t count, ncclDataType_t datatype,
                                    ncclRedOp_t op, int root, ncclComm_t comm, cudaStream_t stream) {
  REAL(ncclReduce);
  log_call(comm, "collective", "reduce", count, datatype, root, -1);
  return p_ncclReduce ? p_ncclReduce(sendbuff, recvbuff, count, datatype, op, root, comm, stream) : 1;
}

SHIM_EXPORT ncclResult_t ncclAllGather(const void* sendbuff, void* recvbuff, size_t sendcount,
                                       ncclDataType_t datatype, ncclComm_t comm, cudaStream_t stream) {
  REAL(ncclAllGather);
  log_call(comm, "collective", "allgather", sendcount, datatype, -1, -1);
  return p_ncclAllGather ? p_ncclAllGather(sendbuff, recvbuff, sendcount, datatype, comm, stream) : 1;
}

SHIM_EXPORT ncclResult_t ncclReduceScatter(const void* sendbuff, void* recvbuff, size_t recvcount,
                                           ncclDataType_t datatype, ncclRedOp_t op, ncclComm_t comm,
                                           cudaStream_t stream) {
  REAL(ncclReduceScatter);
  log_call(comm, "collective", "reducescatter", recvcount, datatype, -1, -1);
  return p_ncclReduceScatter ? p_ncclReduceScatter(sendbuff, recvbuff, recvcount, datatype, op, comm, stream) : 1;
}

SHIM_EXPORT ncclResult_t ncclSend(const void* sendbuff, size_t count, ncclDataType_t datatype, int peer,
                                  ncclComm_t comm, cudaStream_t stream) {
  REAL(ncclSend);
  log_call(comm, "send", NULL, count, datatype, -1, peer);
  return p_ncclSend ? p_ncclSend(sendbuff, count, datatype, peer, comm, stream) : 1;
}

SHIM_EXPORT ncclResult_t ncclRecv(void* recvbuff, size_t count, ncclDataType_t datatype, int peer, ncclComm_t comm,
                                  cudaStream_t stream) {
  REAL(ncclRecv);
  log_call(comm, "recv", NULL, count, datatype, -1, peer);
  return p_ncclRecv ? p_ncclRecv(recvbuff, count, datatype, peer, comm, stream) : 1;
}
