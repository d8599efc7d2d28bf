/* Mock NCCL (test infrastructure, no GPU): the NCCL signatures the interposer forwards
 * to, with communicators as plain structs.  Collectives return 0, except count == 999
 * which returns 5 (checks that the shim passes the status through verbatim). */
#include <stdlib.h>
#include <string.h>

typedef struct ncclComm { int rank, nranks, dev; } *ncclComm_t;
typedef struct { char internal[128]; } ncclUniqueId;

int ncclCommInitRank(ncclComm_t* comm, int nranks, ncclUniqueId id, int rank) {
  (void)id;
  *comm = (ncclComm_t)calloc(1, sizeof(struct ncclComm));
  (*comm)->rank = rank; (*comm)->nranks = nranks; (*comm)->dev = rank + 10;
  return 0;
}
int ncclCommInitAll(ncclComm_t* comms, int ndev, const int* devlist) {
  for (int i = 0; i < ndev; i++) {
    comms[i] = (ncclComm_t)calloc(1, sizeof(struct ncclComm));
    comms[i]->rank = i; comms[i]->nranks = ndev; comms[i]->dev = devlist ? devlist[i] : i;
  }
  return 0;
}
int ncclCommSplit(ncclComm_t comm, int color, int key, ncclComm_t* newcomm, void* config) {
  (void)color; (void)config;
  *newcomm = (ncclComm_t)calloc(1, sizeof(struct ncclComm));
  (*newcomm)->rank = key; (*newcomm)->nranks = comm->nranks; (*newcomm)->dev = comm->dev;
  return 0;
}
int ncclCommDestroy(ncclComm_t comm) { free(comm); return 0; }
int ncclCommAbort(ncclComm_t comm) { free(comm); return 0; }
int ncclCommUserRank(const ncclComm_t c, int* r) { *r = c->rank; return 0; }
int ncclCommCount(const ncclComm_t c, int* n) { *n = c->nranks; return 0; }
int ncclCommCuDevice(const ncclComm_t c, int* d) { *d = c->dev; return 0; }
static int ret(size_t count) { return count == 999 ? 5 : 0; }
int ncclAllReduce(const void* s, void* r, size_t n, int t, int op, ncclComm_t c, void* st) { (void)s; (void)r; (void)t; (void)op; (void)c; (void)st; return ret(n); }
int ncclBroadcast(const void* s, void* r, size_t n, int t, int root, ncclComm_t c, void* st) { (void)s; (void)r; (void)t; (void)root; (void)c; (void)st; return ret(n); }
int ncclReduce(const void* s, void* r, size_t n, int t, int op, int root, ncclComm_t c, void* st) { (void)s; (void)r; (void)t; (void)op; (void)root; (void)c; (void)st; return ret(n); }
int ncclAllGather(const void* s, void* r, size_t n, int t, ncclComm_t c, void* st) { (void)s; (void)r; (void)t; (void)c; (void)st; return ret(n); }
int ncclReduceScatter(const void* s, void* r, size_t n, int t, int op, ncclComm_t c, void* st) { (void)s; (void)r; (void)t; (void)op; (void)c; (void)st; return ret(n); }
int ncclSend(const void* s, size_t n, int t, int peer, ncclComm_t c, void* st) { (void)s; (void)t; (void)peer; (void)c; (void)st; return ret(n); }
int ncclRecv(void* r, size_t n, int t, int peer, ncclComm_t c, void* st) { (void)r; (void)t; (void)peer; (void)c; (void)st; return ret(n); }
