/*
 * CPU ORACLE — test infrastructure only, never on the product path.
 *
 * Plain-C restatement of the reference analysis path (arXiv 2110.10401 ``commtrace``:
 * group_collectives grouping.py:82-183, match_p2p decompose.py:342-394, the algorithm
 * models decompose.py:104-316, accumulation matrix.py:82-113 / 316-347) over the packed
 * 32-byte records (include/commtrace_b200.h).  It is written per INSTANCE, like the
 * reference, with sorts for the joins — an independent formulation from the kernels'
 * rank-attributed streaming one.  Used by tests/ (exact parity at millions of records,
 * against the GPU result) and by bench.py's CPU baseline / --impl reference legs.
 * Pinned: tests/test_c_oracle.py checks it against the Python oracle and the golden
 * fixtures produced by the real reference.
 *
 * Output cells use the kernels' internal index layout (host 0, net 1, gpu g -> g + 2)
 * so results compare cell for cell; sums are exact (128-bit) with overflow reported.
 */
#define _GNU_SOURCE
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../include/commtrace_b200.h"

typedef unsigned __int128 u128;

static const int WIDTH[10] = {1, 1, 4, 4, 8, 8, 2, 2, 4, 8};

#define KIND(r) ((r)->kc & 7)
#define COLL(r) (((r)->kc >> 3) & 7)
#define HAS_ROOT(r) (((r)->kc >> 6) & 1)
#define ALGO(r) ((r)->ad & 3)
#define DTYPE(r) (((r)->ad >> 2) & 15)
#define CKIND(r) (((r)->ad >> 6) & 3)

typedef struct {
  const ct_record* R;
  int g2, gcap;
  int64_t d;            /* matrix GPU count */
  int explicit_d;
  u128* cells;          /* [9][g2][g2] */
  uint64_t* freq;
  u128 pay[CT_NTYPES];
  uint64_t calls[CT_NTYPES];
  uint64_t diag[CT_NDIAG];
  int status;
  uint64_t tree_threshold;
  const uint16_t* ring;
  int ring_len, ring_valid;
} Ctx;

/* ------------------------------------------------------------------ accumulation */
static int ep_index(Ctx* c, int ep) { /* ep: gpu g >= 0, -1 host, -2 net */
  if (ep == -1) return 0;
  if (ep == -2) return 1;
  if (ep >= c->d || ep >= c->gcap) {
    if (!c->status) c->status = CT_ERR_ENDPOINT_RANGE;
    return -1;
  }
  return ep + 2;
}

static void add(Ctx* c, int type, int src, int dst, u128 bytes) {
  int a = ep_index(c, src), b = ep_index(c, dst);
  if (a < 0 || b < 0) return;
  size_t k = ((size_t)type * c->g2 + a) * c->g2 + b;
  c->cells[k] += bytes;
  c->freq[k] += 1;
}

/* ------------------------------------------------------------------ models */
static u128 ring_block(u128 s, u128 chunk, int i) {
  u128 off = (u128)i * chunk;
  if (off >= s) return 0;
  u128 rest = s - off;
  return rest < chunk ? rest : chunk;
}

/* in-order tree over positions [lo, hi): root completes the largest perfect left
 * subtree (trees.py:57-78) */
static void build_tree(int lo, int hi, int up, int* parent) {
  if (lo >= hi) return;
  int size = hi - lo, k = 0;
  while ((1 << (k + 1)) <= size) k++;
  int root = lo + (1 << k) - 1;
  parent[root] = up;
  build_tree(lo, root, root, parent);
  build_tree(root + 1, hi, root, parent);
}

typedef struct { int a, b; u128 v; } Edge;
static int edge_cmp(const void* x, const void* y) {
  const Edge *p = (const Edge*)x, *q = (const Edge*)y;
  if (p->a != q->a) return p->a < q->a ? -1 : 1;
  return p->b < q->b ? -1 : p->b > q->b;
}

/* one valid instance: members[r] = record of rank r (decompose_instance, decompose.py:292) */
static void decompose(Ctx* c, const ct_record* const* m, int n) {
  const ct_record* h = m[0];
  const int coll = COLL(h);
  int algo = ALGO(h);
  u128 blk = (u128)h->count * (u128)WIDTH[DTYPE(h)];
  u128 s = (coll == CT_COLL_ALLGATHER || coll == CT_COLL_REDUCESCATTER) ? blk * (u128)n : blk;
  if (coll == CT_COLL_ALLREDUCE) {
    if (algo == CT_ALGO_AUTO) algo = s < (u128)c->tree_threshold ? CT_ALGO_TREE : CT_ALGO_RING;
  } else {
    if (algo == CT_ALGO_TREE || algo == CT_ALGO_COLLNET) { if (!c->status) c->status = CT_ERR_WRONG_ALGORITHM; return; }
    algo = CT_ALGO_RING;
  }
  c->calls[coll] += 1;
  c->pay[coll] += s;
  if (algo == CT_ALGO_COLLNET) {
    if (s == 0) return;
    for (int r = 0; r < n; r++) {
      add(c, coll, m[r]->dev, -2, s);
      add(c, coll, -2, m[r]->dev, s);
    }
    return;
  }
  if ((coll == CT_COLL_BROADCAST || coll == CT_COLL_REDUCE) && !HAS_ROOT(h)) {
    if (!c->status) c->status = CT_ERR_MISSING_ROOT;
    return;
  }
  if (n == 1 || s == 0) return;
  Edge* e = (Edge*)malloc(sizeof(Edge) * (size_t)(4 * n + 4));
  int ne = 0;
  if (algo == CT_ALGO_TREE) {
    int* par = (int*)malloc(sizeof(int) * (size_t)n);
    build_tree(0, n, -1, par);
    u128 share[2] = {s - s / 2, s / 2};
    for (int t = 0; t < 2; t++) {
      if (share[t] == 0) continue;
      for (int pos = 0; pos < n; pos++) {
        if (par[pos] < 0) continue;
        int a = (pos + t) % n, b = (par[pos] + t) % n;
        e[ne].a = a; e[ne].b = b; e[ne].v = share[t]; ne++;
        e[ne].a = b; e[ne].b = a; e[ne].v = share[t]; ne++;
      }
    }
    free(par);
  } else {
    const uint16_t* order = NULL;
    int* inv = NULL;
    if (n == c->ring_len) {
      if (!c->ring_valid) { if (!c->status) c->status = CT_ERR_INVALID_CONFIG; free(e); return; }
      order = c->ring;
    }
    inv = (int*)malloc(sizeof(int) * (size_t)n);
    for (int p = 0; p < n; p++) inv[order ? order[p] : p] = p;
#define ORD(p) (order ? (int)order[(p)] : (p))
    if (coll == CT_COLL_BROADCAST || coll == CT_COLL_REDUCE) {
      int rp = inv[h->aux];
      int start = coll == CT_COLL_REDUCE ? rp + 1 : rp;
      for (int t = 0; t < n - 1; t++) {
        e[ne].a = ORD((start + t) % n); e[ne].b = ORD((start + t + 1) % n); e[ne].v = s; ne++;
      }
    } else {
      u128 chunk = s ? (s + (u128)(n - 1)) / (u128)n : 0;
      for (int p = 0; p < n; p++) {
        u128 out;
        if (coll == CT_COLL_ALLREDUCE) out = 2 * s - ring_block(s, chunk, (p + 1) % n) - ring_block(s, chunk, (p + 2) % n);
        else if (coll == CT_COLL_ALLGATHER) out = s - ring_block(s, chunk, (p + 1) % n);
        else out = s - ring_block(s, chunk, p);
        e[ne].a = ORD(p); e[ne].b = ORD((p + 1) % n); e[ne].v = out; ne++;
      }
    }
#undef ORD
    free(inv);
  }
  qsort(e, (size_t)ne, sizeof(Edge), edge_cmp);
  for (int i = 0; i < ne;) {
    int j = i;
    u128 v = 0;
    while (j < ne && e[j].a == e[i].a && e[j].b == e[i].b) v += e[j++].v;
    if (v > 0) add(c, coll, m[e[i].a]->dev, m[e[i].b]->dev, v);
    i = j;
  }
  free(e);
}

/* ------------------------------------------------------------------ joins */

static int cmp_stream(const void* x, const void* y, void* ctx) { /* (comm, rank, seq) */
  const ct_record* G = (const ct_record*)ctx;
  const ct_record *p = G + *(const uint64_t*)x, *q = G + *(const uint64_t*)y;
  if (p->comm != q->comm) return p->comm < q->comm ? -1 : 1;
  if (p->rank != q->rank) return p->rank < q->rank ? -1 : 1;
  if (p->seq != q->seq) return p->seq < q->seq ? -1 : 1;
  return 0;
}

typedef struct { uint64_t idx, ordinal; } Ord;
static int cmp_group(const void* x, const void* y, void* ctx) { /* (comm, ordinal, rank) */
  const ct_record* G = (const ct_record*)ctx;
  const Ord *a = (const Ord*)x, *b = (const Ord*)y;
  const ct_record *p = G + a->idx, *q = G + b->idx;
  if (p->comm != q->comm) return p->comm < q->comm ? -1 : 1;
  if (a->ordinal != b->ordinal) return a->ordinal < b->ordinal ? -1 : 1;
  return p->rank < q->rank ? -1 : p->rank > q->rank;
}

static int cmp_p2p(const void* x, const void* y, void* ctx) { /* (comm, src, dst, is_recv, seq, idx) */
  const ct_record* G = (const ct_record*)ctx;
  uint64_t i = *(const uint64_t*)x, j = *(const uint64_t*)y;
  const ct_record *p = G + i, *q = G + j;
  int pr = KIND(p) == CT_KIND_RECV, qr = KIND(q) == CT_KIND_RECV;
  uint32_t ps = pr ? p->aux : p->rank, pd = pr ? p->rank : p->aux;
  uint32_t qs = qr ? q->aux : q->rank, qd = qr ? q->rank : q->aux;
  if (p->comm != q->comm) return p->comm < q->comm ? -1 : 1;
  if (ps != qs) return ps < qs ? -1 : 1;
  if (pd != qd) return pd < qd ? -1 : 1;
  if (pr != qr) return pr < qr ? -1 : 1;
  if (p->seq != q->seq) return p->seq < q->seq ? -1 : 1;
  return i < j ? -1 : i > j; /* stable FIFO ties (decompose.py:359-360 sorts stably) */
}

static int sig_equal(const ct_record* a, const ct_record* b) {
  return ((a->kc ^ b->kc) & 0x78) == 0 && ((a->ad ^ b->ad) & 0x3F) == 0 && a->count == b->count &&
         (!HAS_ROOT(a) || a->aux == b->aux);
}

/* Returns the status; cells/freq are [9][g2][g2] with g2 = gcap + 2 (caller allocated,
 * zeroed here).  payload is returned as lo/hi words.  err[0..1]: fatal detail. */
int cto_analyze(const ct_record* R, uint64_t n, int64_t d_explicit, uint64_t tree_threshold,
                const uint16_t* ring, int ring_len, int gcap, uint64_t* cells_out, uint64_t* freq_out,
                uint64_t* calls, uint64_t* pay_lo, uint64_t* pay_hi, uint64_t* diag, int64_t* d_out,
                int* overflow) {
  Ctx c;
  memset(&c, 0, sizeof c);
  c.R = R;
  c.gcap = gcap;
  c.g2 = gcap + 2;
  c.tree_threshold = tree_threshold;
  c.ring = ring;
  c.ring_len = ring_len > 0 ? ring_len : -1;
  c.ring_valid = 1;
  if (ring_len > 0) {
    char* seen = (char*)calloc((size_t)ring_len, 1);
    for (int i = 0; i < ring_len; i++) {
      if (ring[i] >= ring_len || seen[ring[i]]) c.ring_valid = 0;
      else seen[ring[i]] = 1;
    }
    free(seen);
  }
  const size_t ncell = (size_t)9 * c.g2 * c.g2;
  c.cells = (u128*)calloc(ncell, sizeof(u128));
  c.freq = freq_out;
  memset(freq_out, 0, ncell * sizeof(uint64_t));
  /* d (matrix.py:250-258) */
  int64_t top = -1;
  for (uint64_t i = 0; i < n; i++) {
    const ct_record* r = R + i;
    if ((int64_t)r->dev > top) top = r->dev;
    if (KIND(r) >= CT_KIND_MEMCPY) {
      if (CKIND(r) != CT_CKIND_H2D && (int64_t)r->aux > top) top = r->aux;
      if (CKIND(r) != CT_CKIND_D2H && (int64_t)r->aux2 > top) top = r->aux2;
    }
  }
  c.d = d_explicit >= 0 ? d_explicit : top + 1;
  c.explicit_d = d_explicit >= 0;
  *d_out = c.d;
  /* ---- collectives: nranks agreement (grouping.py:97-109) */
  uint64_t nc = 0;
  for (uint64_t i = 0; i < n; i++) nc += KIND(R + i) == CT_KIND_COLLECTIVE;
  uint64_t* ci = (uint64_t*)malloc(sizeof(uint64_t) * (nc + 1));
  uint64_t k = 0;
  for (uint64_t i = 0; i < n; i++)
    if (KIND(R + i) == CT_KIND_COLLECTIVE) ci[k++] = i;
  {
    /* first-seen nranks per comm: comm ids are dense interned ids */
    uint32_t maxc = 0;
    for (uint64_t j = 0; j < nc; j++) if (R[ci[j]].comm > maxc) maxc = R[ci[j]].comm;
    uint16_t* first_n = (uint16_t*)calloc((size_t)maxc + 1, sizeof(uint16_t));
    char* has = (char*)calloc((size_t)maxc + 1, 1);
    for (uint64_t j = 0; j < nc; j++) {
      const ct_record* r = R + ci[j];
      if (!has[r->comm]) { has[r->comm] = 1; first_n[r->comm] = r->nranks; }
      else if (first_n[r->comm] != r->nranks) {
        free(first_n); free(has); free(ci); free(c.cells);
        return CT_ERR_INVARIANT;
      }
    }
    free(first_n); free(has);
  }
  qsort_r(ci, (size_t)nc, sizeof(uint64_t), cmp_stream, (void*)R);
  Ord* ord = (Ord*)malloc(sizeof(Ord) * (nc + 1));
  for (uint64_t j = 0; j < nc; j++) {
    const ct_record* r = R + ci[j];
    if (j && R[ci[j - 1]].comm == r->comm && R[ci[j - 1]].rank == r->rank) {
      if (R[ci[j - 1]].seq == r->seq) { free(ord); free(ci); free(c.cells); return CT_ERR_INVARIANT; }
      ord[j].ordinal = ord[j - 1].ordinal + 1;
    } else {
      ord[j].ordinal = 0;
    }
    ord[j].idx = ci[j];
  }
  free(ci);
  qsort_r(ord, (size_t)nc, sizeof(Ord), cmp_group, (void*)R);
  const ct_record** mem = (const ct_record**)malloc(sizeof(void*) * 65536);
  for (uint64_t j = 0; j < nc;) {
    uint64_t e = j;
    while (e < nc && R[ord[e].idx].comm == R[ord[j].idx].comm && ord[e].ordinal == ord[j].ordinal) e++;
    const int nn = R[ord[j].idx].nranks;
    const uint64_t cnt = e - j;
    if (cnt < (uint64_t)nn) {
      c.diag[CT_DIAG_INCOMPLETE]++;
    } else {
      for (uint64_t q = j; q < e; q++) mem[R[ord[q].idx].rank] = R + ord[q].idx;
      int ok = 1;
      for (int r = 1; r < nn && ok; r++) ok = sig_equal(mem[r], mem[0]);
      if (!ok) {
        c.diag[CT_DIAG_INCOMPATIBLE]++;
      } else {
        int dup = 0;
        for (int a = 0; a < nn && !dup; a++)
          for (int b = a + 1; b < nn; b++)
            if (mem[a]->dev == mem[b]->dev) { dup = 1; break; }
        if (dup) c.diag[CT_DIAG_DUPLICATE_DEVICE]++;
        else decompose(&c, mem, nn);
      }
    }
    j = e;
  }
  free(mem);
  free(ord);
  /* ---- p2p FIFO matching per channel */
  uint64_t np = 0;
  for (uint64_t i = 0; i < n; i++) np += KIND(R + i) == CT_KIND_SEND || KIND(R + i) == CT_KIND_RECV;
  uint64_t* pi = (uint64_t*)malloc(sizeof(uint64_t) * (np + 1));
  k = 0;
  for (uint64_t i = 0; i < n; i++)
    if (KIND(R + i) == CT_KIND_SEND || KIND(R + i) == CT_KIND_RECV) pi[k++] = i;
  qsort_r(pi, (size_t)np, sizeof(uint64_t), cmp_p2p, (void*)R);
  for (uint64_t j = 0; j < np;) {
    const ct_record* f = R + pi[j];
    int fr = KIND(f) == CT_KIND_RECV;
    uint32_t fs = fr ? f->aux : f->rank, fd = fr ? f->rank : f->aux;
    uint64_t e = j, ns = 0;
    while (e < np) {
      const ct_record* g = R + pi[e];
      int gr = KIND(g) == CT_KIND_RECV;
      uint32_t gs = gr ? g->aux : g->rank, gd = gr ? g->rank : g->aux;
      if (g->comm != f->comm || gs != fs || gd != fd) break;
      ns += !gr;
      e++;
    }
    uint64_t nr = e - j - ns, pairs = ns < nr ? ns : nr;
    for (uint64_t q = 0; q < pairs; q++) {
      const ct_record* s = R + pi[j + q];
      const ct_record* r = R + pi[j + ns + q];
      if (s->count != r->count || DTYPE(s) != DTYPE(r)) { c.diag[CT_DIAG_MISMATCHED_P2P]++; continue; }
      u128 nb = (u128)s->count * (u128)WIDTH[DTYPE(s)];
      c.calls[CT_T_SENDRECV]++;
      c.pay[CT_T_SENDRECV] += nb;
      if (s->dev != r->dev) add(&c, CT_T_SENDRECV, s->dev, r->dev, nb);
    }
    c.diag[CT_DIAG_UNMATCHED_SEND] += ns - pairs;
    c.diag[CT_DIAG_UNMATCHED_RECV] += nr - pairs;
    j = e;
  }
  free(pi);
  /* ---- copies */
  for (uint64_t i = 0; i < n; i++) {
    const ct_record* r = R + i;
    const int kind = KIND(r);
    if (kind < CT_KIND_MEMCPY) continue;
    const int t = CT_T_EXPLICIT + (kind - CT_KIND_MEMCPY);
    c.calls[t]++;
    c.pay[t] += r->count;
    add(&c, t, CKIND(r) == CT_CKIND_H2D ? -1 : (int)r->aux, CKIND(r) == CT_CKIND_D2H ? -1 : (int)r->aux2, r->count);
  }
  /* ---- outputs; 63-bit cell bound on the combined matrix (matrix.py:110-113) */
  *overflow = 0;
  for (size_t q = 0; q < ncell; q++) {
    if (c.cells[q] >> 64) *overflow = 1;
    cells_out[q] = (uint64_t)c.cells[q];
  }
  const size_t plane = (size_t)c.g2 * c.g2;
  for (size_t q = 0; q < plane; q++) {
    u128 sum = 0;
    for (int t = 0; t < 9; t++) sum += c.cells[t * plane + q];
    if (sum > (u128)INT64_MAX) *overflow = 1;
  }
  for (int t = 0; t < CT_NTYPES; t++) {
    calls[t] = c.calls[t];
    pay_lo[t] = (uint64_t)c.pay[t];
    pay_hi[t] = (uint64_t)(c.pay[t] >> 64);
  }
  for (int q = 0; q < CT_NDIAG; q++) diag[q] = c.diag[q];
  free(c.cells);
  return c.status;
}
