/*
 * _ctpack: native host packer, TraceEvent objects -> 32-byte ct_record array
 * (include/commtrace_b200.h), the front end of analyze_events(list[TraceEvent])
 * (reference pkg/src/commtrace/matrix.py:316-347).
 *
 *   pack(events, comm_ids, codes) -> (records: bytearray, ts: bytearray(int64) | None, bad: int)
 *
 * ``comm_ids`` (dict name -> id) is extended in first-seen order.  ``codes`` is a tuple
 * of dicts mapping enum ``_value_`` strings to the record codes: (kind, coll, algo,
 * dtype, ckind, endpoint kind).  Every event is checked against the conditions of
 * TraceEvent.validate (events.py:166-236) and the packed field ranges; the first event
 * that fails ANY check stops packing and its index is returned in ``bad`` (-1: all
 * packed) -- the Python caller then re-runs the reference-mirroring validate / range
 * check on that event so the exception class and message are exactly the reference's
 * (or RecordRangeError).  ``ts`` is None when some timestamp does not fit int64.
 *
 * Events are read through their instance __dict__ (frozen dataclasses: one dict lookup
 * per field with interned keys) and fall back to getattr for other objects, so both
 * this package's and the reference's TraceEvent work.  Host format conversion only: no
 * grouping, matching or expansion happens here.
 */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <structmember.h>
#include <stdint.h>
#include <string.h>

enum { F_SEQ, F_TS, F_KIND, F_COMM, F_NRANKS, F_RANK, F_DEV, F_COLL, F_ALGO, F_ROOT, F_PEER, F_COUNT, F_DTYPE,
       F_CKIND, F_SRC, F_DST, F_BYTES, F_INDEX, F_VALUE, NF };
static const char* kNames[NF] = {"seq", "ts_ns", "kind", "comm", "n_ranks", "rank", "device", "collective",
                                 "algorithm", "root", "peer", "count", "dtype", "copy_kind", "copy_src",
                                 "copy_dst", "bytes", "index", "_value_"};
static PyObject* g_names[NF];

typedef struct {
  uint64_t count, seq;
  uint32_t comm;
  uint16_t nranks, rank, dev, aux, aux2;
  uint8_t kc, ad;
} Rec;

/* Slotted classes (this package's TraceEvent / Endpoint are dataclass(slots=True)): the
 * byte offset of every field's member descriptor, resolved once per type; a field is then
 * one load from the object.  Other classes (the reference's TraceEvent) use getattr. */
#define NTYPES_CACHED 32
typedef struct { PyTypeObject* type; Py_ssize_t off[NF]; } SlotCache;
static SlotCache g_slots[NTYPES_CACHED];

static const SlotCache* slots_of(PyTypeObject* tp) {
  for (int k = 0; k < NTYPES_CACHED; k++)
    if (g_slots[k].type == tp) return g_slots[k].off[0] == -2 ? NULL : &g_slots[k];
  int k = 0;
  while (k < NTYPES_CACHED && g_slots[k].type) k++;
  if (k == NTYPES_CACHED) return NULL;  /* cache full: getattr */
  SlotCache* c = &g_slots[k];
  c->type = tp;
  Py_INCREF(tp);
  int any = 0;
  for (int f = 0; f < NF; f++) {
    c->off[f] = -1;
    PyObject* d = _PyType_Lookup(tp, g_names[f]);  /* borrowed */
    if (d && Py_TYPE(d) == &PyMemberDescr_Type) {
      PyMemberDef* m = ((PyMemberDescrObject*)d)->d_member;
      if (m->type == Py_T_OBJECT_EX) { c->off[f] = m->offset; any = 1; }
    }
  }
  if (!any) { c->off[0] = -2; return NULL; }
  return c;
}

/* borrowed reference to attribute ``f`` of ``o`` (through its __dict__ when it has one) */
static PyObject* field(PyObject* o, PyObject* dict, int f) {
  const SlotCache* sc = slots_of(Py_TYPE(o));
  if (sc && sc->off[f] >= 0) return *(PyObject**)((char*)o + sc->off[f]);  /* NULL: unset slot */
  if (dict) {
    PyObject* v = PyDict_GetItemWithError(dict, g_names[f]);
    if (v || PyErr_Occurred()) return v;
  }
  PyObject* v = PyObject_GetAttr(o, g_names[f]);
  if (!v) { PyErr_Clear(); return NULL; }
  Py_DECREF(v); /* attributes of a live object stay alive while the object does */
  return v;
}

/* enum members are singletons: the last member seen per enum field and its code */
typedef struct { PyObject* obj; int code; } Memo;

/* enum member -> code via its _value_ string; -1 when absent / unknown */
static int code_of(PyObject* member, PyObject* map);

static int code_memo(PyObject* member, PyObject* map, Memo* m) {
  if (member && member == m->obj) return m->code;
  const int c = code_of(member, map);
  if (c >= 0) { m->obj = member; m->code = c; }
  return c;
}

static int code_of(PyObject* member, PyObject* map) {
  if (!member || member == Py_None) return -1;
  PyObject* dict = NULL;
  PyObject** dp = _PyObject_GetDictPtr(member);
  if (dp) dict = *dp;
  PyObject* val = field(member, dict, F_VALUE);
  if (!val) return -1;
  PyObject* c = PyDict_GetItemWithError(map, val);
  if (!c) { PyErr_Clear(); return -1; }
  return (int)PyLong_AsLong(c);
}

/* exact int (bool included, as Python comparisons treat it) -> int64 / uint64 */
static int as_i64(PyObject* v, long long* out) {
  if (!v || !PyLong_Check(v)) return 0;
  int of = 0;
  *out = PyLong_AsLongLongAndOverflow(v, &of);
  if (of || (*out == -1 && PyErr_Occurred())) { PyErr_Clear(); return 0; }
  return 1;
}

static int as_u64(PyObject* v, uint64_t* out) {
  if (!v || !PyLong_Check(v)) return 0;
  if (_PyLong_Sign(v) < 0) return 0;
  unsigned long long x = PyLong_AsUnsignedLongLong(v);
  if (x == (unsigned long long)-1 && PyErr_Occurred()) { PyErr_Clear(); return 0; }
  *out = x;
  return 1;
}

/* endpoint -> (kind code, index); 0 on failure */
static int endpoint(PyObject* ep, PyObject* epmap, Memo* memo, int* kind, long long* idx) {
  if (!ep || ep == Py_None) return 0;
  PyObject* dict = NULL;
  PyObject** dp = _PyObject_GetDictPtr(ep);
  if (dp) dict = *dp;
  *kind = code_memo(field(ep, dict, F_KIND), epmap, memo);
  return *kind >= 0 && as_i64(field(ep, dict, F_INDEX), idx);
}

static PyObject* pack(PyObject* self, PyObject* args) {
  PyObject *events, *comm_ids, *codes;
  if (!PyArg_ParseTuple(args, "OO!O!", &events, &PyDict_Type, &comm_ids, &PyTuple_Type, &codes)) return NULL;
  if (PyTuple_GET_SIZE(codes) != 6) {
    PyErr_SetString(PyExc_ValueError, "codes must hold 6 maps");
    return NULL;
  }
  PyObject* seqf = PySequence_Fast(events, "events must be a sequence");
  if (!seqf) return NULL;
  PyObject *kmap = PyTuple_GET_ITEM(codes, 0), *cmap = PyTuple_GET_ITEM(codes, 1), *amap = PyTuple_GET_ITEM(codes, 2),
           *dmap = PyTuple_GET_ITEM(codes, 3), *ckmap = PyTuple_GET_ITEM(codes, 4), *epmap = PyTuple_GET_ITEM(codes, 5);
  const Py_ssize_t n = PySequence_Fast_GET_SIZE(seqf);
  PyObject** items = PySequence_Fast_ITEMS(seqf);
  /* bytearrays: numpy views them writable without a copy */
  PyObject* recs = PyByteArray_FromStringAndSize(NULL, n * (Py_ssize_t)sizeof(Rec));
  PyObject* tsb = PyByteArray_FromStringAndSize(NULL, n * (Py_ssize_t)sizeof(int64_t));
  if (!recs || !tsb) { Py_XDECREF(recs); Py_XDECREF(tsb); Py_DECREF(seqf); return NULL; }
  Rec* out = (Rec*)PyByteArray_AS_STRING(recs);
  int64_t* ts = (int64_t*)PyByteArray_AS_STRING(tsb);
  int ts_ok = 1;
  Py_ssize_t bad = -1;
  PyObject* last_comm = NULL;  /* consecutive events usually share a communicator */
  Memo mk = {0}, mc = {0}, ma = {0}, md = {0}, mck = {0}, mep = {0};
  uint32_t last_id = 0;
  for (Py_ssize_t i = 0; i < n; i++) {
    PyObject* ev = items[i];
    PyObject* dict = NULL;  /* getattr (inline instance values; a __dict__ would be materialised) */
    Rec r;
    memset(&r, 0, sizeof r);
    long long nr, rank, dev, t;
    uint64_t seq;
    const int kind = code_memo(field(ev, dict, F_KIND), kmap, &mk);
    PyObject* comm = field(ev, dict, F_COMM);
    /* common fields (validate: nranks >= 1, 0 <= rank < nranks, seq / dev >= 0; ranges) */
    if (kind < 0 || !comm || !PyUnicode_Check(comm) || !as_i64(field(ev, dict, F_NRANKS), &nr) ||
        !as_i64(field(ev, dict, F_RANK), &rank) || !as_i64(field(ev, dict, F_DEV), &dev) ||
        !as_u64(field(ev, dict, F_SEQ), &seq) || nr < 1 || nr > 0xFFFF || rank < 0 || rank >= nr || dev < 0 ||
        dev > 0xFFFF) { bad = i; break; }
    if (as_i64(field(ev, dict, F_TS), &t)) ts[i] = t;
    else { ts_ok = 0; ts[i] = 0; }
    r.seq = seq;
    r.nranks = (uint16_t)nr;
    r.rank = (uint16_t)rank;
    r.dev = (uint16_t)dev;
    r.kc = (uint8_t)kind;
    PyObject* root = field(ev, dict, F_ROOT);
    PyObject* peer = field(ev, dict, F_PEER);
    PyObject* ck = field(ev, dict, F_CKIND);
    if (kind == 0) { /* collective (events.py:184-210) */
      const int coll = code_memo(field(ev, dict, F_COLL), cmap, &mc);
      const int algo = code_memo(field(ev, dict, F_ALGO), amap, &ma);
      const int dt = code_memo(field(ev, dict, F_DTYPE), dmap, &md);
      uint64_t count;
      if (coll < 0 || algo < 0 || dt < 0 || !as_u64(field(ev, dict, F_COUNT), &count)) { bad = i; break; }
      if ((algo == 1 || algo == 2) && coll != 0) { bad = i; break; }  /* tree / collnet: allreduce only */
      const int rooted = coll == 1 || coll == 2;
      long long rt = 0;
      if (rooted) {
        if (!as_i64(root, &rt) || rt < 0 || rt >= nr) { bad = i; break; }
        r.kc |= 1 << 6;
        r.aux = (uint16_t)rt;
      } else if (root && root != Py_None) { bad = i; break; }
      if ((peer && peer != Py_None) || (ck && ck != Py_None)) { bad = i; break; }
      r.kc |= (uint8_t)(coll << 3);
      r.ad = (uint8_t)(algo | dt << 2);
      r.count = count;
    } else if (kind == 1 || kind == 2) { /* send / recv (events.py:212-220) */
      const int dt = code_memo(field(ev, dict, F_DTYPE), dmap, &md);
      long long pr;
      uint64_t count;
      if (dt < 0 || !as_i64(peer, &pr) || !as_u64(field(ev, dict, F_COUNT), &count) || pr == rank || pr < 0 ||
          pr >= nr) { bad = i; break; }
      r.aux = (uint16_t)pr;
      r.ad = (uint8_t)(dt << 2);
      r.count = count;
    } else { /* copies (events.py:222-236): h2d host -> gpu, d2h gpu -> host, d2d two GPUs */
      const int ckc = code_memo(ck, ckmap, &mck);
      int sk, dk;
      long long si, di;
      uint64_t nbytes;
      if (ckc < 0 || !endpoint(field(ev, dict, F_SRC), epmap, &mep, &sk, &si) ||
          !endpoint(field(ev, dict, F_DST), epmap, &mep, &dk, &di) || !as_u64(field(ev, dict, F_BYTES), &nbytes)) {
        bad = i; break;
      }
      /* endpoint kind codes: 0 host, 1 gpu, 2 net */
      const int want_s = ckc == 0 ? 0 : 1, want_d = ckc == 1 ? 0 : 1;
      if (sk != want_s || dk != want_d || (ckc == 2 && si == di)) { bad = i; break; }
      if (si < 0 || si > 0xFFFF || di < 0 || di > 0xFFFF) { bad = i; break; }
      r.aux = sk == 1 ? (uint16_t)si : 0;
      r.aux2 = dk == 1 ? (uint16_t)di : 0;
      r.ad = (uint8_t)(ckc << 6);
      r.count = nbytes;
    }
    /* communicator id in first-seen order */
    if (comm == last_comm) {
      r.comm = last_id;
    } else {
      PyObject* cid = PyDict_GetItemWithError(comm_ids, comm);
      if (cid) {
        r.comm = (uint32_t)PyLong_AsUnsignedLong(cid);
      } else {
        if (PyErr_Occurred()) { bad = i; PyErr_Clear(); break; }
        const Py_ssize_t k = PyDict_GET_SIZE(comm_ids);
        PyObject* v = PyLong_FromSsize_t(k);
        if (!v || PyDict_SetItem(comm_ids, comm, v) < 0) {
          Py_XDECREF(v); Py_DECREF(recs); Py_DECREF(tsb); Py_DECREF(seqf);
          return NULL;
        }
        Py_DECREF(v);
        r.comm = (uint32_t)k;
      }
      last_comm = comm;
      last_id = r.comm;
    }
    out[i] = r;
  }
  Py_DECREF(seqf);
  if (!ts_ok) {
    Py_DECREF(tsb);
    Py_INCREF(Py_None);
    tsb = Py_None;
  }
  return Py_BuildValue("(NNn)", recs, tsb, bad);
}

/*
 * unpack(records, ts, comms, tables) -> list[TraceEvent]: the inverse, for slotted event
 * classes (instances are allocated and their slots filled directly; the records come
 * from this package's packers or the device loader, so they are valid by construction).
 *   records  buffer of n * 32 bytes
 *   ts       buffer of n int64, or a list of n ints (timestamps beyond int64)
 *   comms    list of comm names by id
 *   tables   (TraceEvent type, Endpoint type, kinds[6], colls[5], algos[4], dtypes[10],
 *             ckinds[3], HOST endpoint, GPU endpoint kind)
 */
static int set_slot(PyObject* o, const SlotCache* sc, int f, PyObject* v) { /* steals v */
  if (!v) return -1;
  PyObject** slot = (PyObject**)((char*)o + sc->off[f]);
  Py_XSETREF(*slot, v);
  return 0;
}

static PyObject* unpack(PyObject* self, PyObject* args) {
  Py_buffer rb, tb;
  PyObject *tsobj, *comms, *tables;
  if (!PyArg_ParseTuple(args, "y*OO!O!", &rb, &tsobj, &PyList_Type, &comms, &PyTuple_Type, &tables)) return NULL;
  PyObject* out = NULL;
  int ts_list = PyList_Check(tsobj), have_tb = 0;
  if (!ts_list) {
    if (PyObject_GetBuffer(tsobj, &tb, PyBUF_SIMPLE) < 0) goto done;
    have_tb = 1;
  }
  if (PyTuple_GET_SIZE(tables) != 9) { PyErr_SetString(PyExc_ValueError, "tables must hold 9 entries"); goto done; }
  PyTypeObject* evt = (PyTypeObject*)PyTuple_GET_ITEM(tables, 0);
  PyTypeObject* ept = (PyTypeObject*)PyTuple_GET_ITEM(tables, 1);
  PyObject *kinds = PyTuple_GET_ITEM(tables, 2), *colls = PyTuple_GET_ITEM(tables, 3), *algos = PyTuple_GET_ITEM(tables, 4),
           *dtypes = PyTuple_GET_ITEM(tables, 5), *ckinds = PyTuple_GET_ITEM(tables, 6);
  PyObject *host = PyTuple_GET_ITEM(tables, 7), *gpu_kind = PyTuple_GET_ITEM(tables, 8);
  if (!PyType_Check(evt) || !PyType_Check(ept)) { PyErr_SetString(PyExc_TypeError, "event / endpoint types"); goto done; }
  const SlotCache* se = slots_of(evt);
  const SlotCache* sp = slots_of(ept);
  if (!se || !sp || sp->off[F_KIND] < 0 || sp->off[F_INDEX] < 0) {
    PyErr_SetString(PyExc_TypeError, "unpack needs slotted event and endpoint classes");
    goto done;
  }
  for (int f = 0; f < F_INDEX; f++)
    if (se->off[f] < 0) { PyErr_SetString(PyExc_TypeError, "event class lacks a field slot"); goto done; }
  const Py_ssize_t n = rb.len / 32;
  if (ts_list ? PyList_GET_SIZE(tsobj) != n : tb.len / 8 != n) {
    PyErr_SetString(PyExc_ValueError, "records and timestamps differ in length");
    goto done;
  }
  out = PyList_New(n);
  if (!out) goto done;
  PyObject* gpu_ep[256] = {0};  /* endpoints of GPUs 0..255, shared (frozen, hashable) */
  const Py_ssize_t ncomms = PyList_GET_SIZE(comms);
  const uint8_t* base = (const uint8_t*)rb.buf;
  for (Py_ssize_t i = 0; i < n; i++) {
    Rec r;
    memcpy(&r, base + 32 * i, 32);
    const int kind = r.kc & 7;
    if (kind > 5 || r.comm >= ncomms) { PyErr_SetString(PyExc_ValueError, "malformed record"); Py_CLEAR(out); goto done; }
    PyObject* ev = evt->tp_alloc(evt, 0);
    if (!ev) { Py_CLEAR(out); goto done; }
    PyList_SET_ITEM(out, i, ev);
    for (int f = 0; f < F_INDEX; f++) { Py_INCREF(Py_None); set_slot(ev, se, f, Py_None); }
    PyObject* tsv = ts_list ? Py_NewRef(PyList_GET_ITEM(tsobj, i)) : PyLong_FromLongLong(((const int64_t*)tb.buf)[i]);
    PyObject* cm = PyList_GET_ITEM(comms, r.comm);
    if (set_slot(ev, se, F_SEQ, PyLong_FromUnsignedLongLong(r.seq)) || set_slot(ev, se, F_TS, tsv) ||
        set_slot(ev, se, F_KIND, Py_NewRef(PyTuple_GET_ITEM(kinds, kind))) || set_slot(ev, se, F_COMM, Py_NewRef(cm)) ||
        set_slot(ev, se, F_NRANKS, PyLong_FromLong(r.nranks)) || set_slot(ev, se, F_RANK, PyLong_FromLong(r.rank)) ||
        set_slot(ev, se, F_DEV, PyLong_FromLong(r.dev))) { Py_CLEAR(out); goto done; }
    int bad = 0;
    if (kind == 0) {
      const int coll = (r.kc >> 3) & 7, algo = r.ad & 3, dt = (r.ad >> 2) & 15;
      if (coll > 4 || dt > 9) { bad = 1; }
      else {
        bad |= set_slot(ev, se, F_COLL, Py_NewRef(PyTuple_GET_ITEM(colls, coll)));
        bad |= set_slot(ev, se, F_ALGO, Py_NewRef(PyTuple_GET_ITEM(algos, algo)));
        if ((r.kc >> 6) & 1) bad |= set_slot(ev, se, F_ROOT, PyLong_FromLong(r.aux));
        bad |= set_slot(ev, se, F_COUNT, PyLong_FromUnsignedLongLong(r.count));
        bad |= set_slot(ev, se, F_DTYPE, Py_NewRef(PyTuple_GET_ITEM(dtypes, dt)));
      }
    } else if (kind <= 2) {
      const int dt = (r.ad >> 2) & 15;
      if (dt > 9) { bad = 1; }
      else {
        bad |= set_slot(ev, se, F_PEER, PyLong_FromLong(r.aux));
        bad |= set_slot(ev, se, F_COUNT, PyLong_FromUnsignedLongLong(r.count));
        bad |= set_slot(ev, se, F_DTYPE, Py_NewRef(PyTuple_GET_ITEM(dtypes, dt)));
      }
    } else {
      const int ck = (r.ad >> 6) & 3;
      if (ck > 2) { bad = 1; }
      else {
        PyObject* ends[2] = {NULL, NULL};
        const int is_host[2] = {ck == 0, ck == 1};
        const uint16_t idx[2] = {r.aux, r.aux2};
        for (int e = 0; e < 2 && !bad; e++) {
          if (is_host[e]) { ends[e] = Py_NewRef(host); continue; }
          PyObject* g = idx[e] < 256 ? gpu_ep[idx[e]] : NULL;
          if (!g) {
            g = ept->tp_alloc(ept, 0);
            if (!g || set_slot(g, sp, F_KIND, Py_NewRef(gpu_kind)) || set_slot(g, sp, F_INDEX, PyLong_FromLong(idx[e]))) {
              Py_XDECREF(g);
              bad = 1;
              break;
            }
            if (idx[e] < 256) gpu_ep[idx[e]] = g;  /* the cache holds this reference */
            else { ends[e] = g; continue; }
          }
          ends[e] = Py_NewRef(g);
        }
        if (!bad) {
          bad |= set_slot(ev, se, F_CKIND, Py_NewRef(PyTuple_GET_ITEM(ckinds, ck)));
          bad |= set_slot(ev, se, F_SRC, ends[0]);
          bad |= set_slot(ev, se, F_DST, ends[1]);
          bad |= set_slot(ev, se, F_BYTES, PyLong_FromUnsignedLongLong(r.count));
        } else {
          Py_XDECREF(ends[0]);
          Py_XDECREF(ends[1]);
        }
      }
    }
    if (bad) {
      if (!PyErr_Occurred()) PyErr_SetString(PyExc_ValueError, "malformed record");
      for (int k = 0; k < 256; k++) Py_XDECREF(gpu_ep[k]);
      Py_CLEAR(out);
      goto done;
    }
  }
  for (int k = 0; k < 256; k++) Py_XDECREF(gpu_ep[k]);
done:
  PyBuffer_Release(&rb);
  if (have_tb) PyBuffer_Release(&tb);
  return out;
}

static PyMethodDef kMethods[] = {
    {"pack", pack, METH_VARARGS, "pack(events, comm_ids, codes) -> (records, ts, bad)"},
    {"unpack", unpack, METH_VARARGS, "unpack(records, ts, comms, tables) -> list[TraceEvent]"},
    {NULL, NULL, 0, NULL}};

static struct PyModuleDef kModule = {PyModuleDef_HEAD_INIT, "_ctpack", "native TraceEvent packer", -1, kMethods};

PyMODINIT_FUNC PyInit__ctpack(void) {
  for (int f = 0; f < NF; f++) {
    g_names[f] = PyUnicode_InternFromString(kNames[f]);
    if (!g_names[f]) return NULL;
  }
  return PyModule_Create(&kModule);
}
