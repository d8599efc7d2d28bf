"""CPU ORACLE — test infrastructure only, never on the product path.

A plain-Python restatement of the reference analysis path (arXiv 2110.10401's
``commtrace`` package) used as the checker for the sm_100a kernels.  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg may
import it.  Parity is PINNED: ``tests/test_oracle_golden.py`` checks this module
against fixtures produced by running the real reference
(``tests/golden/make_golden.py``).

It is written per *instance* (the reference's formulation, decompose.py), not
per record like the kernels, so agreement between the two is
a real cross-check of the rank-attributed expansion.

Reference anchors (pkg/src/commtrace/...):
  grouping      grouping.py:82-183          ordinals by seq, diagnostics, fatal errors
  p2p matching  decompose.py:342-394        FIFO per (comm, src, dst)
  ring blocks   decompose.py:104-107
  ring AR       decompose.py:130-153        2S - b[p+1] - b[p+2]
  AG / RS       decompose.py:156-189        S - b[p+1] / S - b[p]
  bcast/reduce  decompose.py:192-224        pipeline from root / into root
  tree          decompose.py:227-255, trees.py:57-106
  collnet       decompose.py:258-273
  auto          decompose.py:276-316
  p2p / copy    decompose.py:319-339, 397-406
  matrix        matrix.py:82-113 (index map, 63-bit bound), 157-178
  analyze       matrix.py:225-347 (typed order, stats, per-primitive keys)
  frequency     SURVEY A19 (new): +1 per accumulated transfer
"""

from __future__ import annotations

from dataclasses import dataclass

INT64_MAX = (1 << 63) - 1
WIDTH = {"int8": 1, "uint8": 1, "int32": 4, "uint32": 4, "int64": 8, "uint64": 8,
         "float16": 2, "bfloat16": 2, "float32": 4, "float64": 8}
COLLECTIVES = ("allreduce", "broadcast", "reduce", "reducescatter", "allgather")
TYPES = COLLECTIVES + ("sendrecv", "explicit_transfer", "unified_memory", "zero_copy")
COPY_TYPE = {"memcpy": "explicit_transfer", "um": "unified_memory", "zerocopy": "zero_copy"}


class OracleError(Exception):
    """Carries the reference exception class name and message."""

    def __init__(self, kind: str, message: str):
        super().__init__(message)
        self.kind = kind
        self.message = message


def _v(x):
    return None if x is None else getattr(x, "value", x)


@dataclass
class Ev:
    """Flattened event (duck-typed from any TraceEvent-like object)."""

    idx: int
    kind: str
    comm: str
    n: int
    rank: int
    dev: int
    seq: int
    coll: str | None
    algo: str | None
    count: int | None
    dtype: str | None
    root: int | None
    peer: int | None
    src: tuple | None  # ("host"|"gpu"|"net", idx)
    dst: tuple | None
    nbytes: int | None


def flatten(events) -> list[Ev]:
    out = []
    for i, e in enumerate(events):
        src = dst = None
        if e.copy_src is not None:
            src = (_v(e.copy_src.kind), e.copy_src.index)
            dst = (_v(e.copy_dst.kind), e.copy_dst.index)
        out.append(Ev(i, _v(e.kind), e.comm, e.n_ranks, e.rank, e.device, e.seq, _v(e.collective),
                      _v(e.algorithm), e.count, _v(e.dtype), e.root, e.peer, src, dst, e.bytes))
    return out


# ---------------------------------------------------------------- loader

_KINDS = ("collective", "send", "recv", "memcpy", "um", "zerocopy")
_COLLS = ("allreduce", "broadcast", "reduce", "reducescatter", "allgather")
_ALGOS = ("ring", "tree", "collnet", "auto")
_DTYPES = ("int8", "uint8", "int32", "uint32", "int64", "uint64", "float16", "bfloat16", "float32", "float64")
_CKINDS = {"h2d": ("host", "gpu"), "d2h": ("gpu", "host"), "d2d": ("gpu", "gpu")}


def _need(obj, key, typ, line_no):
    """events.py:294-301: present, of the JSON type, and never a bool."""
    if key not in obj:
        raise OracleError("SchemaViolation", f"line {line_no}: field {key!r} missing")
    v = obj[key]
    if not isinstance(v, typ) or isinstance(v, bool):
        raise OracleError("SchemaViolation", f"line {line_no}: field {key!r} expected {typ.__name__}")
    return v


def _need_enum(obj, key, values, line_no):
    """events.py:304-309."""
    v = _need(obj, key, str, line_no)
    if v not in values:
        raise OracleError("SchemaViolation", f"line {line_no}: field {key!r} unknown value {v!r}")
    return v


def _need_ep(obj, key, line_no):
    """events.py:312-319 (Endpoint.__post_init__ events.py:52-56)."""
    raw = _need(obj, key, dict, line_no)
    kind = _need_enum(raw, "kind", ("host", "gpu", "net"), line_no)
    idx = _need(raw, "idx", int, line_no)
    if idx < 0 or (kind != "gpu" and idx != 0):
        raise OracleError("SchemaViolation", f"line {line_no}: field {key!r} bad endpoint")
    return (kind, idx)


def _validate(e: "Ev", line_no):
    """TraceEvent.validate (events.py:166-236), messages shortened."""
    bad = None
    if e.n < 1 or not 0 <= e.rank < e.n or e.seq < 0 or e.dev < 0:
        bad = "rank / nranks / seq / dev"
    elif e.kind == "collective":
        if e.count < 0 or (e.algo in ("tree", "collnet") and e.coll != "allreduce"):
            bad = "count / algo"
        elif e.coll in ("broadcast", "reduce"):
            if e.root is None or not 0 <= e.root < e.n:
                bad = "root"
        elif e.root is not None:
            bad = "root"
    elif e.kind in ("send", "recv"):
        if e.peer == e.rank or not 0 <= e.peer < e.n or e.count < 0:
            bad = "peer / count"
    else:
        if e.nbytes < 0 or (e.src[0], e.dst[0]) != _CKINDS[e.ckind] or (e.ckind == "d2d" and e.src == e.dst):
            bad = "copy"
    if bad:
        raise OracleError("InvariantViolation", f"line {line_no}: {bad}")


def parse_jsonl(text) -> list:
    """parse_trace (events.py:352-384) restated to flat ``Ev`` rows: UTF-8 decode,
    str.splitlines, skip blank lines, json.loads, the field readers of
    _event_from_obj (events.py:322-349) and validate.  Used to time the reference's
    whole CPU path (parse + analyze) in bench.py's reference arm."""
    import json

    if isinstance(text, (bytes, bytearray)):
        text = text.decode("utf-8")
    out = []
    for line_no, line in enumerate(text.splitlines(), start=1):
        if not line.strip():
            continue
        try:
            obj = json.loads(line)
        except json.JSONDecodeError as exc:
            raise OracleError("MalformedLine", f"line {line_no}: not a valid JSON object ({exc.msg})") from None
        if not isinstance(obj, dict):
            raise OracleError("MalformedLine", f"line {line_no}: not a valid JSON object (not a JSON object)")
        kind = _need_enum(obj, "kind", _KINDS, line_no)
        seq = _need(obj, "seq", int, line_no)
        _need(obj, "ts", int, line_no)
        comm = _need(obj, "comm", str, line_no)
        n = _need(obj, "nranks", int, line_no)
        rank = _need(obj, "rank", int, line_no)
        dev = _need(obj, "dev", int, line_no)
        coll = algo = count = dtype = root = peer = src = dst = nbytes = ckind = None
        if kind == "collective":
            coll = _need_enum(obj, "coll", _COLLS, line_no)
            algo = _need_enum(obj, "algo", _ALGOS, line_no)
            count = _need(obj, "count", int, line_no)
            dtype = _need_enum(obj, "dtype", _DTYPES, line_no)
            if "root" in obj or coll in ("broadcast", "reduce"):
                root = _need(obj, "root", int, line_no)
        elif kind in ("send", "recv"):
            peer = _need(obj, "peer", int, line_no)
            count = _need(obj, "count", int, line_no)
            dtype = _need_enum(obj, "dtype", _DTYPES, line_no)
        else:
            ckind = _need_enum(obj, "ckind", tuple(_CKINDS), line_no)
            src = _need_ep(obj, "src", line_no)
            dst = _need_ep(obj, "dst", line_no)
            nbytes = _need(obj, "bytes", int, line_no)
        e = Ev(len(out), kind, comm, n, rank, dev, seq, coll, algo, count, dtype, root, peer, src, dst, nbytes)
        e.ckind = ckind
        _validate(e, line_no)
        out.append(e)
    return out


def analyze_flat(evs, d=None, ring_order=None, tree_threshold=1 << 20):
    """``analyze`` on already-flat rows (from parse_jsonl)."""
    try:
        return _analyze(evs, d, ring_order, tree_threshold)
    except OracleError as exc:
        return {"error": {"type": exc.kind, "message": exc.message}}


# ---------------------------------------------------------------- grouping

def group(evs: list[Ev]):
    """Instances and diagnostics (grouping.py:82-183)."""
    comm_order, streams, sizes = [], {}, {}
    for e in evs:
        if e.kind != "collective":
            continue
        if e.comm not in streams:
            streams[e.comm] = {}
            sizes[e.comm] = e.n
            comm_order.append(e.comm)
        elif sizes[e.comm] != e.n:
            raise OracleError("InvariantViolation",
                              f"comm {e.comm!r}: events disagree on nranks ({sizes[e.comm]} vs {e.n})")
        streams[e.comm].setdefault(e.rank, []).append(e)
    instances, diags = [], []
    for comm in comm_order:
        n = sizes[comm]
        per_rank = streams[comm]
        for rank, lst in per_rank.items():
            lst.sort(key=lambda e: e.seq)
            for a, b in zip(lst, lst[1:]):
                if a.seq == b.seq:
                    raise OracleError("InvariantViolation",
                                      f"comm {comm!r} rank {rank}: duplicate seq {a.seq}")
        depth = max(len(v) for v in per_rank.values())
        for k in range(depth):
            members = {r: lst[k] for r, lst in per_rank.items() if k < len(lst)}
            if len(members) < n:
                missing = sorted(set(range(n)) - set(members))
                diags.append(("incomplete", comm, k, f"missing ranks {missing}",
                              [members[r].idx for r in sorted(members)]))
                continue
            if len({(m.coll, m.algo, m.count, m.dtype, m.root) for m in members.values()}) > 1:
                diags.append(("incompatible_arguments", comm, k,
                              "ranks disagree on (collective, algo, count, dtype, root)",
                              [members[r].idx for r in sorted(members)]))
                continue
            devs = tuple(members[r].dev for r in range(n))
            if len(set(devs)) < n:
                diags.append(("duplicate_device", comm, k, f"ranks share GPU devices: {devs}",
                              [members[r].idx for r in range(n)]))
                continue
            p = members[0]
            instances.append({"comm": comm, "ordinal": k, "coll": p.coll, "algo": p.algo, "n": n,
                              "count": p.count, "dtype": p.dtype, "root": p.root, "devs": devs})
    return instances, diags


def match(evs: list[Ev]):
    """Send/recv pairing per (comm, src, dst) in seq order (decompose.py:342-394)."""
    sends, recvs = {}, {}
    for e in evs:
        if e.kind == "send":
            sends.setdefault((e.comm, e.rank, e.peer), []).append(e)
        elif e.kind == "recv":
            recvs.setdefault((e.comm, e.peer, e.rank), []).append(e)
    pairs, diags = [], []
    for key in sorted(set(sends) | set(recvs)):
        comm, s, d = key
        ss = sorted(sends.get(key, []), key=lambda e: e.seq)
        rr = sorted(recvs.get(key, []), key=lambda e: e.seq)
        for k, (a, b) in enumerate(zip(ss, rr)):
            if a.count != b.count or a.dtype != b.dtype:
                diags.append(("mismatched_p2p", comm, k,
                              f"send({s}->{d}) count/dtype disagree with recv", [a.idx, b.idx]))
            else:
                pairs.append((a, b))
        for a in ss[len(rr):]:
            diags.append(("unmatched_send", comm, None, f"send {s}->{d} seq {a.seq} has no recv", [a.idx]))
        for b in rr[len(ss):]:
            diags.append(("unmatched_recv", comm, None, f"recv {s}->{d} seq {b.seq} has no send", [b.idx]))
    return pairs, diags


# ---------------------------------------------------------------- models

def payload(inst) -> int:
    block = inst["count"] * WIDTH[inst["dtype"]]
    return inst["n"] * block if inst["coll"] in ("allgather", "reducescatter") else block


def ring_blocks(s: int, n: int) -> list[int]:
    chunk = -(-s // n) if s else 0
    return [max(0, min(chunk, s - i * chunk)) for i in range(n)]


def tree_shape(n: int):
    """In-order binary tree over positions: parent[pos], children[pos] (trees.py:57-78)."""
    parent, children = {}, {p: [] for p in range(n)}

    def build(lo, hi):
        if lo >= hi:
            return None
        k = 0
        while (1 << (k + 1)) <= hi - lo:
            k += 1
        root = lo + (1 << k) - 1
        for sub in (build(lo, root), build(root + 1, hi)):
            if sub is not None:
                parent[sub] = root
                children[root].append(sub)
        return root

    r = build(0, n)
    parent[r] = None
    return parent, children


def rank_edges(inst, ring_order, threshold):
    """Rank-pair edge map of one instance, or ('net', transfers) for collnet."""
    n, s = inst["n"], payload(inst)
    coll, algo = inst["coll"], inst["algo"]
    if algo == "auto":
        algo = ("tree" if s < threshold else "ring") if coll == "allreduce" else "ring"
    if coll != "allreduce" and algo != "ring":
        raise OracleError("WrongAlgorithm", f"{coll} supports only the ring algorithm")
    if coll == "allreduce" and algo == "collnet":
        return "net", ([] if s == 0 else [(r, s) for r in range(n)])
    if coll in ("broadcast", "reduce") and inst["root"] is None:
        raise OracleError("MissingRoot", f"{coll} instance has no root")
    if n == 1 or s == 0:
        return "edges", {}
    edges = {}
    if algo == "tree":
        parent, _ = tree_shape(n)
        for shift, share in ((0, s - s // 2), (1, s // 2)):
            if share == 0:
                continue
            for pos, ppos in parent.items():
                if ppos is None:
                    continue
                a, b = (pos + shift) % n, (ppos + shift) % n
                edges[(a, b)] = edges.get((a, b), 0) + share
                edges[(b, a)] = edges.get((b, a), 0) + share
        return "edges", edges
    order = tuple(range(n)) if ring_order is None else tuple(ring_order)
    if sorted(order) != list(range(n)):
        raise OracleError("InvalidConfig", f"ring order {order} is not a permutation of 0..{n - 1}")
    if coll in ("broadcast", "reduce"):
        rp = order.index(inst["root"])
        start = rp + 1 if coll == "reduce" else rp
        for t in range(n - 1):
            edges[(order[(start + t) % n], order[(start + t + 1) % n])] = s
        return "edges", edges
    b = ring_blocks(s, n)
    for p in range(n):
        if coll == "allreduce":
            out = 2 * s - b[(p + 1) % n] - b[(p + 2) % n]
        elif coll == "allgather":
            out = s - b[(p + 1) % n]
        else:
            out = s - b[p]
        edges[(order[p], order[(p + 1) % n])] = out
    return "edges", edges


def instance_transfers(inst, ring_order, threshold):
    """Endpoint transfers (src, dst, bytes) in reference order (decompose.py:88-97)."""
    mode, data = rank_edges(inst, ring_order, threshold)
    devs = inst["devs"]
    if mode == "net":
        out = []
        for r, s in data:
            out.append((("gpu", devs[r]), ("net", 0), s))
            out.append((("net", 0), ("gpu", devs[r]), s))
        return out
    return [(("gpu", devs[a]), ("gpu", devs[b]), v) for (a, b), v in sorted(data.items()) if v > 0]


# ---------------------------------------------------------------- matrices

class Mat:
    """Dict-free restatement of CommMatrix (matrix.py:53-113) plus frequency."""

    def __init__(self, d):
        self.d, self.agg = d, False
        self.cells = [[0] * (d + 1) for _ in range(d + 1)]
        self.freq = [[0] * (d + 1) for _ in range(d + 1)]

    def idx(self, ep):
        kind, i = ep
        if kind == "host":
            return 0
        if kind == "gpu":
            if i >= self.d:
                raise OracleError("EndpointOutOfRange", f"gpu{i} does not fit a {self.d}-GPU matrix")
            return i + 1
        if not self.agg:
            self.agg = True
            for m in (self.cells, self.freq):
                for row in m:
                    row.append(0)
                m.append([0] * (self.d + 2))
        return self.d + 1

    def add(self, src, dst, v):
        i, j = self.idx(src), self.idx(dst)
        t = self.cells[i][j] + v
        if t > INT64_MAX:
            raise OracleError("OverflowError", f"cell ({i},{j}) exceeds 64-bit byte counter")
        self.cells[i][j] = t
        self.freq[i][j] += 1


def analyze(events, d=None, ring_order=None, tree_threshold=1 << 20):
    """The whole path: returns a fixture-shaped dict (see tests/golden/make_golden.py)."""
    evs = flatten(events)
    try:
        return _analyze(evs, d, ring_order, tree_threshold)
    except OracleError as exc:
        return {"error": {"type": exc.kind, "message": exc.message}}


def infer_d(evs) -> int:
    top = -1
    for e in evs:
        top = max(top, e.dev)
        for ep in (e.src, e.dst):
            if ep is not None and ep[0] == "gpu":
                top = max(top, ep[1])
    return top + 1


def _analyze(evs, d, ring_order, threshold):
    if d is None:
        d = infer_d(evs)
    instances, gdiags = group(evs)
    typed = []
    for inst in instances:
        ro = ring_order if ring_order is not None and len(ring_order) == inst["n"] else None
        typed.append((inst["coll"], payload(inst), instance_transfers(inst, ro, threshold)))
    pairs, pdiags = match(evs)
    for a, b in pairs:
        nb = a.count * WIDTH[a.dtype]
        tr = [(("gpu", a.dev), ("gpu", b.dev), nb)] if a.dev != b.dev else []
        typed.append(("sendrecv", nb, tr))
    for e in evs:
        if e.kind in COPY_TYPE:
            typed.append((COPY_TYPE[e.kind], e.nbytes, [(e.src, e.dst, e.nbytes)]))
    combined = Mat(d)
    per = {}
    calls = {t: 0 for t in TYPES}
    pay = {t: 0 for t in TYPES}
    wire = {t: 0 for t in TYPES}
    for key, p, trs in typed:
        for src, dst, v in trs:
            combined.add(src, dst, v)
        if key not in per:
            per[key] = Mat(d)
        for src, dst, v in trs:
            per[key].add(src, dst, v)
        calls[key] += 1
        pay[key] += p
        wire[key] += sum(v for _, _, v in trs)
    diags = gdiags + pdiags
    return {"result": {
        "d": d,
        "combined": combined.cells, "combined_agg": combined.agg, "combined_freq": combined.freq,
        "per_primitive": [[k, m.cells, m.agg, m.freq] for k, m in per.items()],
        "stats": {t: [calls[t], pay[t], wire[t]] for t in TYPES},
        "instances": len(instances),
        "n_diagnostics": len(diags),
        "diagnostics": [list(x) for x in diags],
        "instance_list": [[i["comm"], i["ordinal"], i["coll"], i["algo"], i["n"], i["count"],
                           i["dtype"], i["root"], list(i["devs"])] for i in instances],
    }}


def decompose(coll, algo, n, count, dtype, root, devs, ring_order=None, tree_threshold=1 << 20):
    """Transfers of one instance as [(src_idx|-1 for net, dst_idx|-1, bytes)]."""
    inst = {"coll": coll, "algo": algo, "n": n, "count": count, "dtype": dtype, "root": root,
            "devs": tuple(devs)}
    out = []
    for src, dst, v in instance_transfers(inst, ring_order, tree_threshold):
        out.append([-1 if src[0] == "net" else src[1], -1 if dst[0] == "net" else dst[1], v])
    return out
