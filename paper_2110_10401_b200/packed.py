"""The packed trace-record format: 32 bytes per record, the roofline unit.

Every kernel on the path streams this layout and nothing else; its size is the
algorithmic-bytes-per-record figure in every roofline this repo reports.  The
C view is ``ct_record`` in ``include/commtrace_b200.h``; the two must agree
byte for byte (checked by ``tests/test_packed.py``).

    offset size field     meaning
    0      8    count     collective/p2p element count; copy byte count
    8      8    seq       per-(comm, rank) sequence counter
    16     4    comm      interned communicator id (first-seen order)
    20     2    nranks    communicator size N
    22     2    rank      caller rank
    24     2    dev       caller GPU id
    26     2    aux       root (bcast/reduce) | peer (send/recv) | copy source GPU
    28     2    aux2      copy destination GPU
    30     1    kc        kind[0:3] | coll[3:6] | has_root[6]
    31     1    ad        algo[0:2] | dtype[2:6] | ckind[6:8]

``ts`` is not on the device (informational only, reference events.py:11); it is
kept host-side so materialised diagnostics can return the original events.

Packing is host-side format conversion of caller-supplied Python objects
(the reference's ``TraceEvent`` list); it performs no grouping, matching or
expansion.  Large traces are produced directly in this format on the device
(``workload.generate_device``) or by the JSONL loader.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import RecordRangeError
from .events import (
    Algorithm,
    CollectiveKind,
    CopyKind,
    DataType,
    Endpoint,
    EndpointKind,
    EventKind,
    HOST,
    TraceEvent,
    gpu,
)

RECORD_BYTES = 32

RECORD_DTYPE = np.dtype(
    [
        ("count", "<u8"),
        ("seq", "<u8"),
        ("comm", "<u4"),
        ("nranks", "<u2"),
        ("rank", "<u2"),
        ("dev", "<u2"),
        ("aux", "<u2"),
        ("aux2", "<u2"),
        ("kc", "u1"),
        ("ad", "u1"),
    ]
)
assert RECORD_DTYPE.itemsize == RECORD_BYTES

# enum codes (must match CT_KIND_*, CT_COLL_*, ... in include/commtrace_b200.h)
KIND_CODE = {
    EventKind.COLLECTIVE: 0, EventKind.SEND: 1, EventKind.RECV: 2,
    EventKind.MEMCPY: 3, EventKind.UNIFIED_MEMORY: 4, EventKind.ZERO_COPY: 5,
}
COLL_CODE = {
    CollectiveKind.ALLREDUCE: 0, CollectiveKind.BROADCAST: 1, CollectiveKind.REDUCE: 2,
    CollectiveKind.REDUCESCATTER: 3, CollectiveKind.ALLGATHER: 4,
}
ALGO_CODE = {Algorithm.RING: 0, Algorithm.TREE: 1, Algorithm.COLLNET: 2, Algorithm.AUTO: 3}
DTYPE_CODE = {dt: i for i, dt in enumerate(DataType)}
CKIND_CODE = {CopyKind.H2D: 0, CopyKind.D2H: 1, CopyKind.D2D: 2}

KINDS = {v: k for k, v in KIND_CODE.items()}
COLLS = {v: k for k, v in COLL_CODE.items()}
ALGOS = {v: k for k, v in ALGO_CODE.items()}
DTYPES = {v: k for k, v in DTYPE_CODE.items()}
CKINDS = {v: k for k, v in CKIND_CODE.items()}

#: element width by dtype code (reference events.py:109-120)
WIDTH_BY_CODE = np.array([DTYPES[i].width_bytes for i in range(10)], dtype=np.uint64)

U16_MAX = (1 << 16) - 1
U64_MAX = (1 << 64) - 1


@dataclass
class PackedTrace:
    """A trace in the device record format plus its host-side side tables.

    ``records``  numpy structured array (RECORD_DTYPE), file order
    ``comms``    comm id -> communicator name
    ``ts``       per-record timestamps (host only; may be None)
    ``events``   the original TraceEvent objects when packed from them
    """

    records: np.ndarray
    comms: list[str] = field(default_factory=list)
    ts: list[int] | None = None
    events: list | None = None

    def __len__(self) -> int:
        return int(self.records.shape[0])

    @property
    def nbytes(self) -> int:
        return len(self) * RECORD_BYTES

    def event(self, i: int) -> TraceEvent:
        """The TraceEvent for record ``i`` (original object when available)."""
        if self.events is not None:
            return self.events[i]
        rec = self.records[i]
        if not isinstance(rec, np.void):  # device records (torch tensor rows)
            rec = np.frombuffer(rec.cpu().numpy().tobytes(), dtype=RECORD_DTYPE)[0]
        return unpack_record(rec, self.comms, 0 if self.ts is None else self.ts[i])


def _check_range(val: int, hi: int, what: str) -> int:
    if val < 0 or val > hi:
        raise RecordRangeError(f"{what} {val} does not fit the packed record range [0, {hi}]")
    return val


def _endpoint_gpu(ep: Endpoint) -> int:
    return _check_range(ep.index, U16_MAX, "copy endpoint GPU") if ep.kind is EndpointKind.GPU else 0


_NATIVE_CODES = (
    {k.value: v for k, v in KIND_CODE.items()},
    {k.value: v for k, v in COLL_CODE.items()},
    {k.value: v for k, v in ALGO_CODE.items()},
    {k.value: v for k, v in DTYPE_CODE.items()},
    {k.value: v for k, v in CKIND_CODE.items()},
    {"host": 0, "gpu": 1, "net": 2},
)


def _native():
    try:
        from . import _ctpack
        return _ctpack
    except ImportError:
        return None


def pack_events(events, comms: dict | None = None) -> PackedTrace:
    """TraceEvent list → PackedTrace.

    Events must satisfy ``TraceEvent.validate()`` (``parse_trace`` guarantees it);
    values must fit the record fields (u64 count/seq/bytes, u16 ranks/devices).
    Works on any object with the reference's TraceEvent attributes.

    The native packer (``csrc/ct_pack.c``, CPython C API) does the work; it stops at
    the first event failing validate() or a record range, and that event is then
    checked here with the reference-mirroring code so the exception is exact.  An
    event the native checks reject but Python accepts (an exotic duck type) sends the
    whole list through the Python packer below.
    """
    events = list(events)
    native = _native()
    if native is not None:
        comm_ids: dict[str, int] = {} if comms is None else dict(comms)
        raw, ts, bad = native.pack(events, comm_ids, _NATIVE_CODES)
        if bad < 0:
            # the packer's bytearrays: writable numpy views, no copy
            rec = np.frombuffer(raw, dtype=RECORD_DTYPE) if events else np.zeros(0, RECORD_DTYPE)
            ts_out = np.frombuffer(ts, dtype=np.int64) if ts is not None else [e.ts_ns for e in events]
            names = [None] * len(comm_ids)
            for name, cid in comm_ids.items():
                names[cid] = name
            return PackedTrace(rec, names, ts_out, events)
        _pack_python([events[bad]])  # raises the reference's exception (or RecordRangeError)
    return _pack_python(events, comms)


def _pack_python(events, comms: dict | None = None) -> PackedTrace:
    """The reference-mirroring packer (validate + range checks, exact messages)."""
    n = len(events)
    rec = np.zeros(n, dtype=RECORD_DTYPE)
    comm_ids: dict[str, int] = {} if comms is None else dict(comms)
    cols = {name: [0] * n for name in RECORD_DTYPE.names}
    ts = [0] * n
    for i, ev in enumerate(events):
        ev.validate()
        cid = comm_ids.get(ev.comm)
        if cid is None:
            cid = comm_ids[ev.comm] = len(comm_ids)
        kind = KIND_CODE[_enum(EventKind, ev.kind)]
        cols["seq"][i] = _check_range(ev.seq, U64_MAX, "seq")
        cols["comm"][i] = cid
        cols["nranks"][i] = _check_range(ev.n_ranks, U16_MAX, "nranks")
        cols["rank"][i] = ev.rank
        cols["dev"][i] = _check_range(ev.device, U16_MAX, "dev")
        ts[i] = ev.ts_ns
        kc = kind
        ad = 0
        if kind == 0:
            coll = COLL_CODE[_enum(CollectiveKind, ev.collective)]
            kc |= coll << 3
            if ev.root is not None:
                kc |= 1 << 6
                cols["aux"][i] = ev.root
            ad = ALGO_CODE[_enum(Algorithm, ev.algorithm)] | (DTYPE_CODE[_enum(DataType, ev.dtype)] << 2)
            cols["count"][i] = _check_range(ev.count, U64_MAX, "count")
        elif kind in (1, 2):
            cols["aux"][i] = ev.peer
            ad = DTYPE_CODE[_enum(DataType, ev.dtype)] << 2
            cols["count"][i] = _check_range(ev.count, U64_MAX, "count")
        else:
            ad = CKIND_CODE[_enum(CopyKind, ev.copy_kind)] << 6
            cols["aux"][i] = _endpoint_gpu(ev.copy_src)
            cols["aux2"][i] = _endpoint_gpu(ev.copy_dst)
            cols["count"][i] = _check_range(ev.bytes, U64_MAX, "bytes")
        cols["kc"][i] = kc
        cols["ad"][i] = ad
    for name in RECORD_DTYPE.names:
        rec[name] = np.array(cols[name], dtype=RECORD_DTYPE[name]) if n else rec[name]
    names = [None] * len(comm_ids)
    for name, cid in comm_ids.items():
        names[cid] = name
    return PackedTrace(rec, names, ts, events)


def _enum(cls, val):
    """Accept our enums or the reference's (same ``.value`` strings)."""
    return val if isinstance(val, cls) else cls(val.value)


def unpack_record(r, comms, ts: int = 0) -> TraceEvent:
    """One packed record → TraceEvent (inverse of pack_events except ``ts``)."""
    kc, ad = int(r["kc"]), int(r["ad"])
    kind = KINDS[kc & 7]
    base = dict(seq=int(r["seq"]), ts_ns=int(ts), kind=kind, comm=comms[int(r["comm"])],
                n_ranks=int(r["nranks"]), rank=int(r["rank"]), device=int(r["dev"]))
    if kind is EventKind.COLLECTIVE:
        return TraceEvent(**base, collective=COLLS[(kc >> 3) & 7], algorithm=ALGOS[ad & 3],
                          root=int(r["aux"]) if (kc >> 6) & 1 else None,
                          count=int(r["count"]), dtype=DTYPES[(ad >> 2) & 15])
    if kind in (EventKind.SEND, EventKind.RECV):
        return TraceEvent(**base, peer=int(r["aux"]), count=int(r["count"]),
                          dtype=DTYPES[(ad >> 2) & 15])
    ck = CKINDS[(ad >> 6) & 3]
    src = HOST if ck is CopyKind.H2D else gpu(int(r["aux"]))
    dst = HOST if ck is CopyKind.D2H else gpu(int(r["aux2"]))
    return TraceEvent(**base, copy_kind=ck, copy_src=src, copy_dst=dst, bytes=int(r["count"]))


def _unpack_tables():
    return (TraceEvent, Endpoint, tuple(KINDS[i] for i in range(6)), tuple(COLLS[i] for i in range(5)),
            tuple(ALGOS[i] for i in range(4)), tuple(DTYPES[i] for i in range(10)), tuple(CKINDS[i] for i in range(3)),
            HOST, EndpointKind.GPU)


def unpack(trace: PackedTrace) -> list[TraceEvent]:
    """The TraceEvent objects of a packed trace (the original objects when it was packed
    from them).  The native unpacker (``csrc/ct_pack.c``) builds the slotted objects
    directly; without it, record by record in Python."""
    if trace.events is not None:
        return list(trace.events)
    native = _native()
    n = len(trace)
    if native is not None and n:
        rec = trace.records
        if not isinstance(rec, np.ndarray):  # device records (a CUDA tensor of rows)
            rec = rec.cpu().numpy()
        raw = np.ascontiguousarray(rec).view(np.uint8).reshape(-1)
        ts = trace.ts
        if ts is None:
            ts = np.zeros(n, np.int64)
        elif not isinstance(ts, np.ndarray):
            ts = [int(t) for t in ts]
        else:
            ts = np.ascontiguousarray(ts, dtype=np.int64)
        import gc

        was = gc.isenabled()
        gc.disable()  # millions of new container objects would trigger collections all along
        try:
            return native.unpack(raw, ts, list(trace.comms), _unpack_tables())
        finally:
            if was:
                gc.enable()
    return [trace.event(i) for i in range(n)]
