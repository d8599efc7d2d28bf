"""The native packer (csrc/ct_pack.c) against the reference-mirroring Python packer:
identical records, comm ids and timestamps on every golden trace and the loader fuzz
corpus, identical exceptions (class + message) on invalid or out-of-range events, and
the reference's own TraceEvent objects accepted (duck typing)."""

import random

import numpy as np
import pytest

from paper_2110_10401_b200 import packed as PK
from paper_2110_10401_b200.events import (
    HOST, Algorithm, CollectiveKind, CopyKind, DataType, EventKind, TraceEvent, gpu, parse_trace,
)
from tests.conftest import load_golden


def _both(events):
    out = []
    for fn in (PK.pack_events, PK._pack_python):
        try:
            tr = fn(events)
            out.append((tr.records.tobytes(), tr.comms, [int(t) for t in tr.ts]))
        except Exception as exc:  # noqa: BLE001 - compared by class and message
            out.append((type(exc).__name__, str(exc)))
    return out


def test_native_extension_is_built():
    assert PK._native() is not None


def test_golden_traces_pack_identically(golden_traces):
    for case in golden_traces:
        a, b = _both(parse_trace(case["jsonl"]))
        assert a == b, case["name"]


def test_fuzz_corpus_packs_identically():
    for row in load_golden("loader_fuzz.json.gz"):
        try:
            events = parse_trace(row["text"])
        except Exception:  # noqa: BLE001
            continue
        a, b = _both(events)
        assert a == b, row["text"][:200]


def _coll(**kw):
    base = dict(seq=0, ts_ns=0, kind=EventKind.COLLECTIVE, comm="c", n_ranks=4, rank=1, device=1,
                collective=CollectiveKind.ALLREDUCE, algorithm=Algorithm.RING, count=8, dtype=DataType.INT8)
    base.update(kw)
    return TraceEvent(**base)


BAD = [
    _coll(n_ranks=0), _coll(rank=4), _coll(rank=-1), _coll(seq=-1), _coll(device=-2), _coll(count=-1),
    _coll(algorithm=Algorithm.TREE, collective=CollectiveKind.BROADCAST, root=0),
    _coll(collective=CollectiveKind.BROADCAST), _coll(collective=CollectiveKind.REDUCE, root=9),
    _coll(root=1), _coll(peer=2), _coll(collective=None), _coll(count=None),
    _coll(seq=1 << 64), _coll(count=1 << 64), _coll(n_ranks=70000, rank=3), _coll(device=65536),
    TraceEvent(seq=0, ts_ns=0, kind=EventKind.SEND, comm="p", n_ranks=2, rank=0, device=0, peer=0, count=1,
               dtype=DataType.INT8),
    TraceEvent(seq=0, ts_ns=0, kind=EventKind.RECV, comm="p", n_ranks=2, rank=0, device=0, peer=5, count=1,
               dtype=DataType.INT8),
    TraceEvent(seq=0, ts_ns=0, kind=EventKind.SEND, comm="p", n_ranks=2, rank=0, device=0, peer=1, count=-3,
               dtype=DataType.INT8),
    TraceEvent(seq=0, ts_ns=0, kind=EventKind.MEMCPY, comm="x", n_ranks=1, rank=0, device=0,
               copy_kind=CopyKind.H2D, copy_src=gpu(1), copy_dst=HOST, bytes=1),
    TraceEvent(seq=0, ts_ns=0, kind=EventKind.MEMCPY, comm="x", n_ranks=1, rank=0, device=0,
               copy_kind=CopyKind.D2D, copy_src=gpu(1), copy_dst=gpu(1), bytes=1),
    TraceEvent(seq=0, ts_ns=0, kind=EventKind.UNIFIED_MEMORY, comm="x", n_ranks=1, rank=0, device=0,
               copy_kind=CopyKind.D2D, copy_src=gpu(1), copy_dst=gpu(70000), bytes=1),
    TraceEvent(seq=0, ts_ns=0, kind=EventKind.ZERO_COPY, comm="x", n_ranks=1, rank=0, device=0,
               copy_kind=CopyKind.H2D, copy_src=HOST, copy_dst=gpu(1), bytes=1 << 64),
    TraceEvent(seq=0, ts_ns=0, kind=EventKind.ZERO_COPY, comm="x", n_ranks=1, rank=0, device=0,
               copy_kind=CopyKind.H2D, copy_src=HOST, copy_dst=gpu(1), bytes=None),
]


@pytest.mark.parametrize("k", range(len(BAD)))
def test_invalid_events_raise_identically(k):
    good = [_coll(seq=s, rank=r, device=r) for s in range(2) for r in range(4)]
    events = good[:5] + [BAD[k]] + good[5:]
    a, b = _both(events)
    assert a == b and isinstance(a[0], str), (a, b)


def test_big_timestamps_and_bools():
    evs = [_coll(ts_ns=1 << 70, rank=r, device=r) for r in range(4)] + [_coll(seq=1, rank=True, device=1)]
    a, b = _both(evs)
    assert a == b


def test_reference_event_objects():
    """The reference's own TraceEvent objects (duck typing through enum _value_)."""
    import sys
    if "/root/reference/pkg/src" not in sys.path and not __import__("os").path.isdir("/root/reference/pkg/src"):
        pytest.skip("reference not present")
    sys.path.insert(0, "/root/reference/pkg/src")
    try:
        from commtrace.events import parse_trace as ref_parse
    finally:
        sys.path.pop(0)
    for case in load_golden("traces.json.gz")[:60]:
        ours, theirs = parse_trace(case["jsonl"]), ref_parse(case["jsonl"])
        a = PK.pack_events(theirs)
        b = PK._pack_python(ours)
        assert a.records.tobytes() == b.records.tobytes() and a.comms == b.comms


def test_native_packer_speed():
    """Sanity bound: well above the reference analyze_events rate (~110K events/s)."""
    import time
    rng = random.Random(0)
    evs = [_coll(seq=s, rank=r, device=r, count=rng.randrange(1 << 30)) for s in range(25000) for r in range(4)]
    t0 = time.perf_counter()
    tr = PK.pack_events(evs)
    dt = time.perf_counter() - t0
    assert len(tr) == len(evs) and len(evs) / dt > 1_000_000, len(evs) / dt


def test_native_unpack_round_trip(golden_traces):
    """unpack (csrc/ct_pack.c) rebuilds exactly the events the records came from: every
    golden trace (all kinds, copies to / from the host, GPU endpoints, rooted and
    unrooted collectives), big timestamps (list ts), GPUs beyond the endpoint cache."""
    for case in golden_traces:
        evs = parse_trace(case["jsonl"])
        if not evs:
            continue
        tr = PK.pack_events(evs)
        back = PK.unpack(PK.PackedTrace(tr.records, tr.comms, tr.ts, None))
        assert back == evs
    evs = [
        TraceEvent(seq=1, ts_ns=1 << 70, kind=EventKind.MEMCPY, comm="c", n_ranks=1, rank=0, device=3,
                   copy_kind=CopyKind.D2D, copy_src=gpu(300), copy_dst=gpu(7), bytes=1 << 63),
        TraceEvent(seq=(1 << 64) - 1, ts_ns=-5, kind=EventKind.COLLECTIVE, comm="d", n_ranks=4, rank=3,
                   device=65535, collective=CollectiveKind.REDUCE, algorithm=Algorithm.RING, root=2,
                   count=0, dtype=DataType.BFLOAT16),
        TraceEvent(seq=0, ts_ns=0, kind=EventKind.UNIFIED_MEMORY, comm="c", n_ranks=1, rank=0, device=0,
                   copy_kind=CopyKind.D2H, copy_src=gpu(0), copy_dst=HOST, bytes=0),
    ]
    tr = PK.pack_events(evs)
    assert PK.unpack(PK.PackedTrace(tr.records, tr.comms, tr.ts, None)) == evs
