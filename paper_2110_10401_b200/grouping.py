"""Collective instances and diagnostics (mirror of reference ``grouping.py``).

``CollectiveInstance`` / ``Diagnostic`` are the reference's value types
(grouping.py:24-75).  ``group_collectives`` (grouping.py:82-183) runs the device
join in ``csrc/ct_exact.cu`` — CUB radix sorts by (comm, rank, seq) and by
(comm first-seen, ordinal) — and only converts its row output to Python objects.
"""

from __future__ import annotations

from dataclasses import dataclass, field, replace

import numpy as np

from . import _lib
from .errors import EndpointOutOfRange, InvariantViolation  # noqa: F401  (re-export parity)
from .events import Algorithm, CollectiveKind, DataType, TraceEvent
from .packed import PackedTrace, pack_events

DIAG_REASONS = ("incomplete", "incompatible_arguments", "duplicate_device",
                "unmatched_send", "unmatched_recv", "mismatched_p2p")


@dataclass(frozen=True)
class CollectiveInstance:
    """One logical collective call assembled from N per-rank events (grouping.py:24-57)."""

    comm: str
    ordinal: int
    collective: CollectiveKind
    algorithm: Algorithm
    n_ranks: int
    count: int
    dtype: DataType
    root: int | None = None
    per_rank_devices: tuple[int, ...] = ()

    @property
    def payload_bytes(self) -> int:
        block = self.count * self.dtype.width_bytes
        if self.collective in (CollectiveKind.ALLGATHER, CollectiveKind.REDUCESCATTER):
            return self.n_ranks * block
        return block

    def device_of(self, rank: int) -> int:
        return self.per_rank_devices[rank]

    def with_algorithm(self, algorithm: Algorithm) -> "CollectiveInstance":
        return replace(self, algorithm=algorithm)


@dataclass(frozen=True)
class Diagnostic:
    """Non-fatal grouping/matching problem (grouping.py:60-75)."""

    reason: str
    comm: str
    ordinal: int | None
    detail: str
    events: tuple[TraceEvent, ...] = field(default=())

    def __str__(self):
        where = f"comm={self.comm}"
        if self.ordinal is not None:
            where += f" ordinal={self.ordinal}"
        return f"{self.reason}: {where}: {self.detail}"


def _as_trace(events) -> PackedTrace:
    return events if isinstance(events, PackedTrace) else pack_events(events)


def materialize(trace: PackedTrace, ctx=None, with_pairs: bool = False):
    """Device join → (instances, group diagnostics, p2p diagnostics) as Python objects."""
    import ctypes as C

    ctx = ctx or _lib.context()
    recs = trace.records
    ptr, n, on_dev = _lib.records_pointer(recs)
    summ = _lib.CtSummary()
    rc = ctx.lib.ct_materialize(ctx.handle, C.c_void_p(ptr), n, on_dev, max(len(trace.comms), 1),
                                C.byref(summ))
    ctx.check(rc, "ct_materialize")
    if rc != _lib.CT_OK:
        from .matrix import raise_status
        raise_status(summ, trace, None)
    nr, nm = C.c_uint64(), C.c_uint64()
    rc = ctx.lib.ct_result_groups(ctx.handle, None, 0, None, 0, C.byref(nr), C.byref(nm))
    ctx.check(rc, "ct_result_groups")
    rows = np.zeros((max(nr.value, 1), 5), dtype=np.uint64)
    members = np.zeros(max(nm.value, 1), dtype=np.uint64)
    rc = ctx.lib.ct_result_groups(ctx.handle, rows.ctypes.data, nr.value, members.ctypes.data,
                                  nm.value, C.byref(nr), C.byref(nm))
    ctx.check(rc, "ct_result_groups")
    np_ = C.c_uint64()
    ctx.lib.ct_result_p2p_diags(ctx.handle, None, 0, C.byref(np_))
    prow = np.zeros((max(np_.value, 1), 7), dtype=np.uint64)
    rc = ctx.lib.ct_result_p2p_diags(ctx.handle, prow.ctypes.data, np_.value, C.byref(np_))
    ctx.check(rc, "ct_result_p2p_diags")

    instances, gdiags = [], []
    for comm_id, ordinal, status, cnt, off in rows[: nr.value].tolist():
        idx = members[off: off + cnt].tolist()
        evs = tuple(trace.event(i) for i in idx)
        comm = trace.comms[comm_id]
        if status == 0:
            p = evs[0]
            instances.append(CollectiveInstance(
                comm=comm, ordinal=ordinal, collective=p.collective, algorithm=p.algorithm,
                n_ranks=p.n_ranks, count=p.count, dtype=p.dtype, root=p.root,
                per_rank_devices=tuple(e.device for e in evs)))
            continue
        reason = DIAG_REASONS[status - 1]
        n = evs[0].n_ranks
        if reason == "incomplete":
            missing = sorted(set(range(n)) - {e.rank for e in evs})
            detail = f"missing ranks {missing}"
        elif reason == "incompatible_arguments":
            detail = "ranks disagree on (collective, algo, count, dtype, root)"
        else:
            detail = f"ranks share GPU devices: {tuple(e.device for e in evs)}"
        gdiags.append(Diagnostic(reason, comm, ordinal, detail, evs))

    pdiags, pairs = [], []
    for reason, comm_id, src, dst, k, si, ri in prow[: np_.value].tolist():
        comm = trace.comms[comm_id]
        if reason == len(DIAG_REASONS):  # a matched pair
            pairs.append(((comm, src, dst), (trace.event(si), trace.event(ri))))
            continue
        name = DIAG_REASONS[reason]
        if name == "mismatched_p2p":
            d = Diagnostic(name, comm, k, f"send({src}->{dst}) count/dtype disagree with recv",
                           (trace.event(si), trace.event(ri)))
        elif name == "unmatched_send":
            ev = trace.event(si)
            d = Diagnostic(name, comm, None, f"send {src}->{dst} seq {ev.seq} has no recv", (ev,))
        else:
            ev = trace.event(ri)
            d = Diagnostic(name, comm, None, f"recv {src}->{dst} seq {ev.seq} has no send", (ev,))
        pdiags.append(((comm, src, dst), d))
    pdiags.sort(key=lambda x: x[0])  # reference iterates sorted (comm, src, dst) keys
    pairs.sort(key=lambda x: x[0])
    if with_pairs:
        return instances, gdiags, [d for _, d in pdiags], [p for _, p in pairs]
    return instances, gdiags, [d for _, d in pdiags]


def group_collectives(events) -> tuple[list[CollectiveInstance], list[Diagnostic]]:
    """Instances in (comm first-seen, ordinal) order plus group diagnostics
    (grouping.py:82-183); raises InvariantViolation on duplicate seq / nranks
    disagreement exactly like the reference."""
    trace = _as_trace(events)
    instances, gdiags, _ = materialize(trace)
    return instances, gdiags


def materialize_p2p(events):
    """(pairs, p2p diagnostics) as match_p2p returns them (decompose.py:342-394)."""
    trace = _as_trace(events)
    _, _, pdiags, pairs = materialize(trace, with_pairs=True)
    return pairs, pdiags
