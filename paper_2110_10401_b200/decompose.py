"""Per-call decompositions (mirror of reference ``decompose.py``).

``PairTransfer`` / ``Decomposition`` are the reference's value types
(decompose.py:47-85).  The decompose_* functions run the sm_100a emit kernel
(``csrc/ct_emit.cu``: per-record expansion, prefix-summed output slots) on the
instance laid out as one canonical block of records, so the per-instance API and
the matrix path share one implementation of the algorithm models.  Batched use
(``decompose_many``) amortises the launch over thousands of instances.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import (
    DegenerateTree, InvalidConfig, InvariantViolation, MissingRoot, WrongAlgorithm,
)
from .events import (
    Algorithm, CollectiveKind, EventKind, HOST, NET_AGGREGATOR, Endpoint, TraceEvent, gpu,
)

DEFAULT_TREE_THRESHOLD = 1 << 20
_EMIT_COLS = 7


@dataclass(frozen=True)
class PairTransfer:
    src: Endpoint
    dst: Endpoint
    bytes: int

    def __post_init__(self):
        if self.src == self.dst:
            raise InvariantViolation("transfer endpoints must differ")
        if self.bytes < 0:
            raise InvariantViolation("transfer bytes must be non-negative")


@dataclass(frozen=True)
class Decomposition:
    transfers: tuple = ()
    sent_by_rank: dict = field(default_factory=dict)
    recv_by_rank: dict = field(default_factory=dict)

    @property
    def total_bytes(self) -> int:
        return sum(t.bytes for t in self.transfers)

    def by_pair(self) -> dict:
        agg = {}
        for t in self.transfers:
            agg[(t.src, t.dst)] = agg.get((t.src, t.dst), 0) + t.bytes
        return agg


def select_algorithm(inst, tree_threshold: int = DEFAULT_TREE_THRESHOLD) -> Algorithm:
    """AUTO resolution (decompose.py:276-289): the same rule the kernels apply."""
    if inst.collective is not CollectiveKind.ALLREDUCE:
        return Algorithm.RING
    if inst.algorithm is not Algorithm.AUTO:
        return inst.algorithm
    return Algorithm.TREE if inst.payload_bytes < tree_threshold else Algorithm.RING


def _ep(code: int) -> Endpoint:
    if code == -1:
        return NET_AGGREGATOR
    if code == -2:
        return HOST
    return gpu(code)


def _block_events(inst, k: int = 0):
    return [TraceEvent(seq=k, ts_ns=0, kind=EventKind.COLLECTIVE, comm=inst.comm, n_ranks=inst.n_ranks,
                       rank=r, device=inst.per_rank_devices[r], collective=inst.collective,
                       algorithm=inst.algorithm, root=inst.root, count=inst.count, dtype=inst.dtype)
            for r in range(inst.n_ranks)]


def _emit(events, ring_order=None, tree_threshold=DEFAULT_TREE_THRESHOLD, validate=False):
    """Run the emit kernel; returns int64 rows [id, src, dst, lo, hi, rank, sub]."""
    from .packed import RECORD_DTYPE, pack_events

    if validate:
        trace = pack_events(events)
        recs = trace.records
    else:
        recs = _pack_unvalidated(events, RECORD_DTYPE)
    ctx = _lib.context()
    cfg = _lib.make_config(tree_threshold=tree_threshold, ring_order=ring_order)
    n_rows = C.c_uint64()
    ptr = recs.ctypes.data
    rc = ctx.lib.ct_emit_transfers(ctx.handle, C.c_void_p(ptr), recs.shape[0], 0, C.byref(cfg), None, 0,
                                   C.byref(n_rows))
    ctx.check(rc, "ct_emit_transfers")
    _raise(rc, ring_order)
    rows = np.zeros((max(n_rows.value, 1), _EMIT_COLS), dtype=np.int64)
    rc = ctx.lib.ct_emit_transfers(ctx.handle, C.c_void_p(ptr), recs.shape[0], 0, C.byref(cfg),
                                   rows.ctypes.data, n_rows.value, C.byref(n_rows))
    ctx.check(rc, "ct_emit_transfers")
    _raise(rc, ring_order)
    return rows[: n_rows.value]


def _raise(rc, ring_order):
    if rc == _lib.CT_ERR_INVALID_CONFIG:
        order = tuple(ring_order)
        raise InvalidConfig(f"ring order {order} is not a permutation of 0..{len(order) - 1}")
    if rc == _lib.CT_ERR_WRONG_ALGORITHM:
        raise WrongAlgorithm("collective supports only the ring algorithm")
    if rc == _lib.CT_ERR_MISSING_ROOT:
        raise MissingRoot("rooted collective instance has no root")


def _pack_unvalidated(events, dtype):
    """Pack instance blocks without TraceEvent.validate (instances are not events)."""
    from .packed import ALGO_CODE, COLL_CODE, DTYPE_CODE, KIND_CODE

    rec = np.zeros(len(events), dtype=dtype)
    for i, e in enumerate(events):
        kc = KIND_CODE[e.kind] | (COLL_CODE[e.collective] << 3)
        if e.root is not None:
            kc |= 1 << 6
            rec["aux"][i] = e.root
        rec["kc"][i] = kc
        rec["ad"][i] = ALGO_CODE[e.algorithm] | (DTYPE_CODE[e.dtype] << 2)
        rec["count"][i] = e.count
        rec["seq"][i] = e.seq
        rec["nranks"][i] = e.n_ranks
        rec["rank"][i] = e.rank
        rec["dev"][i] = e.device
    return rec


def _decomposition(rows, n, collnet=False, rank_attributed=True) -> Decomposition:
    sent = {r: 0 for r in range(n)}
    recv = {r: 0 for r in range(n)}
    items = []
    for _, src, dst, lo, hi, rank, sub in rows.tolist():
        b = (lo & ((1 << 64) - 1)) | ((hi & ((1 << 64) - 1)) << 64)
        items.append(((rank, sub), PairTransfer(_ep(src), _ep(dst), b)))
        if rank_attributed:
            if collnet:
                if sub == 0:
                    sent[rank] += b
                else:
                    recv[rank] += b
            else:
                sent[rank] += b
                recv[sub] += b
    items.sort(key=lambda x: x[0])
    return Decomposition(tuple(t for _, t in items), sent, recv)


def _check_instance(inst, dbt):
    if inst.collective in (CollectiveKind.BROADCAST, CollectiveKind.REDUCE) and inst.root is None:
        raise MissingRoot(f"{inst.collective.value} instance has no root")
    if dbt is not None:
        n = inst.n_ranks
        if dbt.n_ranks != n or not dbt.spans(n):
            raise DegenerateTree(f"tree does not span ranks 0..{n - 1}")
        from .trees import build_double_binary_tree
        if dbt != build_double_binary_tree(n):
            raise NotImplementedError("custom double binary trees are not supported on the device path")


def _require(inst, collective, algorithm):
    if inst.collective is not collective:
        raise WrongAlgorithm(f"expected {collective.value}, got {inst.collective.value}")
    if inst.algorithm is not algorithm:
        raise WrongAlgorithm(f"instance uses {inst.algorithm.value}, not {algorithm.value}")


def decompose_many(instances, ring_order=None, tree_threshold=DEFAULT_TREE_THRESHOLD) -> list[Decomposition]:
    """Batched decompose_instance: one emit launch for all instances."""
    events, heads = [], []
    for k, inst in enumerate(instances):
        _check_instance(inst, None)
        if inst.collective is not CollectiveKind.ALLREDUCE and inst.algorithm not in (Algorithm.RING, Algorithm.AUTO):
            raise WrongAlgorithm(f"{inst.collective.value} supports only the ring algorithm")
        heads.append(len(events))
        events.extend(_block_events(inst, k))
    rows = _emit(events, ring_order, tree_threshold) if events else np.zeros((0, _EMIT_COLS), np.int64)
    out = []
    order = np.argsort(rows[:, 0], kind="stable") if len(rows) else np.zeros(0, np.int64)
    rows = rows[order]
    starts = np.searchsorted(rows[:, 0], heads) if len(rows) else np.zeros(len(heads), np.int64)
    ends = np.searchsorted(rows[:, 0], heads, side="right") if len(rows) else np.zeros(len(heads), np.int64)
    for inst, a, b in zip(instances, starts, ends):
        collnet = inst.collective is CollectiveKind.ALLREDUCE and select_algorithm(inst, tree_threshold) is Algorithm.COLLNET
        out.append(_decomposition(rows[a:b], inst.n_ranks, collnet=collnet))
    return out


def decompose_instance(inst, ring_order=None, dbt=None, tree_threshold=DEFAULT_TREE_THRESHOLD) -> Decomposition:
    """Dispatch an instance to its algorithm model (decompose.py:292-316)."""
    _check_instance(inst, dbt)
    return decompose_many([inst], ring_order=ring_order, tree_threshold=tree_threshold)[0]


def decompose_allreduce_ring(inst, ring_order=None):
    _require(inst, CollectiveKind.ALLREDUCE, Algorithm.RING)
    return decompose_instance(inst, ring_order)


def decompose_allgather_ring(inst, ring_order=None):
    _require(inst, CollectiveKind.ALLGATHER, Algorithm.RING)
    return decompose_instance(inst, ring_order)


def decompose_reducescatter_ring(inst, ring_order=None):
    _require(inst, CollectiveKind.REDUCESCATTER, Algorithm.RING)
    return decompose_instance(inst, ring_order)


def decompose_broadcast_ring(inst, ring_order=None):
    _require(inst, CollectiveKind.BROADCAST, Algorithm.RING)
    return decompose_instance(inst, ring_order)


def decompose_reduce_ring(inst, ring_order=None):
    _require(inst, CollectiveKind.REDUCE, Algorithm.RING)
    return decompose_instance(inst, ring_order)


def decompose_allreduce_tree(inst, dbt=None):
    _require(inst, CollectiveKind.ALLREDUCE, Algorithm.TREE)
    return decompose_instance(inst, dbt=dbt)


def decompose_allreduce_collnet(inst):
    _require(inst, CollectiveKind.ALLREDUCE, Algorithm.COLLNET)
    return decompose_instance(inst)


def decompose_p2p(send: TraceEvent, recv: TraceEvent) -> Decomposition:
    """Matched send/recv (decompose.py:319-339)."""
    if send.kind is not EventKind.SEND or recv.kind is not EventKind.RECV:
        raise InvariantViolation("decompose_p2p needs a (send, recv) pair")
    if (send.comm != recv.comm or send.peer != recv.rank or recv.peer != send.rank
            or send.count != recv.count or send.dtype != recv.dtype):
        raise InvariantViolation("send/recv events are not counterparts")
    rows = _emit([send, recv], validate=True)
    nbytes = send.count * send.dtype.width_bytes
    transfers = tuple(PairTransfer(_ep(int(r[1])), _ep(int(r[2])), nbytes) for r in rows)
    return Decomposition(transfers, {send.rank: nbytes}, {recv.rank: nbytes})


def decompose_copy(event: TraceEvent) -> Decomposition:
    """Explicit/implicit copy (decompose.py:397-406)."""
    if event.kind in (EventKind.COLLECTIVE, EventKind.SEND, EventKind.RECV):
        raise InvariantViolation("decompose_copy needs a copy-kind event")
    rows = _emit([event], validate=True)
    transfers = tuple(PairTransfer(_ep(int(r[1])), _ep(int(r[2])), int(r[3]) & ((1 << 64) - 1)) for r in rows)
    return Decomposition(transfers, {}, {})


def match_p2p(events):
    """FIFO send/recv pairing per channel (decompose.py:342-394) via the device join."""
    from .grouping import materialize_p2p
    return materialize_p2p(events)
