"""Communication matrices, statistics and the ``analyze_events`` driver.

Mirror of the reference ``pkg/src/commtrace/matrix.py``.  ``CommMatrix``,
``accumulate`` and ``merge`` are the reference's small host-side value type and its
O(d^2) helpers (matrix.py:53-178).  ``analyze_events`` (matrix.py:316-347) — the
drop-in boundary — packs the events, hands the 32-byte record stream to
``ct_analyze`` (one fused sm_100a kernel on canonical traces, a device sort-based
join first otherwise) and converts the returned cells/statistics back into the
reference's objects, adding the frequency matrices.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .decompose import DEFAULT_TREE_THRESHOLD, Decomposition
from .errors import (
    EndpointOutOfRange, InvalidConfig, InvariantViolation, MissingRoot, WrongAlgorithm,
)
from .events import CollectiveKind, Endpoint, EndpointKind
from .packed import PackedTrace, pack_events

_INT64_MAX = (1 << 63) - 1

COLLECTIVE_TYPES = tuple(k.value for k in CollectiveKind)
SENDRECV = "sendrecv"
EXPLICIT = "explicit_transfer"
UNIFIED = "unified_memory"
ZEROCOPY = "zero_copy"
ALL_TYPES = COLLECTIVE_TYPES + (SENDRECV, EXPLICIT, UNIFIED, ZEROCOPY)


class CommMatrix:
    """Directed (d+1)x(d+1) byte matrix, host at 0, GPU g at g+1, net at d+1."""

    def __init__(self, d: int, with_aggregator: bool = False):
        if d < 0:
            raise ValueError("device count must be non-negative")
        self.d = d
        self.with_aggregator = with_aggregator
        self._cells = [[0] * self.size for _ in range(self.size)]

    @property
    def size(self) -> int:
        return self.d + 1 + (1 if self.with_aggregator else 0)

    @classmethod
    def from_rows(cls, d: int, rows, with_aggregator: bool = False) -> "CommMatrix":
        out = cls(d, with_aggregator)
        if len(rows) != out.size or any(len(r) != out.size for r in rows):
            raise ValueError(f"expected {out.size}x{out.size} rows")
        out._cells = [[int(v) for v in row] for row in rows]
        return out

    def labels(self) -> list[str]:
        return ["host"] + [f"gpu{g}" for g in range(self.d)] + (["net"] if self.with_aggregator else [])

    def index_of(self, ep: Endpoint) -> int:
        if ep.kind is EndpointKind.HOST:
            return 0
        if ep.kind is EndpointKind.GPU:
            if ep.index >= self.d:
                raise EndpointOutOfRange(f"gpu{ep.index} does not fit a {self.d}-GPU matrix")
            return ep.index + 1
        self.widen()
        return self.d + 1

    def widen(self):
        if self.with_aggregator:
            return
        self.with_aggregator = True
        for row in self._cells:
            row.append(0)
        self._cells.append([0] * self.size)

    def __getitem__(self, key):
        i, j = key
        return self._cells[i][j]

    def add(self, src: Endpoint, dst: Endpoint, nbytes: int):
        i, j = self.index_of(src), self.index_of(dst)
        total = self._cells[i][j] + nbytes
        if total > _INT64_MAX:
            raise OverflowError(f"cell ({i},{j}) exceeds 64-bit byte counter")
        self._cells[i][j] = total

    def rows(self) -> list[list[int]]:
        return [list(r) for r in self._cells]

    def as_array(self) -> np.ndarray:
        return np.array(self._cells, dtype=np.int64)

    @property
    def max_cell(self) -> int:
        return max(max(r) for r in self._cells)

    def row_sum(self, i: int) -> int:
        return sum(self._cells[i])

    def col_sum(self, j: int) -> int:
        return sum(r[j] for r in self._cells)

    def symmetrized(self) -> "CommMatrix":
        out = CommMatrix(self.d, self.with_aggregator)
        n = self.size
        out._cells = [[self._cells[i][j] + self._cells[j][i] for j in range(n)] for i in range(n)]
        return out

    def copy(self) -> "CommMatrix":
        out = CommMatrix(self.d, self.with_aggregator)
        out._cells = [list(r) for r in self._cells]
        return out

    def __eq__(self, other):
        return (isinstance(other, CommMatrix) and self.d == other.d
                and self.with_aggregator == other.with_aggregator and self._cells == other._cells)

    def __repr__(self):
        return f"CommMatrix(d={self.d}, aggregator={self.with_aggregator})"


def accumulate(matrix: CommMatrix, dec: Decomposition) -> CommMatrix:
    """Add one decomposition's transfers in place (matrix.py:157-161)."""
    for t in dec.transfers:
        matrix.add(t.src, t.dst, t.bytes)
    return matrix


def merge(a: CommMatrix, b: CommMatrix) -> CommMatrix:
    """Cellwise sum, widening for the aggregator (matrix.py:164-178)."""
    if a.d != b.d:
        raise EndpointOutOfRange(f"matrix sizes differ: d={a.d} vs d={b.d}")
    out = a.copy()
    if b.with_aggregator:
        out.widen()
    for i in range(b.size):
        for j in range(b.size):
            v = out._cells[i][j] + b._cells[i][j]
            if v > _INT64_MAX:
                raise OverflowError(f"cell ({i},{j}) exceeds 64-bit byte counter")
            out._cells[i][j] = v
    return out


@dataclass(frozen=True)
class TypeStats:
    call_count: int = 0
    payload_bytes: int = 0
    wire_bytes: int = 0


@dataclass
class StatsSummary:
    types: dict = field(default_factory=lambda: {t: TypeStats() for t in ALL_TYPES})
    instances: int = 0
    diagnostics: int = 0

    def get(self, type_key: str) -> TypeStats:
        return self.types[type_key]


@dataclass(frozen=True)
class ModelConfig:
    """Ring order (applied where N == len) and auto tree threshold (matrix.py:207-222)."""

    ring_order: tuple | None = None
    tree_threshold: int = DEFAULT_TREE_THRESHOLD

    def ring_for(self, n_ranks: int):
        if self.ring_order is not None and len(self.ring_order) == n_ranks:
            return self.ring_order
        return None


class AnalysisResult:
    """Result of analyze_events (matrix.py:304-313) plus the frequency matrices.

    ``instances`` / ``diagnostics`` are materialised lazily from the device join on
    first access (counts are always available in ``stats``).
    """

    def __init__(self, d, combined, per_primitive, stats, combined_frequency,
                 per_primitive_frequency, trace=None, path=0, timing=None,
                 instances=None, diagnostics=None):
        self.d = d
        self.combined = combined
        self.per_primitive = per_primitive
        self.stats = stats
        self.combined_frequency = combined_frequency
        self.per_primitive_frequency = per_primitive_frequency
        self.path = path          # 1 fast (canonical layout), 2 exact join
        self.timing = timing or {}
        self._trace = trace
        self._instances = instances
        self._diagnostics = diagnostics

    def _materialize(self):
        from .grouping import materialize
        if self._trace is None:
            self._instances, self._diagnostics = [], []
            return
        inst, gd, pd = materialize(self._trace)
        self._instances, self._diagnostics = inst, gd + pd

    @property
    def instances(self):
        if self._instances is None:
            self._materialize()
        return self._instances

    @property
    def diagnostics(self):
        if self._diagnostics is None:
            self._materialize()
        return self._diagnostics


# ------------------------------------------------------------------- driver

def _config(config) -> ModelConfig:
    return config if config is not None else ModelConfig()


def raise_status(summ, trace: PackedTrace | None, config: ModelConfig | None):
    """Map a ct_status onto the reference's exception with its exact message."""
    st = summ.status
    comms = trace.comms if trace is not None else []

    def comm_name(cid):
        return comms[cid] if cid < len(comms) else f"comm{cid}"

    if st == _lib.CT_ERR_INVARIANT:
        kind = summ.err_aux[3]
        if kind == 1:
            raise InvariantViolation(
                f"comm {comm_name(summ.err_aux[0])!r}: events disagree on nranks "
                f"({summ.err_aux[1]} vs {summ.err_aux[2]})")
        raise InvariantViolation(
            f"comm {comm_name(summ.err_aux[0])!r} rank {summ.err_aux[1]}: duplicate seq {summ.err_aux[2]}")
    if st == _lib.CT_ERR_INVALID_CONFIG:
        order = tuple((config or ModelConfig()).ring_order or ())
        raise InvalidConfig(f"ring order {order} is not a permutation of 0..{len(order) - 1}")
    if st == _lib.CT_ERR_ENDPOINT_RANGE:
        raise EndpointOutOfRange(f"gpu{summ.err_aux[0]} does not fit a {summ.err_aux[1]}-GPU matrix")
    if st == _lib.CT_ERR_OVERFLOW:
        d = summ.d
        a, b = summ.err_aux[0] >> 32, summ.err_aux[0] & 0xFFFFFFFF
        remap = lambda x: 0 if x == 0 else (d + 1 if x == 1 else x - 1)  # noqa: E731
        raise OverflowError(f"cell ({remap(a)},{remap(b)}) exceeds 64-bit byte counter")
    if st == _lib.CT_ERR_WRONG_ALGORITHM:
        raise WrongAlgorithm("collective supports only the ring algorithm")
    if st == _lib.CT_ERR_MISSING_ROOT:
        raise MissingRoot("rooted collective instance has no root")
    raise RuntimeError(f"ct_analyze failed with status {st}")


def _remap(cells: np.ndarray, t: int, g2: int, d: int, agg: bool) -> list[list[int]]:
    """Internal [src][dst] (host 0, net 1, gpu g+2) -> reference layout rows."""
    size = d + 1 + (1 if agg else 0)
    src = [0] + [g + 2 for g in range(d)] + ([1] if agg else [])
    block = cells[t * g2 * g2:(t + 1) * g2 * g2].reshape(g2, g2)
    sub = block[np.ix_(src, src)] if size else block[:0, :0]
    return [[int(v) for v in row] for row in sub.tolist()]


def analyze_packed(trace, d=None, config=None, *, device=None, force_path=_lib.FORCE_AUTO,
                   dev_hint=0, n_comms=None, keep_trace=True) -> AnalysisResult:
    """analyze_events on a PackedTrace (host records) or CUDA tensor of records."""
    config = _config(config)
    ctx = _lib.context(device)
    records = trace.records if isinstance(trace, PackedTrace) else trace
    if n_comms is None:
        n_comms = len(trace.comms) if isinstance(trace, PackedTrace) else 1
    if dev_hint == 0 and isinstance(trace, PackedTrace) and len(trace):
        dev_hint = 16
    ptr, n, on_dev = _lib.records_pointer(records)
    cfg = _lib.make_config(d=d, tree_threshold=config.tree_threshold, ring_order=config.ring_order,
                           force_path=force_path, dev_hint=dev_hint, n_comms=n_comms)
    summ = _lib.CtSummary()
    # CUDA records: run on torch's current stream so kernels that wrote them (clone,
    # cat, index copies in cli / loader) are ordered before the analysis
    stream = _lib.torch_stream(records) if on_dev else None
    rc = ctx.lib.ct_analyze(ctx.handle, C.c_void_p(ptr), n, on_dev, C.byref(cfg), C.byref(summ), stream)
    ctx.check(rc, "ct_analyze")
    if rc != _lib.CT_OK:
        raise_status(summ, trace if isinstance(trace, PackedTrace) else None, config)
    return _build_result(ctx, summ, trace if (keep_trace and isinstance(trace, PackedTrace)) else None)


def _build_result(ctx, summ, trace) -> AnalysisResult:
    d = int(summ.d)
    g2 = int(summ.g_cap) + 2
    ncell = 9 * g2 * g2
    bytes_ = np.zeros(ncell, dtype=np.uint64)
    freq = np.zeros(ncell, dtype=np.uint64)
    rc = ctx.lib.ct_result_cells(ctx.handle, bytes_.ctypes.data, freq.ctypes.data, ncell)
    ctx.check(rc, "ct_result_cells")
    net = int(summ.net_used)
    combined_agg = net != 0
    comb = np.zeros(g2 * g2, dtype=object)
    combf = np.zeros(g2 * g2, dtype=object)
    for t in range(9):
        comb = comb + bytes_[t * g2 * g2:(t + 1) * g2 * g2].astype(object)
        combf = combf + freq[t * g2 * g2:(t + 1) * g2 * g2].astype(object)
    combined = CommMatrix.from_rows(d, _remap(comb, 0, g2, d, combined_agg), combined_agg)
    combined_f = CommMatrix.from_rows(d, _remap(combf, 0, g2, d, combined_agg), combined_agg)
    order = sorted((int(summ.type_first[t]), t) for t in range(9) if summ.calls[t])
    per, perf = {}, {}
    types = {}
    for t, key in enumerate(ALL_TYPES):
        calls = int(summ.calls[t])
        payload = int(summ.payload_lo[t]) + (int(summ.payload_hi[t]) << 64)
        wire = int(bytes_[t * g2 * g2:(t + 1) * g2 * g2].astype(object).sum()) if calls else 0
        types[key] = TypeStats(calls, payload, wire)
    for _, t in order:
        agg = bool(net >> t & 1)
        per[ALL_TYPES[t]] = CommMatrix.from_rows(d, _remap(bytes_, t, g2, d, agg), agg)
        perf[ALL_TYPES[t]] = CommMatrix.from_rows(d, _remap(freq, t, g2, d, agg), agg)
    n_inst = sum(int(summ.calls[t]) for t in range(5))
    stats = StatsSummary(types=types, instances=n_inst, diagnostics=int(sum(summ.diag)))
    timing = {"ms_total": summ.ms_total, "ms_kernel": summ.ms_kernel, "launches": summ.n_launches}
    return AnalysisResult(d, combined, per, stats, combined_f, perf, trace=trace,
                          path=int(summ.path), timing=timing)


def analyze_events(events, d: int | None = None, config: ModelConfig = ModelConfig()) -> AnalysisResult:
    """Group, decompose and accumulate a parsed trace (matrix.py:316-347) on the GPU."""
    trace = events if isinstance(events, PackedTrace) else pack_events(events)
    return analyze_packed(trace, d=d, config=config)


def infer_device_count(events) -> int:
    """Smallest d fitting every device id / GPU endpoint (matrix.py:250-258)."""
    trace = events if isinstance(events, PackedTrace) else pack_events(events)
    ctx = _lib.context()
    ptr, n, on_dev = _lib.records_pointer(trace.records)
    out = C.c_int64()
    rc = ctx.lib.ct_infer_device_count(ctx.handle, C.c_void_p(ptr), n, on_dev, C.byref(out))
    ctx.check(rc, "ct_infer_device_count")
    return int(out.value)


def _instances_trace(instances, events) -> PackedTrace:
    """Canonical blocks for a caller-supplied instance list plus the non-collective
    events: the form split_by_primitive / summarize decompose (matrix.py:225-247)."""
    from .events import EventKind, TraceEvent

    synth = []
    for k, inst in enumerate(instances):
        for r in range(inst.n_ranks):
            synth.append(TraceEvent(seq=k, ts_ns=0, kind=EventKind.COLLECTIVE, comm=inst.comm,
                                    n_ranks=inst.n_ranks, rank=r, device=inst.per_rank_devices[r],
                                    collective=inst.collective, algorithm=inst.algorithm,
                                    root=inst.root, count=inst.count, dtype=inst.dtype))
    others = [e for e in events if getattr(e.kind, "value", e.kind) != "collective"]
    return pack_events(synth + others)


def _list_type_order(instances, events, per: dict) -> dict:
    """Re-key a per-type dict into the reference's first-occurrence order over the
    caller's lists (matrix.py:225-247, 271-276): collective types by their first
    instance in ``instances`` (list order), then sendrecv, then the copy types by their
    first event -- not by the device's comm-major grouping order."""
    rank = {}
    for k, inst in enumerate(instances):
        rank.setdefault(getattr(inst.collective, "value", inst.collective), k)
    rank[SENDRECV] = len(instances)
    copy_type = {"memcpy": EXPLICIT, "um": UNIFIED, "zerocopy": ZEROCOPY}
    for k, ev in enumerate(events):
        t = copy_type.get(getattr(ev.kind, "value", ev.kind))
        if t is not None:
            rank.setdefault(t, len(instances) + 1 + k)
    return {t: per[t] for t in sorted(per, key=rank.__getitem__)}


def split_by_primitive(instances, events, d=None, config: ModelConfig = ModelConfig()) -> dict:
    """One matrix per communication type present (matrix.py:261-276)."""
    if d is None:
        d = infer_device_count(events)
    per = analyze_packed(_instances_trace(instances, events), d=d, config=config).per_primitive
    return _list_type_order(instances, events, per)


def summarize(instances, events, config: ModelConfig = ModelConfig(), diagnostics=None) -> StatsSummary:
    """Calls / payload / wire per type (matrix.py:279-301)."""
    trace = _instances_trace(instances, events)
    res = analyze_packed(trace, d=None, config=config)
    n_p2p = res.stats.diagnostics  # only p2p problems can arise from canonical blocks
    return StatsSummary(types=res.stats.types, instances=len(instances),
                        diagnostics=n_p2p + (len(diagnostics) if diagnostics else 0))
