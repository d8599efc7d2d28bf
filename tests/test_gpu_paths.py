"""GPU parity for the fast kernel's internal paths, against the C restatement of the
reference (oracle/ct_oracle.c) on the same packed records:

* mixed canonical traces (all collectives and algorithms, n = 1..8, p2p pairs, copies,
  in-layout diagnostics: incompatible blocks, duplicate devices, mismatched pairs) whose
  per-communicator devices change now and then -- exercises the per-lane ring
  accumulator's key changes and flushes;
* devices >= 64 and > 16 GPUs (pairwise distinctness fallback, global-atomics histogram);
* communicators of up to 32 ranks and a configured ring order (decompose.py:110-116);
* collective counts >= 2^40 (128-bit byte counts);
* a cell overflow reached only through accumulated repeats (matrix.py:108-113).
"""

import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

# (kind, coll) codes of include/commtrace_b200.h
COLL, SEND, RECV, MEMCPY = 0, 1, 2, 3
AR, BC, RD, RS, AG = 0, 1, 2, 3, 4
RING, TREE, COLLNET, AUTO = 0, 1, 2, 3


def _rec(out, count, seq, comm, n, rank, dev, aux=0, aux2=0, kind=COLL, coll=0, root=False, algo=0, dtype=8,
         ck=0):
    kc = kind | (coll << 3) | ((1 << 6) if root else 0)
    ad = algo | (dtype << 2) | (ck << 6)
    out.append((count, seq, comm, n, rank, dev, aux, aux2, kc, ad))


class Gen:
    """Canonical-layout trace builder (blocks contiguous in rank order, per-(comm, rank)
    seq increasing, p2p channels FIFO)."""

    def __init__(self, rng, n_comms, max_n=8, dev_pool=8, wide=0.0, diag=0.0, dev_change=0.01, ragged=0.0):
        self.rng, self.recs = rng, []
        self.ragged = ragged  # probability that a block's ranks carry different seqs
        self.wide, self.diag, self.dev_change, self.dev_pool = wide, diag, dev_change, dev_pool
        self.n = [int(rng.integers(1, max_n + 1)) for _ in range(n_comms)]
        self.devs = [self._perm(n) for n in self.n]
        self.seq = [0] * n_comms
        self.rseq = [[0] * 32 for _ in range(n_comms)]  # per-(comm, rank) counters
        self.p2p_comm, self.copy_comm = n_comms, n_comms + 1
        self.chan = {}

    def _perm(self, n):
        return [int(x) for x in self.rng.permutation(self.dev_pool)[:n]]

    def block(self, c):
        rng = self.rng
        n = self.n[c]
        if rng.random() < self.dev_change:
            self.devs[c] = self._perm(n)
        coll = int(rng.integers(0, 5))
        algo = int(rng.integers(0, 4)) if coll == AR else RING
        dtype = int(rng.integers(0, 10))
        count = int(rng.integers(1 << 40, 1 << 42)) if rng.random() < self.wide else int(2 ** rng.uniform(0, 24))
        rooted = coll in (BC, RD)
        root = int(rng.integers(0, n))
        seq = self.seq[c] = max(self.seq[c], max(self.rseq[c][:n])) + int(rng.integers(1, 3))
        if rng.random() < self.ragged:  # per-rank seqs, each still strictly increasing
            seqs = [max(self.rseq[c][r], seq) + int(rng.integers(0, 3)) for r in range(n)]
        else:
            seqs = [seq] * n
        for r in range(n):
            self.rseq[c][r] = seqs[r]
        bad = rng.random() < self.diag
        devs = list(self.devs[c])
        if bad and n > 1 and rng.random() < 0.5:
            devs[1] = devs[0]  # duplicate device
            bad = False
        for r in range(n):
            cnt = count + (1 if bad and r == n - 1 else 0)  # incompatible signature
            _rec(self.recs, cnt, seqs[r], c, n, r, devs[r], aux=root if rooted else 0, coll=coll, root=rooted,
                 algo=algo, dtype=dtype)

    def pair(self):
        rng = self.rng
        a, b = (int(x) for x in rng.choice(8, 2, replace=False))
        key = (a, b)
        s = self.chan[key] = self.chan.get(key, 0) + 1
        count, dtype = int(2 ** rng.uniform(0, 20)), int(rng.integers(0, 10))
        mis = rng.random() < self.diag
        _rec(self.recs, count, s, self.p2p_comm, 8, a, a % 6, aux=b, kind=SEND, dtype=dtype)
        _rec(self.recs, count + (1 if mis else 0), s, self.p2p_comm, 8, b, b % 6, aux=a, kind=RECV, dtype=dtype)

    def copy(self):
        rng = self.rng
        kind, ck = MEMCPY + int(rng.integers(0, 3)), int(rng.integers(0, 3))
        a, b = (int(x) for x in rng.choice(8, 2, replace=False))
        _rec(self.recs, int(2 ** rng.uniform(0, 30)), 0, self.copy_comm, 1, 0, a, aux=0 if ck == 0 else a,
             aux2=0 if ck == 1 else b, kind=kind, ck=ck)

    def mixed(self, n_records, p_pair=0.1, p_copy=0.2):
        rng = self.rng
        while len(self.recs) < n_records:
            u = rng.random()
            if u < p_pair:
                self.pair()
            elif u < p_pair + p_copy:
                self.copy()
            else:
                self.block(int(rng.integers(0, len(self.n))))
        return self

    def array(self):
        from paper_2110_10401_b200.packed import RECORD_DTYPE
        return np.array(self.recs, dtype=RECORD_DTYPE)


def _gpu(recs, n_comms, d=None, ring_order=None, force=1, dev_hint=8):
    from paper_2110_10401_b200 import _lib
    ctx = _lib.context(0)
    cfg = _lib.make_config(d=d, ring_order=ring_order, dev_hint=dev_hint, n_comms=n_comms, force_path=force)
    s = _lib.CtSummary()
    rc = ctx.lib.ct_analyze(ctx.handle, C.c_void_p(recs.ctypes.data), recs.shape[0], 0, C.byref(cfg), C.byref(s),
                            None)
    assert rc in (0, 3, 4), ctx.error()
    g2 = s.g_cap + 2
    cells = np.zeros(9 * g2 * g2, np.uint64)
    freq = np.zeros(9 * g2 * g2, np.uint64)
    assert ctx.lib.ct_result_cells(ctx.handle, cells.ctypes.data, freq.ctypes.data, cells.size) == 0
    return s, cells, freq


def _check(recs, n_comms, d=None, ring_order=None):
    from oracle import c_oracle as CO
    s, cells, freq = _gpu(recs, n_comms, d=d, ring_order=ring_order)
    assert s.path == 1, "canonical trace must take the fast path"
    want = CO.analyze_records(recs, d=d, ring_order=ring_order, gcap=s.g_cap)
    want_status = want["status"] or (4 if want["overflow"] else 0)  # CT_ERR_OVERFLOW
    assert s.status == want_status, (s.status, want_status)
    if s.status:
        return s, want
    assert s.d == want["d"]
    assert np.array_equal(cells, want["cells"])
    assert np.array_equal(freq, want["freq"])
    for t in range(9):
        assert s.calls[t] == int(want["calls"][t]), t
        assert s.payload_lo[t] + (s.payload_hi[t] << 64) == want["payload"][t], t
    assert [int(x) for x in s.diag] == [int(x) for x in want["diag"]]
    return s, want


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_mixed_canonical_with_diagnostics(seed):
    rng = np.random.default_rng(seed)
    g = Gen(rng, n_comms=6, diag=0.02, dev_change=0.02, ragged=0.3 if seed else 0.0).mixed(600_000)
    s, _ = _check(g.array(), n_comms=6)
    assert sum(s.diag) > 0


def test_slot_accumulator_write_outs(monkeypatch):
    """Many communicators of different sizes (the per-lane accumulator cannot hold them;
    the warp's slot accumulators do) with the write-out threshold forced down to 3
    instances, so full entries are written out and re-keyed all the time."""
    monkeypatch.setenv("CT_SA_FLUSH", "3")
    rng = np.random.default_rng(9)
    g = Gen(rng, n_comms=7, dev_change=0.005)
    g.n = [2, 3, 4, 5, 6, 7, 8]
    g.devs = [g._perm(n) for n in g.n]
    g.mixed(400_000, p_pair=0.02, p_copy=0.02)
    _check(g.array(), n_comms=7)


def test_repeated_ring_blocks_with_device_changes():
    """Long runs of identical ring allreduce / allgather / reduce-scatter instances (the
    register accumulator's case), with the devices and types changing between runs."""
    rng = np.random.default_rng(5)
    g = Gen(rng, n_comms=3, max_n=8)
    g.n = [8, 5, 2]
    g.devs = [g._perm(n) for n in g.n]
    recs = g.recs
    for run in range(400):
        c = run % 3
        n = g.n[c]
        if run % 7 == 0:
            g.devs[c] = g._perm(n)
        coll = [AR, AG, RS][run % 3]
        count = int(rng.integers(1, 1 << 20))
        for _ in range(int(rng.integers(1, 200))):
            seq = g.seq[c] = g.seq[c] + 1
            for r in range(n):
                _rec(recs, count, seq, c, n, r, g.devs[c][r], coll=coll, algo=RING, dtype=8)
    _check(g.array(), n_comms=3)


def test_large_device_ids_global_histogram():
    """Devices >= 64 (pairwise distinctness fallback) and d > 16 (global-atomics cells)."""
    rng = np.random.default_rng(3)
    g = Gen(rng, n_comms=4, dev_pool=70, diag=0.02).mixed(300_000)
    _check(g.array(), n_comms=4)
    _check(g.array(), n_comms=4, d=72)


def test_wide_communicators_and_ring_order():
    rng = np.random.default_rng(4)
    g = Gen(rng, n_comms=3, max_n=32, dev_pool=32)
    g.n = [32, 8, 17]
    g.devs = [g._perm(n) for n in g.n]
    g.mixed(400_000, p_pair=0.05, p_copy=0.05)
    order = [int(x) for x in rng.permutation(8)]
    _check(g.array(), n_comms=3)
    _check(g.array(), n_comms=3, ring_order=order)


def test_wide_counts():
    rng = np.random.default_rng(6)
    g = Gen(rng, n_comms=3, wide=0.05).mixed(200_000)
    _check(g.array(), n_comms=3)


def test_overflow_through_accumulated_repeats():
    """2-rank ring allreduce of 2^39 float64 elements: every edge carries 2^42 bytes, so
    2^21 identical instances push both cells past 2^63 - 1 (OverflowError)."""
    from paper_2110_10401_b200.packed import RECORD_DTYPE
    k = (1 << 21) + 8
    recs = np.zeros(2 * k, dtype=RECORD_DTYPE)
    recs["count"] = 1 << 39
    recs["seq"] = np.repeat(np.arange(1, k + 1, dtype=np.uint64), 2)
    recs["nranks"] = 2
    recs["rank"] = np.tile(np.array([0, 1], np.uint16), k)
    recs["dev"] = recs["rank"]
    recs["ad"] = 9 << 2  # float64, ring
    s, want = _check(recs, n_comms=1)
    assert s.status == 4 and want["overflow"]
    # one instance fewer than the bound stays exact
    m = (1 << 21) - 1
    _check(recs[:2 * m], n_comms=1)


def _check_any_path(recs, n_comms, d=None):
    """Like _check, but the trace may exceed the fast path's per-warp capacities: the host
    then re-runs through the exact (sort-based) path; results must still match."""
    from oracle import c_oracle as CO
    s, cells, freq = _gpu(recs, n_comms, d=d, force=0)
    want = CO.analyze_records(recs, d=d, gcap=s.g_cap)
    want_status = want["status"] or (4 if want["overflow"] else 0)
    assert s.status == want_status
    assert np.array_equal(cells, want["cells"]) and np.array_equal(freq, want["freq"])
    for t in range(9):
        assert s.calls[t] == int(want["calls"][t]), t
    return s


def test_capacity_fallbacks_match():
    """> 8 communicators interleaved within one warp range (comm slots) and communicators
    totalling > 64 ranks (pooled seq tables) leave the fast path; the answer is the same."""
    rng = np.random.default_rng(11)
    g = Gen(rng, n_comms=12, max_n=4).mixed(20_000, p_pair=0.0, p_copy=0.0)
    s = _check_any_path(g.array(), n_comms=12)
    assert s.path in (2, 3)  # the counting canonicaliser or the exact join
    g = Gen(rng, n_comms=3, max_n=32, dev_pool=32)
    g.n = [32, 32, 32]
    g.devs = [g._perm(32) for _ in range(3)]
    g.mixed(20_000, p_pair=0.0, p_copy=0.0)
    s = _check_any_path(g.array(), n_comms=3)
    assert s.path in (2, 3)
