"""Capture-layout traces (ranks interleaved the way an LD_PRELOAD interposer writes them:
each process appends its own calls in order, processes interleave) through the counting
canonicaliser (csrc/ct_canon.cu, path 3).

* the device generator's C4 capture layout (kind 6) equals the canonical C4 analysis
  over the same records, at 100M records, and the C oracle over epoch-aligned shards;
* C2 / C3 / C5 traces re-ordered on the host by a random merge of per-process streams
  (per-(comm, rank) and per-channel order kept) analyse exactly like the canonical file,
  including p2p pairs, copies and diagnostics;
* a per-rank seq inversion or a nranks disagreement leaves the counting path for the
  exact one (the results still match the C oracle / the reference's error)."""

import ctypes as C
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _gen(kind, n, seed=7):
    import torch
    from paper_2110_10401_b200 import _lib
    ctx = _lib.context(0)
    buf = torch.empty(n * 32, dtype=torch.uint8, device="cuda")
    assert ctx.lib.ct_generate(ctx.handle, kind, seed, 0, n, C.c_void_p(buf.data_ptr()), None) == 0
    torch.cuda.synchronize()
    return buf


def _analyze(buf, n, n_comms, force=0, d=None):
    from paper_2110_10401_b200 import _lib
    ctx = _lib.context(0)
    cfg = _lib.make_config(d=d, dev_hint=8, n_comms=n_comms, force_path=force)
    s = _lib.CtSummary()
    rc = ctx.lib.ct_analyze(ctx.handle, C.c_void_p(buf.data_ptr()), n, 1, C.byref(cfg), C.byref(s), None)
    g2 = s.g_cap + 2
    cells = np.zeros(9 * g2 * g2, np.uint64)
    freq = np.zeros(9 * g2 * g2, np.uint64)
    if rc == 0:
        assert ctx.lib.ct_result_cells(ctx.handle, cells.ctypes.data, freq.ctypes.data, cells.size) == 0
    return rc, s, cells, freq


def _same(a, b, copies_from=None):
    """Equal results; the copy types' dict positions follow the file's own copy order
    (matrix.py:244-246), so a re-ordered file compares them against ``copies_from``."""
    ra, sa, ca, fa = a
    rb, sb, cb, fb = b
    assert ra == rb == 0
    assert np.array_equal(ca, cb) and np.array_equal(fa, fb)
    for f in ("calls", "payload_lo", "payload_hi", "diag"):
        assert list(getattr(sa, f)) == list(getattr(sb, f)), f
    assert list(sa.type_first)[:6] == list(sb.type_first)[:6]
    if copies_from is None:
        assert list(sa.type_first) == list(sb.type_first)
    else:
        kinds = copies_from["kc"] & 7
        first = sorted((int(np.argmax(kinds == 3 + t)), t) for t in range(3) if (kinds == 3 + t).any())
        want = {6 + t: 6 + k for k, (_, t) in enumerate(first)}
        assert {t: int(sa.type_first[t]) for t in want} == want
    assert sa.d == sb.d and sa.net_used == sb.net_used


def test_c4_capture_layout_equals_canonical():
    from paper_2110_10401_b200 import _lib
    lib = _lib.load()
    n = lib.ct_generate_boundary(6, 100_000_000)
    cap = _analyze(_gen(6, n, seed=2), n, 1)
    can = _analyze(_gen(4, n, seed=2), n, 1)
    assert cap[1].path == 3 and can[1].path == 1
    _same(cap, can)


def test_c4_capture_layout_matches_c_oracle():
    from oracle import c_oracle as CO
    from paper_2110_10401_b200 import _lib
    from paper_2110_10401_b200.packed import RECORD_DTYPE
    lib = _lib.load()
    n = lib.ct_generate_boundary(6, 4_000_000)
    buf = _gen(6, n, seed=5)
    rc, s, cells, freq = _analyze(buf, n, 1)
    assert rc == 0 and s.path == 3
    recs = buf.cpu().numpy().view(RECORD_DTYPE)
    step = lib.ct_generate_boundary(6, 1)  # epochs are clean cuts
    bounds = list(range(0, n, step)) + [n]
    want = CO.analyze_threads(recs, bounds, os.cpu_count() or 4, gcap=s.g_cap)
    assert want["status"] == 0 and s.d == want["d"]
    assert np.array_equal(cells.astype(object), np.array(want["cells"], dtype=object))
    assert np.array_equal(freq, want["freq"])
    assert [int(x) for x in s.diag] == [int(x) for x in want["diag"]]


def _process_merge(recs, seed):
    """Random merge of per-process streams (process = the record's device), keeping each
    process's own order -- what O_APPEND lines from one-process-per-GPU jobs look like."""
    rng = np.random.default_rng(seed)
    proc = recs["dev"].astype(np.int64)
    t = np.zeros(len(recs))
    for p in np.unique(proc):
        idx = np.nonzero(proc == p)[0]
        t[idx] = np.cumsum(rng.exponential(1.0, len(idx)))
    return recs[np.argsort(t, kind="stable")]


@pytest.mark.parametrize("kind,n_comms", [(2, 1), (3, 3), (5, 7)])
def test_process_merged_traces_equal_canonical(kind, n_comms):
    import torch
    from paper_2110_10401_b200 import _lib
    from paper_2110_10401_b200.packed import RECORD_DTYPE
    lib = _lib.load()
    n = lib.ct_generate_boundary(kind, 400_000)
    buf = _gen(kind, n, seed=11)
    can = _analyze(buf, n, n_comms)
    recs = buf.cpu().numpy().view(RECORD_DTYPE)
    merged = _process_merge(recs, seed=kind)
    mbuf = torch.from_numpy(merged.view(np.uint8).reshape(-1).copy()).cuda()
    cap = _analyze(mbuf, n, n_comms)
    assert can[1].path == 1 and cap[1].path == 3, (can[1].path, cap[1].path)
    _same(cap, can, copies_from=merged)


def test_truncated_capture_counts_incomplete_groups():
    """A capture cut mid-way: lagging ranks leave incomplete groups (diagnostics)."""
    from oracle import c_oracle as CO
    from paper_2110_10401_b200 import _lib
    from paper_2110_10401_b200.packed import RECORD_DTYPE
    lib = _lib.load()
    n = lib.ct_generate_boundary(6, 1) + 777  # one epoch and a partial one
    buf = _gen(6, n, seed=3)
    rc, s, cells, freq = _analyze(buf, n, 1)
    assert rc == 0 and s.path == 3 and s.diag[0] > 0
    want = CO.analyze_records(buf.cpu().numpy().view(RECORD_DTYPE), gcap=s.g_cap)
    assert np.array_equal(cells.astype(object), np.array(want["cells"], dtype=object))
    assert [int(x) for x in s.diag] == [int(x) for x in want["diag"]]


def test_seq_inversion_takes_exact_path():
    import torch
    from oracle import c_oracle as CO
    from paper_2110_10401_b200 import _lib
    from paper_2110_10401_b200.packed import RECORD_DTYPE
    lib = _lib.load()
    n = lib.ct_generate_boundary(6, 1)
    recs = _gen(6, n, seed=4).cpu().numpy().view(RECORD_DTYPE).copy()
    # swap two records of the same (comm, rank): file order no longer seq order
    r0 = np.nonzero(recs["rank"] == 3)[0]
    a, b = r0[10], r0[11]
    recs[[a, b]] = recs[[b, a]]
    buf = torch.from_numpy(recs.view(np.uint8).reshape(-1).copy()).cuda()
    rc, s, cells, freq = _analyze(buf, n, 1)
    assert rc == 0 and s.path == 2
    want = CO.analyze_records(recs, gcap=s.g_cap)
    assert np.array_equal(cells.astype(object), np.array(want["cells"], dtype=object))
    rc3, *_ = _analyze(buf, n, 1, force=3)
    assert rc3 == 22  # outside the counting path's scope: refused, not misanalysed


def test_key_stride_guess_too_small_recounts():
    """The fused meta + count pass guesses the key stride from the first 1024 records;
    a trace whose early records all come from 2-rank communicators and whose later ones
    reach 8 ranks is counted again with the true stride -- and equals the exact path."""
    import torch
    from paper_2110_10401_b200 import _lib
    from paper_2110_10401_b200.packed import RECORD_DTYPE
    lib = _lib.load()
    n = lib.ct_generate_boundary(5, 200_000)
    recs = _gen(5, n, seed=13).cpu().numpy().view(RECORD_DTYPE)
    small = recs[recs["nranks"] == 2]
    rest = recs[recs["nranks"] != 2]
    assert len(small) > 2048
    merged = np.concatenate([_process_merge(small, seed=1), _process_merge(rest, seed=2)])
    buf = torch.from_numpy(merged.view(np.uint8).reshape(-1).copy()).cuda()
    cap = _analyze(buf, n, 7)
    exact = _analyze(buf, n, 7, force=2)
    assert cap[1].path == 3 and exact[1].path == 2
    _same(cap, exact)
