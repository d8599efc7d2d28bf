"""Multi-GPU paths on one device (tests/test_dist_cpu.py covers the host plumbing).

* any layout (``ct_shard_*``): a capture-layout trace cut into arbitrary record ranges
  (4 simulated ranks, one context each, the all-gathers / all-to-all emulated by
  slicing) -> routed parts -> per-part analysis -> partial merge equals the single-GPU
  analysis of the whole trace, cell for cell;
* canonical layout on a LOADED trace (not a generator): element-aligned cuts from the
  device boundary finder (``dist.element_boundary``);
* two real processes (gloo, sharing the GPU) through ``dist.analyze_sharded`` in both
  layouts."""

import ctypes as C
import os
import socket

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


def _single(buf, n, n_comms):
    from paper_2110_10401_b200 import _lib
    ctx = _lib.context(0)
    cfg = _lib.make_config(dev_hint=8, n_comms=n_comms)
    s = _lib.CtSummary()
    assert ctx.lib.ct_analyze(ctx.handle, C.c_void_p(buf.data_ptr()), n, 1, C.byref(cfg), C.byref(s), None) == 0
    g2 = s.g_cap + 2
    cells = np.zeros(2 * 9 * g2 * g2, np.uint64)
    assert ctx.lib.ct_result_cells(ctx.handle, cells.ctypes.data, cells.ctypes.data + 9 * g2 * g2 * 8,
                                   9 * g2 * g2) == 0
    return s, cells


def _cells(lib, h, g2):
    cells = np.zeros(2 * 9 * g2 * g2, np.uint64)
    assert lib.ct_result_cells(h, cells.ctypes.data, cells.ctypes.data + 9 * g2 * g2 * 8, 9 * g2 * g2) == 0
    return cells


def _same_summary(a, b):
    for f in ("calls", "payload_lo", "payload_hi", "diag", "type_first"):
        assert list(getattr(a, f)) == list(getattr(b, f)), f
    assert a.d == b.d and a.net_used == b.net_used and a.status == b.status


def _routed_merge(buf, n, n_comms, cuts):
    """Simulate len(cuts)-1 ranks (one context each) through the ct_shard_* flow."""
    import torch
    from paper_2110_10401_b200 import _lib
    lib = _lib.load()
    world = len(cuts) - 1
    hs = []
    for _ in range(world):
        h = C.c_void_p()
        assert lib.ct_context_create(0, C.byref(h)) == 0
        hs.append(h)
    mw, cw = C.c_uint64(), C.c_uint64()
    lib.ct_shard_words(n_comms, C.byref(mw), C.byref(cw))
    shards = [buf[a * 32:b * 32] for a, b in zip(cuts[:-1], cuts[1:])]
    metas = []
    for r in range(world):
        m = torch.empty(mw.value, dtype=torch.int64, device="cuda")
        assert lib.ct_shard_meta(hs[r], C.c_void_p(shards[r].data_ptr()), shards[r].numel() // 32, n_comms,
                                 C.c_void_p(m.data_ptr()), None) == 0
        metas.append(m)
    allm = torch.cat(metas)
    counts = []
    for r in range(world):
        c = torch.empty(cw.value, dtype=torch.int64, device="cuda")
        rc = lib.ct_shard_count(hs[r], C.c_void_p(shards[r].data_ptr()), shards[r].numel() // 32, n_comms,
                                C.c_void_p(allm.data_ptr()), world, C.c_void_p(c.data_ptr()), None)
        assert rc == 0, lib.ct_last_error(hs[r])
        counts.append(c)
    allc = torch.cat(counts)
    outs, sends, recvs, plens = [], [], [], []
    for r in range(world):
        k = max(shards[r].numel() // 32, 1)
        pos = torch.empty(k, dtype=torch.int64, device="cuda")
        rec = torch.empty((k, 32), dtype=torch.uint8, device="cuda")
        send, recv, plen = (C.c_uint64 * world)(), (C.c_uint64 * world)(), C.c_uint64()
        rc = lib.ct_shard_route(hs[r], n_comms, C.c_void_p(allm.data_ptr()), C.c_void_p(allc.data_ptr()), world, r,
                                C.c_void_p(pos.data_ptr()), C.c_void_p(rec.data_ptr()), send, recv, C.byref(plen),
                                None)
        assert rc == 0, lib.ct_last_error(hs[r])
        outs.append((pos, rec))
        sends.append(list(send))
        recvs.append(list(recv))
        plens.append(plen.value)
    for r in range(world):  # counts agree between senders and receivers
        assert [sends[s][r] for s in range(world)] == recvs[r]
    parts = []
    for r in range(world):  # emulated all-to-all
        pos_in, rec_in = [], []
        for s in range(world):
            off = sum(sends[s][:r])
            pos_in.append(outs[s][0][off:off + sends[s][r]])
            rec_in.append(outs[s][1][off:off + sends[s][r]])
        pin, rin = torch.cat(pos_in), torch.cat(rec_in)
        part = torch.empty((max(plens[r], 1), 32), dtype=torch.uint8, device="cuda")
        rc = lib.ct_shard_assemble(hs[r], C.c_void_p(pin.data_ptr()), C.c_void_p(rin.data_ptr()), pin.shape[0],
                                   C.c_void_p(part.data_ptr()), None)
        assert rc == 0, lib.ct_last_error(hs[r])
        parts.append(part)
    assert sum(plens) == sum(p for p in plens)
    words = C.c_uint64()
    partials = []
    for r in range(world):
        cfg = _lib.make_config(dev_hint=8, n_comms=n_comms, force_path=1)
        s = _lib.CtSummary()
        rc = lib.ct_analyze(hs[r], C.c_void_p(parts[r].data_ptr()), plens[r], 1, C.byref(cfg), C.byref(s), None)
        assert rc == 0, lib.ct_last_error(hs[r])
        lib.ct_partial_size(hs[r], C.byref(words))
        p = torch.empty(words.value, dtype=torch.int64, device="cuda")
        assert lib.ct_partial_export(hs[r], C.c_void_p(p.data_ptr()), words.value, None) == 0
        torch.cuda.synchronize()
        partials.append(p)
    allp = torch.cat(partials)
    m = _lib.CtSummary()
    rc = lib.ct_partial_merge(hs[0], C.c_void_p(allp.data_ptr()), world, words.value, C.byref(m), None)
    assert rc == 0, lib.ct_last_error(hs[0])
    cells = _cells(lib, hs[0], m.g_cap + 2)
    for h in hs:
        lib.ct_context_destroy(h)
    return m, cells


@pytest.mark.parametrize("kind,n_comms,n", [(6, 1, 2_000_000), (6, 1, 300_001), (3, 3, 400_000)])
def test_any_layout_routed_merge_equals_single(kind, n_comms, n):
    """Capture layout (kind 6: cut mid-epoch too) and a canonical C3 cut at arbitrary,
    NOT element-aligned record offsets."""
    buf = _gen(kind, n, seed=9)
    s, cells = _single(buf, n, n_comms)
    cuts = [0, n // 5 + 3, n // 2 + 1, 3 * n // 4 + 7, n]
    m, mcells = _routed_merge(buf, n, n_comms, cuts)
    assert np.array_equal(mcells, cells)
    _same_summary(m, s)


def test_canonical_cuts_on_loaded_trace():
    """Element-aligned cuts of a trace loaded from JSONL (no generator boundary)."""
    import torch
    from paper_2110_10401_b200 import _lib
    from paper_2110_10401_b200.dist import canonical_shard
    from paper_2110_10401_b200.events import write_trace
    from paper_2110_10401_b200.loader import load_trace
    from paper_2110_10401_b200.packed import PackedTrace, RECORD_DTYPE, unpack
    n0 = 60_000
    buf = _gen(3, n0, seed=2)
    rec = np.frombuffer(buf.cpu().numpy().tobytes(), dtype=RECORD_DTYPE).copy()
    text = write_trace(unpack(PackedTrace(rec, ["c0", "c1", "c2"], list(range(n0)), None)))
    tr = load_trace(text)
    recs = tr.records.reshape(-1)
    n = len(tr)
    s, cells = _single(recs, n, 3)
    ctx = _lib.context(0)
    world = 4
    parts = []
    words = C.c_uint64()
    for r in range(world):
        a, b = canonical_shard(tr.records, world, r)
        sub = recs[a * 32:b * 32]
        cfg = _lib.make_config(dev_hint=8, n_comms=3, force_path=1)
        ss = _lib.CtSummary()
        assert ctx.lib.ct_analyze(ctx.handle, C.c_void_p(sub.data_ptr()), b - a, 1, C.byref(cfg), C.byref(ss),
                                  None) == 0
        ctx.lib.ct_partial_size(ctx.handle, C.byref(words))
        p = torch.empty(words.value, dtype=torch.int64, device="cuda")
        assert ctx.lib.ct_partial_export(ctx.handle, C.c_void_p(p.data_ptr()), words.value, None) == 0
        torch.cuda.synchronize()
        parts.append(p)
    allp = torch.cat(parts)
    m = _lib.CtSummary()
    assert ctx.lib.ct_partial_merge(ctx.handle, C.c_void_p(allp.data_ptr()), world, words.value, C.byref(m),
                                    None) == 0
    assert np.array_equal(_cells(ctx.lib, ctx.handle, m.g_cap + 2), cells)
    _same_summary(m, s)


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _worker(rank, world, port, kind, n, n_comms, layout, out):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2110_10401_b200 import _lib
        from paper_2110_10401_b200.dist import analyze_sharded
        torch.cuda.set_device(0)
        ctx = _lib.context(0)
        if layout == "any":
            a, b = n * rank // world + rank, n * (rank + 1) // world + (rank + 1 if rank + 1 < world else 0)
            b = min(b, n)
        else:
            a = ctx.lib.ct_generate_boundary(kind, n * rank // world)
            b = ctx.lib.ct_generate_boundary(kind, n * (rank + 1) // world) if rank + 1 < world else n
        buf = torch.empty(max(b - a, 1) * 32, dtype=torch.uint8, device="cuda")
        assert ctx.lib.ct_generate(ctx.handle, kind, 9, a, b - a, C.c_void_p(buf.data_ptr()), None) == 0
        torch.cuda.synchronize()
        m = analyze_sharded(buf[: (b - a) * 32], n_comms=n_comms, layout=layout)
        g2 = m.g_cap + 2
        cells = np.zeros(2 * 9 * g2 * g2, np.uint64)
        ctx.lib.ct_result_cells(ctx.handle, cells.ctypes.data, cells.ctypes.data + 9 * g2 * g2 * 8, 9 * g2 * g2)
        out[rank] = (cells.tobytes(), [int(x) for x in m.calls], [int(x) for x in m.diag], int(m.d))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("layout,kind,n_comms", [("any", 6, 1), ("canonical", 3, 3)])
def test_two_processes_gloo(layout, kind, n_comms):
    import torch.multiprocessing as mp
    n = 1_000_000
    buf = _gen(kind, n, seed=9)
    s, cells = _single(buf, n, n_comms)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), kind, n, n_comms, layout, out), nprocs=2, join=True)
    for r in range(2):
        c, calls, diag, d = out[r]
        assert np.frombuffer(c, np.uint64).tolist() == cells.tolist()
        assert calls == [int(x) for x in s.calls] and diag == [int(x) for x in s.diag] and d == s.d
