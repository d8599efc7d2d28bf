"""Multi-GPU analysis: one process per GPU, record-range shards, one small exchange.

Canonical-layout traces (instance blocks contiguous, as the reference's generators and
the device generators write them) shard by record range at element boundaries
(``element_boundary`` finds them on any canonical trace): every rank analyses its own
slice with the fused kernel, exports a fixed-size uint64 partial (cells, statistics,
first-occurrence keys, and the boundary blocks/channels needed to re-check seq order
across shards), the partials are all-gathered once (NCCL over NVLink for GPU tensors;
gloo for CPU tensors in tests), and ``ct_partial_merge`` sums them exactly on the
device — the device-side equivalent of the reference's ``merge`` (matrix.py:164-178),
which is the only cross-thread contract the reference specifies.

Traces in any other layout (an interposer's capture, ranks interleaved) take
``layout="any"``: the global grouping (group_collectives grouping.py:82-183 and
match_p2p decompose.py:342-394 over the WHOLE trace) is computed as per-key ordinal
totals exchanged by two small all-gathers, every record is routed to the rank owning
its position in the global canonical stream by one all-to-all, and each rank analyses
its slice of that stream (``ct_shard_*``, include/commtrace_b200.h).
"""

from __future__ import annotations

import ctypes as C

from . import _lib


def _device_of(records):
    """The CUDA device of a records tensor (torch's current device for host arrays)."""
    import torch

    if getattr(records, "is_cuda", False):
        return records.device.index
    return torch.cuda.current_device()


def shard_bounds(n: int, world: int, boundary) -> list[int]:
    """Element-aligned cut points [0, c1, ..., n] for ``world`` shards; ``boundary(x)``
    returns the first element start at or after record x."""
    cuts = [0]
    for r in range(1, world):
        cuts.append(min(max(boundary(n * r // world), cuts[-1]), n))
    cuts.append(n)
    return cuts


def element_boundary(records, at: int) -> int:
    """First element start at or after record ``at`` of a canonical-layout trace (a
    numpy record array or a CUDA tensor of packed records): ``ct_element_boundary``."""
    ctx = _lib.context(_device_of(records))
    ptr, n, on_dev = _lib.records_pointer(records)
    out = C.c_uint64()
    rc = ctx.lib.ct_element_boundary(ctx.handle, C.c_void_p(ptr), n, on_dev, int(at), C.byref(out))
    ctx.check(rc, "ct_element_boundary")
    return int(out.value)


def canonical_shard(records, world: int, rank: int):
    """This rank's element-aligned record range of a canonical trace held in full."""
    _, n, _ = _lib.records_pointer(records)
    cuts = shard_bounds(n, world, lambda x: element_boundary(records, x))
    return cuts[rank], cuts[rank + 1]


def gather_partials(local, group=None):
    """All-gather equal-size 1-D partials in rank order (NCCL on CUDA tensors, otherwise
    whatever backend the default group uses on CPU tensors)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    out = torch.empty(world * local.numel(), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(out, local, group=group)
    return out


def _gather(t, group):
    """all-gather on the backend's device (gloo gathers host tensors)."""
    import torch
    import torch.distributed as dist

    if dist.get_backend(group) == "nccl":
        return gather_partials(t, group)
    torch.cuda.synchronize()
    return gather_partials(t.cpu(), group).cuda()


def _all_to_all(out, inp, out_splits, in_splits, group):
    import torch
    import torch.distributed as dist

    if dist.get_backend(group) == "nccl":
        dist.all_to_all_single(out, inp, out_splits, in_splits, group=group)
        return out
    torch.cuda.synchronize()
    o = out.cpu()
    dist.all_to_all_single(o, inp.cpu(), out_splits, in_splits, group=group)
    out.copy_(o)
    return out


def route_any_layout(records, n_comms: int, group=None, stream=None):
    """Steps 1-5 of the any-layout flow (include/commtrace_b200.h ``ct_shard_*``): this
    rank's slice of the global canonical stream as a CUDA (m, 32) uint8 tensor."""
    import torch
    import torch.distributed as dist

    ctx = _lib.context(_device_of(records))
    lib = ctx.lib
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    ptr, n, on_dev = _lib.records_pointer(records)
    if not on_dev:
        raise TypeError("route_any_layout needs the shard in device memory")
    st = C.c_void_p(stream if stream is not None else torch.cuda.current_stream().cuda_stream)
    mw, cw = C.c_uint64(), C.c_uint64()
    lib.ct_shard_words(n_comms, C.byref(mw), C.byref(cw))
    meta = torch.empty(mw.value, dtype=torch.int64, device="cuda")
    ctx.check(lib.ct_shard_meta(ctx.handle, C.c_void_p(ptr), n, n_comms, C.c_void_p(meta.data_ptr()), st),
              "ct_shard_meta")
    metas = _gather(meta, group)
    cnt = torch.empty(cw.value, dtype=torch.int64, device="cuda")
    ctx.check(lib.ct_shard_count(ctx.handle, C.c_void_p(ptr), n, n_comms, C.c_void_p(metas.data_ptr()), world,
                                 C.c_void_p(cnt.data_ptr()), st), "ct_shard_count")
    counts = _gather(cnt, group)
    out_pos = torch.empty(max(n, 1), dtype=torch.int64, device="cuda")
    out_rec = torch.empty((max(n, 1), 32), dtype=torch.uint8, device="cuda")
    send, recv, part_len = (C.c_uint64 * world)(), (C.c_uint64 * world)(), C.c_uint64()
    ctx.check(lib.ct_shard_route(ctx.handle, n_comms, C.c_void_p(metas.data_ptr()), C.c_void_p(counts.data_ptr()),
                                 world, rank, C.c_void_p(out_pos.data_ptr()), C.c_void_p(out_rec.data_ptr()), send,
                                 recv, C.byref(part_len), st), "ct_shard_route")
    send_s, recv_s = [int(x) for x in send], [int(x) for x in recv]
    n_in = sum(recv_s)
    in_pos = torch.empty(max(n_in, 1), dtype=torch.int64, device="cuda")
    in_rec = torch.empty((max(n_in, 1), 32), dtype=torch.uint8, device="cuda")
    k = sum(send_s)
    _all_to_all(in_pos[:n_in], out_pos[:k], recv_s, send_s, group)
    _all_to_all(in_rec[:n_in], out_rec[:k], recv_s, send_s, group)
    part = torch.empty((max(part_len.value, 1), 32), dtype=torch.uint8, device="cuda")
    ctx.check(lib.ct_shard_assemble(ctx.handle, C.c_void_p(in_pos.data_ptr()), C.c_void_p(in_rec.data_ptr()), n_in,
                                    C.c_void_p(part.data_ptr()), st), "ct_shard_assemble")
    return part[: part_len.value]


def analyze_sharded(records, n_comms: int = 1, d=None, dev_hint: int = 8, tree_threshold: int = 1 << 20,
                    ring_order=None, group=None, stream=None, layout: str = "canonical"):
    """Analyze this rank's shard (a CUDA tensor of packed records) and merge all ranks'
    partials; every rank returns the merged ``CtSummary`` (cells stay in the context).

    ``layout="canonical"``: shards are element-aligned record ranges of a canonical
    trace (``canonical_shard``).  ``layout="any"``: shards are arbitrary record ranges
    (in rank order) of a trace in any layout; records are first routed to the rank
    owning their position in the global canonical stream.

    All ranks must use the same ``d`` / ``dev_hint`` so the partial layouts agree."""
    import torch
    import torch.distributed as dist

    ctx = _lib.context(_device_of(records))
    # Everything runs on ONE stream -- torch's current one unless the caller names
    # another: the async export, the NCCL all-gather (enqueued by torch on its current
    # stream) and the merge are then ordered without extra events.
    if stream is None:
        stream = torch.cuda.current_stream().cuda_stream
    elif stream != torch.cuda.current_stream().cuda_stream:
        torch.cuda.current_stream().synchronize()  # records written by torch work
    force = _lib.FORCE_AUTO
    if layout == "any":
        records = route_any_layout(records, n_comms, group=group, stream=stream)
        force = _lib.FORCE_FAST  # a slice of the canonical stream
    elif layout != "canonical":
        raise ValueError(f"unknown layout {layout!r}")
    ptr, n, on_dev = _lib.records_pointer(records)
    cfg = _lib.make_config(d=d, tree_threshold=tree_threshold, ring_order=ring_order, dev_hint=dev_hint,
                           n_comms=n_comms, force_path=force)
    s = _lib.CtSummary()
    st = C.c_void_p(stream)
    rc = ctx.lib.ct_analyze(ctx.handle, C.c_void_p(ptr), n, on_dev, C.byref(cfg), C.byref(s), st)
    ctx.check(rc, "ct_analyze")
    words = C.c_uint64()
    ctx.lib.ct_partial_size(ctx.handle, C.byref(words))
    part = torch.empty(words.value, dtype=torch.int64, device="cuda")
    rc = ctx.lib.ct_partial_export(ctx.handle, C.c_void_p(part.data_ptr()), words.value, st)
    ctx.check(rc, "ct_partial_export")
    backend = dist.get_backend(group)
    cur = torch.cuda.current_stream()
    if stream != cur.cuda_stream:  # the export ran on the caller's stream: order the gather after it
        cur.wait_stream(torch.cuda.ExternalStream(stream))
    if backend == "nccl":
        allp = gather_partials(part, group)
    else:  # gloo and friends gather host tensors
        torch.cuda.synchronize()
        allp = gather_partials(part.cpu(), group).cuda()
    if stream != cur.cuda_stream:  # and the merge after the gather
        torch.cuda.ExternalStream(stream).wait_stream(cur)
    merged = _lib.CtSummary()
    rc = ctx.lib.ct_partial_merge(ctx.handle, C.c_void_p(allp.data_ptr()), dist.get_world_size(group),
                                  words.value, C.byref(merged), st)
    ctx.check(rc, "ct_partial_merge")
    return merged
