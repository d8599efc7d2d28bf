"""Multi-GPU analysis: one process per GPU, record-range shards, one small exchange.

The trace shards by record range: every rank analyses its own
element-aligned slice with the fused kernel, exports a fixed-size uint64 partial
(cells, statistics, first-occurrence keys, and the boundary blocks/channels needed to
re-check seq order across shards), the partials are all-gathered once (NCCL over
NVLink for GPU tensors; gloo for CPU tensors in tests), and ``ct_partial_merge`` sums
them exactly on the device — the device-side equivalent of the reference's
``merge`` (matrix.py:164-178), which is the only cross-thread contract the reference
specifies.
"""

from __future__ import annotations

import ctypes as C

from . import _lib


def shard_bounds(n: int, world: int, boundary) -> list[int]:
    """Element-aligned cut points [0, c1, ..., n] for ``world`` shards; ``boundary(x)``
    returns the first element start at or after record x."""
    cuts = [0]
    for r in range(1, world):
        cuts.append(min(max(boundary(n * r // world), cuts[-1]), n))
    cuts.append(n)
    return cuts


def gather_partials(local, group=None):
    """All-gather equal-size 1-D partials in rank order (NCCL on CUDA tensors, otherwise
    whatever backend the default group uses on CPU tensors)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    out = torch.empty(world * local.numel(), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(out, local, group=group)
    return out


def analyze_sharded(records, n_comms: int = 1, d=None, dev_hint: int = 8, tree_threshold: int = 1 << 20,
                    ring_order=None, group=None, stream=None):
    """Analyze this rank's shard (a CUDA tensor of packed records) and merge all ranks'
    partials; every rank returns the merged ``CtSummary`` (cells stay in the context).

    All ranks must use the same ``d`` / ``dev_hint`` so the partial layouts agree."""
    import torch
    import torch.distributed as dist

    ctx = _lib.context()
    ptr, n, on_dev = _lib.records_pointer(records)
    cfg = _lib.make_config(d=d, tree_threshold=tree_threshold, ring_order=ring_order, dev_hint=dev_hint,
                           n_comms=n_comms)
    s = _lib.CtSummary()
    # Everything runs on ONE stream -- torch's current one unless the caller names
    # another: the async export, the NCCL all-gather (enqueued by torch on its current
    # stream) and the merge are then ordered without extra events.
    if stream is None:
        stream = torch.cuda.current_stream().cuda_stream
    elif stream != torch.cuda.current_stream().cuda_stream:
        torch.cuda.current_stream().synchronize()  # records written by torch work
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
        ev = torch.cuda.ExternalStream(stream)
        cur.wait_stream(ev)
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
