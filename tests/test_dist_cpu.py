"""Multi-process host logic of the sharded path on CPU (gloo, world_size 2).

The device work (ct_analyze, partial export/merge) is covered on the GPU by
tests/test_gpu_scale.py::test_sharded_merge_equals_single; here the rank-ordered
all-gather of partials and the element-aligned shard cutting run on real processes."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2110_10401_b200.dist import gather_partials, shard_bounds


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # a partial is a fixed-size uint64 vector; rank r fills it with r-tagged words
        local = torch.arange(16, dtype=torch.int64) + 1000 * rank
        allp = gather_partials(local)
        out[rank] = allp.tolist()
    finally:
        dist.destroy_process_group()


def test_gather_partials_rank_order():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    want = list(range(16)) + [1000 + i for i in range(16)]
    assert out[0] == want and out[1] == want


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_shard_bounds_are_element_aligned(world):
    # C4-like layout: elements start on multiples of 8 (blocks of 8 ranks, 8 copies)
    boundary = lambda x: (x + 7) // 8 * 8  # noqa: E731
    n = 8 * 1000
    cuts = shard_bounds(n, world, boundary)
    assert cuts[0] == 0 and cuts[-1] == n and len(cuts) == world + 1
    assert all(a <= b for a, b in zip(cuts, cuts[1:]))
    assert all(c % 8 == 0 for c in cuts)
