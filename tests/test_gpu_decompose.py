"""Emit kernel vs the reference's acceptance grid and 10K seeded instances."""

import pytest

pytestmark = pytest.mark.gpu


def _ep(ep):
    return -1 if ep.kind.value == "net" else ep.index


def test_acceptance_grid(golden_grid):
    from paper_2110_10401_b200 import Algorithm, CollectiveKind, DataType, decompose_many
    from paper_2110_10401_b200.grouping import CollectiveInstance

    names = {"ar_ring": (CollectiveKind.ALLREDUCE, Algorithm.RING),
             "ar_tree": (CollectiveKind.ALLREDUCE, Algorithm.TREE),
             "ar_collnet": (CollectiveKind.ALLREDUCE, Algorithm.COLLNET),
             "allgather": (CollectiveKind.ALLGATHER, Algorithm.RING),
             "reducescatter": (CollectiveKind.REDUCESCATTER, Algorithm.RING),
             "broadcast": (CollectiveKind.BROADCAST, Algorithm.RING),
             "reduce": (CollectiveKind.REDUCE, Algorithm.RING)}
    keys, insts = [], []
    for key in golden_grid:
        name, n, s = key.split("/")
        n, s = int(n), int(s)
        coll, algo = names[name]
        root = s % n if coll in (CollectiveKind.BROADCAST, CollectiveKind.REDUCE) else None
        insts.append(CollectiveInstance("c0", 0, coll, algo, n, s, DataType.INT8, root, tuple(range(n))))
        keys.append(key)
    decs = decompose_many(insts)  # one launch for ~29K instances
    for key, dec in zip(keys, decs):
        got = [[_ep(t.src), _ep(t.dst), t.bytes] for t in dec.transfers]
        assert got == golden_grid[key], key


def test_random_instances(golden_random_instances):
    from paper_2110_10401_b200 import Algorithm, CollectiveKind, DataType, decompose_instance
    from paper_2110_10401_b200.grouping import CollectiveInstance

    for row in golden_random_instances:
        inst = CollectiveInstance("c0", 0, CollectiveKind(row["coll"]), Algorithm(row["algo"]), row["n"],
                                  row["count"], DataType(row["dtype"]), row["root"], tuple(range(row["n"])))
        dec = decompose_instance(inst, ring_order=tuple(row["order"]))
        got = [[_ep(t.src), _ep(t.dst), t.bytes] for t in dec.transfers]
        assert got == row["transfers"]
        # conservation (test_acceptance.py:150-152)
        assert sum(dec.sent_by_rank.values()) == sum(dec.recv_by_rank.values())
