"""Pin the CPU oracle to the real reference's outputs (golden fixtures).

The oracle is only trusted as a checker for the GPU path because these pass:
every fixture in tests/golden was produced by running the reference itself
(tests/golden/make_golden.py).
"""

import pytest

from oracle import commtrace_oracle as O
from paper_2110_10401_b200.events import parse_trace


def test_oracle_matches_reference_on_every_trace(golden_traces):
    assert len(golden_traces) > 200
    for case in golden_traces:
        events = parse_trace(case["jsonl"])
        got = O.analyze(events, d=case["d"], ring_order=case["ring_order"],
                        tree_threshold=case["tree_threshold"])
        want = {k: case[k] for k in ("error", "result") if k in case}
        assert got == want, case["name"]


def test_oracle_appendix_b_goldens(golden_traces):
    c1 = next(c for c in golden_traces if c["name"] == "C1")["result"]
    assert c1["combined"] == [[0, 0, 0, 0, 0], [0, 0, 104980480, 0, 0], [0, 0, 0, 104980480, 0],
                              [0, 0, 0, 0, 104980480], [0, 104755200, 0, 0, 0]]
    assert c1["combined_freq"] == [[0, 0, 0, 0, 0], [0, 0, 2490, 0, 0], [0, 0, 0, 2490, 0],
                                   [0, 0, 0, 0, 2490], [0, 2480, 0, 0, 0]]
    assert c1["stats"]["allreduce"] == [2480, 69836800, 419020800]
    assert c1["stats"]["broadcast"] == [10, 225280, 675840]


def test_oracle_matches_acceptance_grid(golden_grid):
    names = {"ar_ring": ("allreduce", "ring"), "ar_tree": ("allreduce", "tree"),
             "ar_collnet": ("allreduce", "collnet"), "allgather": ("allgather", "ring"),
             "reducescatter": ("reducescatter", "ring"), "broadcast": ("broadcast", "ring"),
             "reduce": ("reduce", "ring")}
    for key, want in golden_grid.items():
        name, n, s = key.split("/")
        n, s = int(n), int(s)
        coll, algo = names[name]
        root = s % n if coll in ("broadcast", "reduce") else None
        got = O.decompose(coll, algo, n, s, "int8", root, range(n))
        assert got == want, key


def test_oracle_matches_random_instances(golden_random_instances):
    for row in golden_random_instances:
        got = O.decompose(row["coll"], row["algo"], row["n"], row["count"], row["dtype"],
                          row["root"], range(row["n"]), ring_order=row["order"])
        assert got == row["transfers"]


@pytest.mark.parametrize("n,s,want", [
    (3, 10, {(0, 1): 14, (1, 2): 14, (2, 0): 12}),
    (5, 13, {(0, 1): 20, (1, 2): 20, (2, 3): 22, (3, 4): 22, (4, 0): 20}),
])
def test_oracle_nondivisible_ring(n, s, want):
    got = O.decompose("allreduce", "ring", n, s, "int8", None, range(n))
    assert {(a, b): v for a, b, v in got} == want
