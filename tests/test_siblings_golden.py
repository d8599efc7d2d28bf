"""The analyze_events siblings against the reference.

``tests/golden/siblings.json.gz`` (made by ``tests/golden/make_golden.py`` with the
reference in this container) holds, per golden trace, the reference's
``split_by_primitive`` and ``summarize`` (matrix.py:261-301) on the grouped instance
list in three caller orders (as grouped, shuffled, reversed -- the per-type dict
order follows the list, matrix.py:271-276), ``infer_device_count``
(matrix.py:250-258), ``accumulate`` over every typed decomposition (matrix.py:157-161,
also into a too-small matrix) and ``merge`` of result matrices (matrix.py:164-178,
widening, d mismatch, overflow).
"""

import pytest

from tests.conftest import load_golden


@pytest.fixture(scope="module")
def sib():
    return load_golden("siblings.json.gz")


def _ep(e):
    from paper_2110_10401_b200.events import Endpoint, EndpointKind

    return Endpoint(EndpointKind(e[0]), e[1])


def _matrix(rows, agg):
    from paper_2110_10401_b200.matrix import CommMatrix

    d = len(rows) - 1 - (1 if agg else 0)
    return CommMatrix.from_rows(d, rows, agg)


def _call(fn):
    try:
        return fn()
    except Exception as exc:  # noqa: BLE001 - compared by class name and message
        return {"error": [type(exc).__name__, str(exc)]}


def _instances(rows):
    from paper_2110_10401_b200.events import Algorithm, CollectiveKind, DataType
    from paper_2110_10401_b200.grouping import CollectiveInstance

    return [CollectiveInstance(c, o, CollectiveKind(k), Algorithm(a), n, cnt, DataType(dt), root, tuple(devs))
            for c, o, k, a, n, cnt, dt, root, devs in rows]


def test_merge_matches_reference(sib):
    from paper_2110_10401_b200.matrix import merge

    n = 0
    for row in sib:
        for a, b, want in row["merges"]:
            got = _call(lambda: merge(_matrix(*a), _matrix(*b)))
            if isinstance(got, dict):
                assert got == want, row["name"]
            else:
                assert [got.rows(), got.with_aggregator] == want, row["name"]
            n += 1
    assert n > 500


def test_accumulate_matches_reference(sib):
    from paper_2110_10401_b200.decompose import Decomposition, PairTransfer
    from paper_2110_10401_b200.matrix import CommMatrix, accumulate

    for row in sib:
        if "decs" not in row:
            continue
        decs = [Decomposition(tuple(PairTransfer(_ep(s), _ep(t), b) for s, t, b in dec)) for dec in row["decs"]]
        for key, d in (("acc_infer", row["infer_d"]), ("acc_small", max(row["infer_d"] - 1, 0))):
            def run():
                m = CommMatrix(d)
                for dec in decs:
                    accumulate(m, dec)
                return m
            got = _call(run)
            want = row[key]
            assert (got if isinstance(got, dict) else [got.rows(), got.with_aggregator]) == want, row["name"]


@pytest.mark.gpu
def test_split_summarize_infer_match_reference(sib, golden_traces):
    from paper_2110_10401_b200.events import parse_trace
    from paper_2110_10401_b200.matrix import ModelConfig, infer_device_count, split_by_primitive, summarize
    from paper_2110_10401_b200.grouping import group_collectives

    cases = {c["name"]: c for c in golden_traces}
    checked = 0
    for row in sib:
        if "orders" not in row:
            continue
        case = cases[row["name"]]
        events = parse_trace(case["jsonl"])
        cfg = ModelConfig(ring_order=tuple(case["ring_order"]) if case["ring_order"] else None,
                          tree_threshold=case["tree_threshold"])
        assert infer_device_count(events) == row["infer_d"], row["name"]
        _, gdiags = group_collectives(events)
        for oname, rec in row["orders"].items():
            insts = _instances(rec["instances"])
            for dname, d in (("auto", None), ("given", case["d"])):
                if "split_" + dname not in rec:
                    continue
                got = _call(lambda: split_by_primitive(insts, events, d=d, config=cfg))
                if not isinstance(got, dict) or "error" not in got:
                    got = [[k, m.rows(), m.with_aggregator] for k, m in got.items()]
                assert got == rec["split_" + dname], (row["name"], oname, dname)
            sm = summarize(insts, events, config=cfg, diagnostics=gdiags)
            assert {"types": {t: [v.call_count, v.payload_bytes, v.wire_bytes] for t, v in sm.types.items()},
                    "instances": sm.instances, "diagnostics": sm.diagnostics} == rec["summary"], (row["name"], oname)
            assert summarize(insts, events, config=cfg).diagnostics == rec["summary_nodiag"]
            checked += 1
    assert checked > 300
