"""Pin the C restatement of the reference path (oracle/ct_oracle.c) to the golden fixtures.

The C oracle is what the large-scale GPU parity tests and the CPU baseline use, so it is
checked here against every trace the real reference analysed (tests/golden)."""

import numpy as np

from oracle import c_oracle as CO
from paper_2110_10401_b200.events import parse_trace
from paper_2110_10401_b200.packed import pack_events

ERR = {1: "InvariantViolation", 2: "InvalidConfig", 3: "EndpointOutOfRange", 5: "WrongAlgorithm",
       6: "MissingRoot"}


def test_c_oracle_matches_reference_goldens(golden_traces):
    checked = 0
    for case in golden_traces:
        events = parse_trace(case["jsonl"])
        tr = pack_events(events)
        gcap = 16
        res = CO.analyze_records(tr.records, d=case["d"], tree_threshold=case["tree_threshold"],
                                 ring_order=case["ring_order"], gcap=gcap)
        if "error" in case:
            kind = case["error"]["type"]
            if kind == "OverflowError":
                assert res["overflow"], case["name"]
            else:
                assert ERR.get(res["status"]) == kind, case["name"]
            continue
        want = case["result"]
        assert res["status"] == 0 and not res["overflow"], case["name"]
        assert res["d"] == want["d"], case["name"]
        g2 = gcap + 2
        for key, rows, agg, freq in want["per_primitive"]:
            t = CO.TYPES.index(key)
            assert CO.reference_layout(res["cells"], t, g2, want["d"], agg) == rows, (case["name"], key)
            assert CO.reference_layout(res["freq"], t, g2, want["d"], agg) == freq, (case["name"], key)
        for t, key in enumerate(CO.TYPES):
            calls, payload, wire = want["stats"][key]
            assert int(res["calls"][t]) == calls and res["payload"][t] == payload, (case["name"], key)
        assert int(res["diag"].sum()) == want["n_diagnostics"], case["name"]
        checked += 1
    assert checked > 200


def test_c_oracle_threads_merge_equals_single(golden_traces):
    c1 = next(c for c in golden_traces if c["name"] == "C1")
    recs = pack_events(parse_trace(c1["jsonl"])).records
    one = CO.analyze_records(recs, gcap=8)
    # instance-aligned shards: blocks of 4 records
    bounds = [0, 4 * 600, 4 * 1300, len(recs)]
    many = CO.analyze_threads(recs, bounds, 3, gcap=8)
    assert np.array_equal(np.array(many["cells"], dtype=object), one["cells"].astype(object))
    assert many["calls"].tolist() == one["calls"].tolist()
