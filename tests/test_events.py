"""Host-side loader/writer mirror against the reference's own behaviour."""

import pytest

from paper_2110_10401_b200 import errors as E
from paper_2110_10401_b200.events import parse_trace, write_trace


def test_loader_cases_match_reference(golden_loader):
    for name, case in golden_loader.items():
        if "error" in case:
            cls = getattr(E, case["error"]["type"])
            with pytest.raises(cls) as exc:
                parse_trace(case["text"])
            assert str(exc.value) == case["error"]["message"], name
            if case["error"]["line_no"] is not None:
                assert exc.value.line_no == case["error"]["line_no"]
        else:
            evs = parse_trace(case["text"])
            assert len(evs) == case["n_events"], name
            assert write_trace(evs).decode() == case["roundtrip"], name


def test_roundtrip_every_golden_trace(golden_traces):
    for case in golden_traces:
        evs = parse_trace(case["jsonl"].encode())
        assert write_trace(evs).decode() == case["jsonl"], case["name"]
