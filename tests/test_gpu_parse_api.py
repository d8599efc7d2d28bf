"""The drop-in ``parse_trace`` / ``parse_trace_file`` (package top level): texts of 1 MB
or more go through the device loader and the native unpacker.  They must return exactly
the reference-mirroring host reader's events (``events.parse_trace``, pinned to the
reference by tests/test_loader_golden.py) and raise its exceptions."""

import json

import pytest

import paper_2110_10401_b200 as P
from paper_2110_10401_b200 import events as E
from paper_2110_10401_b200.loader import DEVICE_PARSE_MIN_BYTES
from tests.test_gpu_loader import _generated_text

pytestmark = pytest.mark.gpu


def _same(text):
    want = E.parse_trace(text)
    got = P.parse_trace(text)
    assert len(got) == len(want) and got == want
    assert all(type(g) is E.TraceEvent for g in got[:10])
    return got


def test_large_generated_texts_equal_host_reader(tmp_path):
    for kind in (2, 3, 5):
        text = _generated_text(kind, 20000, seed=kind)
        assert len(text) >= DEVICE_PARSE_MIN_BYTES
        _same(text)
        _same(text.decode())
    path = tmp_path / "t.jsonl"
    path.write_bytes(text)
    assert P.parse_trace_file(path) == E.parse_trace_file(path)


def test_large_text_errors_and_odd_lines():
    base = _generated_text(3, 20000, seed=9).decode().splitlines()
    # timestamps beyond int64, escaped and non-ASCII comm names, blank lines: same events
    odd = list(base)
    obj = json.loads(odd[10])
    obj["ts"] = 1 << 70
    odd[10] = json.dumps(obj)
    obj = json.loads(odd[20])
    obj["comm"] = "café"
    odd[20] = json.dumps(obj)
    odd.insert(30, "   ")
    _same("\n".join(odd) + "\n")
    # the first bad line raises the host reader's exception
    bad = list(base)
    bad[15000] = bad[15000].replace('"nranks":8', '"nranks":0')
    bad[17000] = "{not json"
    text = "\n".join(bad) + "\n"
    with pytest.raises(Exception) as want:
        E.parse_trace(text)
    with pytest.raises(Exception) as got:
        P.parse_trace(text)
    assert type(got.value) is type(want.value) and str(got.value) == str(want.value)


def test_small_texts_use_the_host_reader():
    text = _generated_text(3, 100, seed=1)
    assert len(text) < DEVICE_PARSE_MIN_BYTES
    _same(text)
