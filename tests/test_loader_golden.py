"""Loader parity against the REFERENCE reader on a frozen fuzz corpus.

``tests/golden/loader_fuzz.json.gz`` holds, for every text of ``tests/loader_fuzz.py``
(2,140 texts: multi-line fuzz, single-line mutations, device-resident cases, escapes
and non-ASCII in every consulted string), the events or the exception that the
reference's ``parse_trace`` (/root/reference/pkg/src/commtrace/events.py:352-384)
produced in this container, for str and bytes input.  The device loader
(``load_trace``) must reproduce them: the same events field by field (timestamps and
comm names included), or the same exception class and message.

Value domain: where the reference accepted a value outside the packed
record (seq / count / bytes >= 2**64, nranks / dev / copy GPU >= 2**16) this
implementation must raise ``RecordRangeError`` instead of truncating.
"""

import pytest

from tests.conftest import load_golden
from tests.loader_fuzz import corpus, event_row

U64, U16 = 1 << 64, 1 << 16


@pytest.fixture(scope="module")
def fuzz_golden():
    return load_golden("loader_fuzz.json.gz")


def out_of_domain(rows):
    for r in rows:
        seq, n, dev, count, src, dst, nbytes = r[0], r[4], r[6], r[11], r[14], r[15], r[16]
        if seq >= U64 or n >= U16 or dev >= U16:
            return True
        if count is not None and count >= U64:
            return True
        if nbytes is not None and nbytes >= U64:
            return True
        if any(ep is not None and ep[0] == "gpu" and ep[1] >= U16 for ep in (src, dst)):
            return True
    return False


def expect(row, form):
    return row.get("bytes", row["str"]) if form == "bytes" else row["str"]


def check(load, src, want):
    from paper_2110_10401_b200 import errors as E

    if "error" in want:
        cls, msg = want["error"]
        with pytest.raises(Exception) as got:
            load(src)
        assert type(got.value).__name__ == cls and str(got.value) == msg, (src, got.value)
        return None
    if out_of_domain(want["events"]):
        with pytest.raises(E.RecordRangeError):
            load(src)
        return None
    got = load(src)
    rows = [event_row(got.event(i)) for i in range(len(got))]
    assert rows == want["events"], src
    return got


def test_corpus_matches_fixture(fuzz_golden):
    """The generator still produces exactly the frozen texts."""
    texts = corpus()
    assert len(texts) == len(fuzz_golden)
    assert all(t == r["text"] and g == r["g"] for (g, t), r in zip(texts, fuzz_golden))


def test_host_mirror_matches_reference(fuzz_golden):
    """The host reader (events.parse_trace + pack_events) that the loader defers to."""
    from paper_2110_10401_b200.events import parse_trace
    from paper_2110_10401_b200.packed import pack_events

    def load(src):
        tr = pack_events(parse_trace(src))
        return tr

    for row in fuzz_golden:
        check(load, row["text"], expect(row, "str"))
        check(load, row["text"].encode("utf-8", "surrogatepass"), expect(row, "bytes"))


@pytest.mark.gpu
@pytest.mark.parametrize("group", ["multi", "single", "device", "escape"])
def test_device_loader_matches_reference(fuzz_golden, group, loader_pipeline):
    from paper_2110_10401_b200.loader import load_trace

    seen = {"ok": 0, "err": 0}
    for row in fuzz_golden:
        if row["g"] != group:
            continue
        got = check(load_trace, row["text"], expect(row, "str"))
        check(load_trace, row["text"].encode("utf-8", "surrogatepass"), expect(row, "bytes"))
        seen["ok" if got is not None else "err"] += 1
    assert seen["ok"] and seen["err"], seen


@pytest.mark.gpu
def test_device_resident_text_matches_reference(fuzz_golden, loader_pipeline):
    """Text already in HBM (on_device=1), aligned and at odd offsets (unstaged path)."""
    import torch

    from paper_2110_10401_b200.loader import load_trace

    for row in fuzz_golden:
        if row["g"] not in ("device", "escape"):
            continue
        data = row["text"].encode("utf-8", "surrogatepass")
        for off in (0, 1, 3):
            buf = torch.zeros(len(data) + off, dtype=torch.uint8, device="cuda")
            if data:
                buf[off:] = torch.frombuffer(bytearray(data), dtype=torch.uint8).cuda()
            check(load_trace, buf[off:], expect(row, "bytes"))


@pytest.mark.gpu
def test_escapes_and_non_ascii_parse_on_device(loader_pipeline):
    """Raw UTF-8 names and \\uXXXX / \\" escapes (the reference's own write_trace escapes
    every non-ASCII name) are decoded on the device: nothing is left to the host reader,
    and one name written both ways is one communicator."""
    import json

    from paper_2110_10401_b200.events import parse_trace
    from paper_2110_10401_b200.loader import load_trace
    from paper_2110_10401_b200.packed import pack_events

    names = ["café", "日本", "\U0001f600", 'q"uote', "back\\slash", "tab\tname", "\ud83d"]
    lines = []
    for k in range(400):
        nm = names[k % len(names)]
        o = {"seq": k // 2, "ts": k, "kind": "collective", "comm": nm, "nranks": 2, "rank": k % 2, "dev": k % 2,
             "coll": "allreduce", "algo": "ring", "count": 100 + k // 2, "dtype": "float32"}
        ascii_form = k % 3 != 0 or "\ud83d" in nm  # write_trace style (\\u escapes) or raw UTF-8
        lines.append(json.dumps(o, separators=(",", ":"), ensure_ascii=ascii_form))
    lines.append(json.dumps({"seq": 0, "ts": 0, "kind": "coll\\u0065ctive"}))  # escaped enum: rejected exactly
    text = "\n".join(lines[:-1]) + "\n"
    data = text.encode("utf-8", "surrogatepass")
    got = load_trace(data)
    ref = pack_events(parse_trace(data.decode("utf-8", "surrogatepass")))
    assert got.load_info["deferred"] == 0
    assert got.records.cpu().numpy().tobytes() == ref.records.tobytes()
    assert got.comms == ref.comms and len(got.comms) == len(names)
