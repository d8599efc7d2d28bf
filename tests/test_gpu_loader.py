"""Device JSONL loader against the reference reader.

Expected values come from the reference-mirroring host reader
(``pack_events(parse_trace(text))``), itself pinned to the reference's own loader
behaviour by ``tests/golden/loader.json.gz`` (``test_events.py``): the same records,
comm ids, timestamps — or the same exception class and message.
"""

import ctypes as C
import json
import random

import numpy as np
import pytest

from paper_2110_10401_b200 import _lib
from paper_2110_10401_b200 import errors as E
from paper_2110_10401_b200.events import parse_trace
from paper_2110_10401_b200.loader import load_trace
from paper_2110_10401_b200.matrix import analyze_events, analyze_packed
from paper_2110_10401_b200.packed import PackedTrace, RECORD_DTYPE, pack_events, unpack
from paper_2110_10401_b200.events import write_trace

pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("loader_pipeline")]


def reference(text):
    try:
        return pack_events(parse_trace(text)), None
    except (E.TraceError, UnicodeDecodeError) as exc:
        return None, exc


def check_same(text):
    ref, err = reference(text)
    if err is not None:
        with pytest.raises(type(err)) as got:
            load_trace(text)
        assert str(got.value) == str(err)
        return None
    got = load_trace(text)
    assert len(got) == len(ref)
    assert got.records.cpu().numpy().tobytes() == ref.records.tobytes()
    assert got.comms == ref.comms
    assert [int(t) for t in got.ts] == [int(t) for t in ref.ts]
    return got


def test_golden_loader_cases(golden_loader):
    for name, case in golden_loader.items():
        for form in (case["text"], case["text"].encode("utf-8")):
            check_same(form)


def test_golden_traces(golden_traces):
    for case in golden_traces:
        got = check_same(case["jsonl"].encode())
        if got is not None and len(got):
            evs = parse_trace(case["jsonl"])
            assert all(got.event(i) == evs[i] for i in (0, len(evs) - 1))


def _generated_text(kind, n, seed=0):
    import torch

    ctx = _lib.context()
    buf = torch.empty(n * 32, dtype=torch.uint8, device="cuda")
    rc = ctx.lib.ct_generate(ctx.handle, kind, seed, 0, n, C.c_void_p(buf.data_ptr()), None)
    assert rc == 0
    torch.cuda.synchronize()
    rec = np.frombuffer(buf.cpu().numpy().tobytes(), dtype=RECORD_DTYPE)
    n_comms = int(rec["comm"].max()) + 1
    trace = PackedTrace(rec.copy(), [f"comm{i}" for i in range(n_comms)], list(range(n)), None)
    return write_trace(unpack(trace))


def test_generated_c3_trace_and_analysis():
    text = _generated_text(3, 20000, seed=5)
    got = check_same(text)
    assert got.load_info["deferred"] == 0 and got.load_info["lines"] == 20000
    evs = parse_trace(text)
    a = analyze_packed(got)
    b = analyze_events(evs)
    assert a.combined.rows() == b.combined.rows()
    assert a.combined_frequency.rows() == b.combined_frequency.rows()
    assert a.stats == b.stats


# ---------------------------------------------------------------- fuzzed lines

BASE = [
    {"seq": 0, "ts": 5, "kind": "collective", "comm": "c0", "nranks": 4, "rank": 1, "dev": 1,
     "coll": "allreduce", "algo": "ring", "count": 1024, "dtype": "float32"},
    {"seq": 1, "ts": 6, "kind": "collective", "comm": "c1", "nranks": 2, "rank": 0, "dev": 3,
     "coll": "broadcast", "algo": "ring", "count": 7, "dtype": "int8", "root": 1},
    {"seq": 2, "ts": 7, "kind": "send", "comm": "p", "nranks": 2, "rank": 0, "dev": 0,
     "peer": 1, "count": 10, "dtype": "bfloat16"},
    {"seq": 2, "ts": 8, "kind": "recv", "comm": "p", "nranks": 2, "rank": 1, "dev": 1,
     "peer": 0, "count": 10, "dtype": "bfloat16"},
    {"seq": 0, "ts": 9, "kind": "memcpy", "comm": "x", "nranks": 1, "rank": 0, "dev": 0,
     "ckind": "d2d", "src": {"kind": "gpu", "idx": 0}, "dst": {"kind": "gpu", "idx": 2}, "bytes": 99},
    {"seq": 0, "ts": -3, "kind": "zerocopy", "comm": "x", "nranks": 1, "rank": 0, "dev": 0,
     "ckind": "h2d", "src": {"kind": "host", "idx": 0}, "dst": {"kind": "gpu", "idx": 5}, "bytes": 0},
    {"seq": 0, "ts": 1, "kind": "um", "comm": "y", "nranks": 1, "rank": 0, "dev": 2,
     "ckind": "d2h", "src": {"kind": "gpu", "idx": 2}, "dst": {"kind": "host", "idx": 0}, "bytes": 4},
]

ODD_VALUES = [True, False, None, 1.0, 1e3, -1, -0, 2 ** 64, 2 ** 63, 2 ** 70, "x", "", [], {}, [1, [2]],
              {"a": {"b": [None]}}, 70000, 65535, 65536, 0]


def mutate(rng, obj):
    o = json.loads(json.dumps(obj))
    op = rng.randrange(14)
    keys = list(o)
    if op == 0:  # unknown key with a nested value
        o["extra%d" % rng.randrange(3)] = rng.choice(ODD_VALUES)
    elif op == 1:  # odd value for a consulted key
        o[rng.choice(keys)] = rng.choice(ODD_VALUES)
    elif op == 2:  # missing key
        del o[rng.choice(keys)]
    elif op == 3:  # key order
        items = list(o.items())
        rng.shuffle(items)
        o = dict(items)
    elif op == 4:  # endpoint variants
        if "src" in o:
            o[rng.choice(["src", "dst"])] = rng.choice([{"kind": "net", "idx": 0}, {"kind": "gpu", "idx": -1},
                                                        {"idx": 1}, {"kind": "gpu", "idx": 1, "z": [1]},
                                                        {"kind": "host", "idx": 2}, "gpu", {"kind": "gpu", "idx": 70000}])
        else:
            o["root"] = rng.choice([0, 1, 5, -1, None])
    elif op == 5:
        o["comm"] = rng.choice(["cé", "c0", " ", "q\"", "a\\b", "c\tx", "x" * 40, "p"])
    elif op == 6:
        o["nranks"] = rng.choice([0, 1, 2, 8, 65535, 65536])
    elif op == 7:
        o["algo"] = rng.choice(["tree", "collnet", "auto", "Ring"])
    elif op == 8:
        o["seq"] = rng.choice([2 ** 64 - 1, 2 ** 64, -5, 3])
    elif op == 9:
        o["ts"] = rng.choice([2 ** 63 - 1, 2 ** 63, -(2 ** 63), -(2 ** 63) - 1, 2 ** 80])
    elif op == 10:
        o["dev"] = rng.choice([65535, 65536, -1])
    elif op == 11:
        o["peer" if "peer" in o else "count"] = rng.choice([0, 1, 3, 2 ** 64 - 1])
    return o


def render(rng, o):
    style = rng.randrange(6)
    if style == 0:
        s = json.dumps(o, separators=(",", ":"))
    elif style == 1:
        s = json.dumps(o)
    elif style == 2:
        s = json.dumps(o, indent=None, separators=(" , ", " : "))
    elif style == 3:
        s = " \t" + json.dumps(o) + "\t "
    elif style == 4:
        s = json.dumps(o, ensure_ascii=False)
    else:
        s = json.dumps(o, separators=(",", ":")).replace('"c0"', '"\\u0063\\u0030"')
    r = rng.random()
    if r < 0.03:
        s = s[: rng.randrange(len(s))]  # truncated
    elif r < 0.05:
        s = s + rng.choice(["x", " {}", ",", "]"])
    elif r < 0.06:
        s = s.replace("1", "01", 1)
    elif r < 0.07:
        s = s.replace(":", ":NaN,\"k\":", 1)
    return s


BREAKS = ["\n", "\r\n", "\r", "\x0b", "\x0c", "\x1c", "\u2028", "\x85"]
BLANKS = ["", "   ", "\t", "\x1f", "\xa0", " \t "]


def fuzz_text(rng, n_lines, p_mut, p_break):
    lines = []
    for _ in range(n_lines):
        if rng.random() < 0.05:
            lines.append(rng.choice(BLANKS))
            continue
        o = rng.choice(BASE)
        if rng.random() < p_mut:
            o = mutate(rng, o)
        lines.append(render(rng, o) if rng.random() < p_mut else json.dumps(o, separators=(",", ":")))
    out = []
    for ln in lines:
        out.append(ln)
        out.append(rng.choice(BREAKS) if rng.random() < p_break else "\n")
    if rng.random() < 0.3:
        out.pop()
    return "".join(out)


@pytest.mark.parametrize("seed", range(12))
def test_fuzzed_texts(seed):
    rng = random.Random(seed)
    seen = {"ok": 0, "err": 0, "deferred": 0, "device": 0}
    for trial in range(25):
        # mostly-valid texts (exercise deferral + merging) and error-first texts
        p_mut = [0.0, 0.02, 0.1, 0.5][trial % 4]
        text = fuzz_text(rng, rng.randrange(1, 60), p_mut, 0.1)
        got = check_same(text)
        check_same(text.encode("utf-8", "surrogatepass"))
        if got is None:
            seen["err"] += 1
        else:
            seen["ok"] += 1
            seen["deferred"] += got.load_info["deferred"]
            seen["device"] += len(got) - got.load_info["deferred"]
    # both outcomes and both line paths are exercised
    assert seen["ok"] and seen["err"] and seen["deferred"] and seen["device"], seen


def test_single_line_mutations():
    rng = random.Random(99)
    for _ in range(600):
        o = mutate(rng, rng.choice(BASE))
        line = render(rng, o)
        check_same(line + "\n" + json.dumps(BASE[0]) + "\n")
        check_same(json.dumps(BASE[2]) + "\n" + line)


def test_invalid_utf8_raises_decode_error():
    bad = (json.dumps(BASE[0]) + "\n").encode() + b'{"comm": "\xff"}\n'
    with pytest.raises(UnicodeDecodeError):
        load_trace(bad)


def test_first_seen_comm_order_with_deferred_lines():
    # a deferred line (escaped name) introduces "c1" before the device-parsed ones
    lines = [json.dumps(dict(BASE[1], comm="\\u0063\\u0031")).replace("\\\\", "\\"),
             json.dumps(BASE[0]), json.dumps(BASE[1]), json.dumps(dict(BASE[0], comm="zé"))]
    check_same("\n".join(lines) + "\n")


def test_device_resident_text_aligned_and_unaligned():
    """on_device=1 through the C ABI; an odd offset takes the unstaged byte path."""
    import torch

    rng = random.Random(7)
    for trial in range(40):
        text = fuzz_text(rng, rng.randrange(1, 300), [0.0, 0.05, 0.3][trial % 3], 0.1)
        data = text.encode("utf-8", "surrogatepass")
        ref, err = reference(data)
        for off in (0, 1, 3):
            buf = torch.zeros(len(data) + off, dtype=torch.uint8, device="cuda")
            if data:
                buf[off:] = torch.frombuffer(bytearray(data), dtype=torch.uint8).cuda()
            src = buf[off:]
            if err is not None:
                with pytest.raises(type(err)) as got:
                    load_trace(src)
                assert str(got.value) == str(err)
                continue
            got = load_trace(src)
            assert got.records.cpu().numpy().tobytes() == ref.records.tobytes()
            assert got.comms == ref.comms
            assert [int(t) for t in got.ts] == [int(t) for t in ref.ts]
