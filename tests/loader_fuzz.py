"""Fuzzed JSONL corpus for the loader parity tests.

The generator is seeded and deterministic: ``corpus()`` returns the exact texts the
GPU loader tests feed to ``load_trace``.  ``tests/golden/make_golden.py`` runs the
REFERENCE reader (``parse_trace``, /root/reference/pkg/src/commtrace/events.py:352-384)
on every one of them, in str and bytes form, and freezes the events or the exception
into ``tests/golden/loader_fuzz.json.gz`` so the device loader is judged against the
reference itself, not against this repo's host mirror.
"""

from __future__ import annotations

import json
import random

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
        o["comm"] = rng.choice(["cé", "c0", " ", "q\"", "a\\b", "c\tx", "x" * 40, "p"])
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


def corpus():
    """(group, text) pairs: 300 multi-line texts (12 seeds x 25 trials), 1200 single-line
    mutations placed first and last, 40 texts for the device-resident (unstaged) path,
    and texts with escapes / non-ASCII in every consulted position."""
    out = []
    for seed in range(12):
        rng = random.Random(seed)
        for trial in range(25):
            p_mut = [0.0, 0.02, 0.1, 0.5][trial % 4]
            out.append(("multi", fuzz_text(rng, rng.randrange(1, 60), p_mut, 0.1)))
    rng = random.Random(99)
    for _ in range(600):
        o = mutate(rng, rng.choice(BASE))
        line = render(rng, o)
        out.append(("single", line + "\n" + json.dumps(BASE[0]) + "\n"))
        out.append(("single", json.dumps(BASE[2]) + "\n" + line))
    rng = random.Random(7)
    for trial in range(40):
        out.append(("device", fuzz_text(rng, rng.randrange(1, 300), [0.0, 0.05, 0.3][trial % 3], 0.1)))
    rng = random.Random(31)
    for _ in range(300):
        out.append(("escape", escape_text(rng)))
    return out


_ESC_NAMES = ["c\\u00e9", "\\u0063\\u0030", "a\\\\b", "q\\\"x", "t\\tab", "n\\nl", "s\\/l", "\\ud83d\\ude00",
              "\\ud83d", "z\\u0000", "café", "日本", "\U0001f600", "\\u2028", "x\\by\\fz\\r"]
_ESC_ENUMS = {"kind": ["coll\\u0065ctive", "s\\u0065nd", "\\u0072ecv", "m\\u0065mcpy"],
              "coll": ["all\\u0072educe", "\\u0062roadcast"], "algo": ["\\u0072ing", "tr\\u0065e"],
              "dtype": ["float\\u00332", "int\\u0038", "bfloat16"], "ckind": ["d\\u0032d", "h2d"]}


def escape_text(rng):
    """Lines whose strings carry escapes or non-ASCII bytes in the comm name, the enum
    values and the keys (the device decodes them; invalid ones still raise)."""
    lines = []
    for _ in range(rng.randrange(1, 12)):
        o = dict(rng.choice(BASE))
        s = json.dumps(o, separators=(",", ":"), ensure_ascii=False)
        r = rng.random()
        if r < 0.45:
            s = s.replace('"comm":"%s"' % o["comm"], '"comm":"%s"' % rng.choice(_ESC_NAMES), 1)
        elif r < 0.75:
            key = rng.choice([k for k in _ESC_ENUMS if k in o] or ["kind"])
            if key in o:
                s = s.replace('"%s":"%s"' % (key, o[key]), '"%s":"%s"' % (key, rng.choice(_ESC_ENUMS[key])), 1)
        elif r < 0.9:
            k = rng.choice(list(o))
            esc = "".join("\\u%04x" % ord(ch) if rng.random() < 0.4 else ch for ch in k)
            s = s.replace('"%s":' % k, '"%s":' % esc, 1)
        else:
            s = s[:-1] + ',"note":"%s"}' % rng.choice(_ESC_NAMES)
        lines.append(s)
    return "\n".join(lines) + rng.choice(["\n", "", "\r\n"])


def event_row(ev):
    """A TraceEvent (reference or mirror) as a plain JSON-able row."""
    def val(x):
        if x is None:
            return None
        if hasattr(x, "kind") and hasattr(x, "index"):
            return [x.kind.value, x.index]
        return getattr(x, "value", x)

    return [val(getattr(ev, f)) for f in ("seq", "ts_ns", "kind", "comm", "n_ranks", "rank", "device",
                                          "collective", "algorithm", "root", "peer", "count", "dtype",
                                          "copy_kind", "copy_src", "copy_dst", "bytes")]
