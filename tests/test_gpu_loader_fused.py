"""The single-pass JSONL loader's own boundaries (ct_jsonl.cu ``k_fused``): 32 KB tiles
with a 4 KB look-behind, per-tile line cap, per-CTA name cache, global name table,
template parser vs slow list, decoupled look-back.  Every text is compared with the
reference-mirroring host reader (``pack_events(parse_trace(text))``, pinned to the
reference by ``test_loader_golden.py``): records, comm ids, timestamps, or the same
exception; ``load_info["fused"]`` says which pipeline took the text."""

import json
import random

import pytest

from tests.test_gpu_loader import check_same

pytestmark = pytest.mark.gpu

TILE = 32 * 1024
TERMS = ["\n", "\r\n", "\r", "\x0b", "\x0c", "\x1c", "\x1d", "\x1e", "\x85", "\u2028", "\u2029"]


def line(k, comm="c0", n=4, kind=None, **kw):
    kind = kind or ("collective", "send", "memcpy")[k % 3]
    o = {"seq": k, "ts": 1000 + k, "kind": kind, "comm": comm, "nranks": n, "rank": k % n, "dev": k % n}
    if kind == "collective":
        o.update(coll=("allreduce", "broadcast", "allgather")[k % 3], algo="ring", count=100 + k, dtype="float32")
        if o["coll"] == "broadcast":
            o["root"] = 0
    elif kind == "send":
        o.update(peer=(k + 1) % n, count=7 + k, dtype="int8")
    else:
        o.update(ckind="h2d", src={"kind": "host", "idx": 0}, dst={"kind": "gpu", "idx": k % n}, bytes=99 + k)
    o.update(kw)
    return json.dumps(o, separators=(",", ":"), ensure_ascii=False)


def fused_ok(text, fused=True):
    got = check_same(text)
    if got is not None:
        assert got.load_info["fused"] is fused, got.load_info
    return got


def test_many_tiles_canonical():
    text = "".join(line(k, comm=f"comm{k % 5}") + "\n" for k in range(6000))
    got = fused_ok(text.encode())
    assert got.load_info["deferred"] == 0 and len(got) == 6000


def test_terminators_straddling_tile_boundaries():
    """Each terminator kind placed to start 2, 1 and 0 bytes before a tile boundary."""
    parts, pos, k = [], 0, 0
    plan = [(t, d) for t in TERMS for d in (-2, -1, 0)]
    for b, (term, d) in enumerate(plan, start=1):
        target = b * TILE + d
        while True:
            ln = line(k)
            if pos + len(ln.encode()) + 400 >= target:
                break
            parts.append(ln + "\n")
            pos += len(ln.encode()) + 1
            k += 1
        base = line(k, comm="")  # pad the comm name: this line's terminator starts at target
        pad = target - pos - len(base.encode())
        assert pad >= 0
        ln = line(k, comm="p" * pad)
        parts.append(ln + term)
        pos += len(ln.encode()) + len(term.encode())
        k += 1
    parts.append(line(k))  # no final terminator
    text = "".join(parts)
    fused_ok(text)
    fused_ok(text.encode())


def test_text_ending_on_a_tile_boundary():
    for final in ("", "\n", "\r\n"):
        body, k = "", 0
        while len(body) < 2 * TILE - 300:
            body += line(k) + "\n"
            k += 1
        pad = 2 * TILE - len(body) - len(line(k, comm="")) - len(final)
        text = body + line(k, comm="x" * pad) + final
        assert len(text) == 2 * TILE
        fused_ok(text.encode())


def test_blank_lines_and_line_cap():
    text = "\n".join(line(k) if k % 4 else "  \t" for k in range(800)) + "\n\n\n"
    fused_ok(text.encode())
    # > 2048 line ends in one tile: the multi-pass pipeline takes the text
    text = line(0) + "\n" * 5000 + line(1) + "\n"
    fused_ok(text.encode(), fused=False)


def test_long_lines():
    # a line longer than the look-behind whose terminator lands in a later tile
    head = "".join(line(k) + "\n" for k in range(130))  # ~20 KB: the long line starts there
    text = head + line(1, pad="y" * 15000) + "\n" + line(2) + "\n"
    fused_ok(text.encode(), fused=False)
    # long lines inside one tile (< 4 KB): the slow list
    text = "".join(line(k, pad="z" * 3000) + "\n" for k in range(30))
    got = fused_ok(text.encode())
    assert got.load_info["deferred"] == 0


def test_comm_names_cache_and_table():
    names = ["a" * 31, "b" * 32, "c" * 33, "d" * 40, "café", "日本", "tab\tin", 'q"t', "b\\s"]
    text = "".join(line(k, comm=names[k % len(names)]) + "\n" for k in range(2000))
    fused_ok(text.encode())
    ascii_text = "".join(json.dumps(json.loads(ln), separators=(",", ":")) + "\n" for ln in text.splitlines())
    got = fused_ok(ascii_text.encode())  # \\uXXXX escapes: decoded on the slow list
    assert got.load_info["deferred"] == 0
    # 200 distinct names in one tile (cache overflow -> slow list), first seen out of order
    rnd = random.Random(3)
    order = list(range(200))
    rnd.shuffle(order)
    text = "".join(line(k, comm=f"n{order[k % 200]}") + "\n" for k in range(3000))
    fused_ok(text.encode())
    # more distinct names than the table holds: multi-pass
    text = "".join(line(k, comm=f"m{k}") + "\n" for k in range(5000))
    fused_ok(text.encode(), fused=False)


def test_slow_and_deferred_lines_across_tiles():
    rnd = random.Random(5)
    lines = []
    for k in range(4000):
        ln = line(k, comm=f"c{k % 7}")
        r = rnd.random()
        if r < 0.05:  # another key order: the slow list (device-parsed)
            ln = json.dumps(dict(reversed(list(json.loads(ln).items()))))
        elif r < 0.07:  # spaces after separators
            ln = json.dumps(json.loads(ln))
        elif r < 0.08 and '"count"' in ln:  # a float count: deferred to the host reader
            o = json.loads(ln)
            o["count"] = 1.0
            ln = json.dumps(o)
        lines.append(ln)
    fused_ok(("\n".join(lines) + "\n").encode())


def test_first_error_wins_across_tiles():
    lines = [line(k) for k in range(3000)]
    lines[2500] = lines[2500].replace('"nranks":4', '"nranks":0')  # later tile
    lines[700] = lines[700].replace('"rank":', '"rank":-')          # earlier tile
    check_same(("\n".join(lines) + "\n").encode())


def test_number_edges():
    cases = [dict(ts=-(1 << 63)), dict(ts=(1 << 63) - 1), dict(ts=-1), dict(ts=0), dict(seq=10 ** 19 - 1),
             dict(seq=(1 << 64) - 1), dict(seq=12345678), dict(seq=123456789), dict(seq=1234567890123456)]
    for kw in cases:
        check_same("".join(line(k, **kw) + "\n" for k in range(3)).encode())
    for bad in ('"seq":01', '"seq":1.5', '"seq":1e3', '"ts":-', '"ts":--1', '"ts":-01'):
        ln = line(0)
        ln = ln.replace('"seq":0', bad) if "seq" in bad else ln.replace('"ts":1000', bad)
        check_same((ln + "\n").encode())


def test_empty_and_blank_texts():
    for text in (b"", b"\n", b"  \n\t\n", b"\r\n\r\n"):
        check_same(text)


def test_random_bytes_multi_tile():
    """Garbage over several tiles (JSON punctuation, digits, terminators, invalid UTF-8,
    fragments of canonical lines): the same records or the same first exception as the
    reference-mirroring reader, through both pipelines."""
    rnd = random.Random(17)
    alphabet = b'{}[]":,0123456789-.eE abcdefghijklmnopqrstuvwxyz\t\n\r\x0b\x0c\x1c\\\xc2\x85\xe2\x80\xa8\xff'
    canon = [line(k).encode() for k in range(50)]
    for trial in range(12):
        parts = []
        while sum(map(len, parts)) < 70_000:
            r = rnd.random()
            if r < 0.6:
                parts.append(rnd.choice(canon) + b"\n")
            elif r < 0.8:  # a canonical line with a few bytes flipped
                b = bytearray(rnd.choice(canon))
                for _ in range(rnd.randint(1, 3)):
                    b[rnd.randrange(len(b))] = rnd.choice(alphabet)
                parts.append(bytes(b) + b"\n")
            else:
                parts.append(bytes(rnd.choice(alphabet) for _ in range(rnd.randint(1, 300))))
        text = b"".join(parts)
        if trial % 3 == 0:  # valid prefix, garbage only after the first tiles
            text = b"".join(c + b"\n" for c in canon * 20) + text
        check_same(text)
