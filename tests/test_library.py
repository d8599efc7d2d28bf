"""CPU-side checks of the C ABI: the library loads and exports every declared symbol,
and the packed record layout matches ``ct_record`` byte for byte."""

import ctypes
import os
import re

import numpy as np

from paper_2110_10401_b200 import RECORD_DTYPE, _lib
from paper_2110_10401_b200.packed import pack_events
from paper_2110_10401_b200.events import parse_trace

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    text = open(os.path.join(ROOT, "include", "commtrace_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ct_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    names = declared_functions()
    assert len(names) >= 15
    for name in names:
        assert hasattr(lib, name), name


def test_record_layout_matches_header():
    # offsets from include/commtrace_b200.h ct_record
    want = {"count": 0, "seq": 8, "comm": 16, "nranks": 20, "rank": 22, "dev": 24, "aux": 26,
            "aux2": 28, "kc": 30, "ad": 31}
    for name, off in want.items():
        assert RECORD_DTYPE.fields[name][1] == off, name
    assert RECORD_DTYPE.itemsize == 32


def test_pack_roundtrip_golden(golden_traces):
    from paper_2110_10401_b200.packed import unpack
    for case in golden_traces[:60]:
        events = parse_trace(case["jsonl"])
        tr = pack_events(events)
        tr.events = None
        back = unpack(tr)
        assert [(e.seq, e.kind, e.comm, e.rank, e.device, e.count, e.bytes, e.root, e.peer) for e in back] == \
               [(e.seq, e.kind, e.comm, e.rank, e.device, e.count, e.bytes, e.root, e.peer) for e in events]
        assert tr.records.dtype == RECORD_DTYPE and isinstance(tr.records, np.ndarray)


def test_generator_boundaries_are_element_starts():
    lib = _lib.load()
    assert lib.ct_generate_boundary(2, 13) == 16
    assert lib.ct_generate_boundary(5, 36) == 70
    assert lib.ct_generate_boundary(3, 13) == 14
    n_t, n_b = ctypes.c_uint64(), ctypes.c_uint64()
    buckets = (ctypes.c_uint64 * 64)()
    lib.ct_c4_shape(ctypes.byref(n_t), ctypes.byref(n_b), buckets)
    assert n_t.value == 161                     # ResNet-50 parameter tensors
    assert sum(buckets[: n_b.value]) == 4 * 25557032
    assert all(b <= 25 << 20 for b in buckets[: n_b.value])
