"""GPU box: where load_trace's end-to-end time goes (host bytes -> records in HBM).

Usage: python tools/load_e2e.py [reps]   (C3 text, 20000 records x reps, as in bench.py)
"""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2110_10401_b200 import _lib  # noqa: E402
from paper_2110_10401_b200.events import write_trace  # noqa: E402
from paper_2110_10401_b200.loader import load_trace  # noqa: E402
from paper_2110_10401_b200.packed import RECORD_BYTES, RECORD_DTYPE, PackedTrace, unpack  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 200
blk = 20000
ctx = _lib.context()
buf = torch.empty(blk * RECORD_BYTES, dtype=torch.uint8, device="cuda")
assert ctx.lib.ct_generate(ctx.handle, 3, 11, 0, blk, C.c_void_p(buf.data_ptr()), None) == 0
torch.cuda.synchronize()
rec = np.frombuffer(buf.cpu().numpy().tobytes(), dtype=RECORD_DTYPE).copy()
names = [f"comm{i}" for i in range(int(rec["comm"].max()) + 1)]
block = write_trace(unpack(PackedTrace(rec, names, list(range(blk)), None)))
text = block * reps
lib = _lib.load()
load_trace(block)
for it in range(3):
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    handle = C.c_void_p()
    info = _lib.CtJsonlInfo()
    rc = lib.ct_jsonl_parse(0, C.cast(C.c_char_p(text), C.c_void_p), len(text), 0, C.byref(handle), C.byref(info))
    assert rc == 0
    t.append(time.perf_counter())
    n = int(info.n_records)
    recs = torch.empty((n, RECORD_BYTES), dtype=torch.uint8, device="cuda")
    ts = np.empty(n, dtype=np.int64)
    t.append(time.perf_counter())
    assert lib.ct_jsonl_records(handle, C.c_void_p(recs.data_ptr()), ts.ctypes.data) == 0
    t.append(time.perf_counter())
    lib.ct_jsonl_free(handle)
    t.append(time.perf_counter())
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    tr = load_trace(text)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    d = np.diff(t) * 1e3
    print(f"it{it}: parse {d[0]:.1f} ms (device {info.ms_device:.2f}), alloc {d[1]:.1f}, records+ts {d[2]:.1f}, "
          f"free {d[3]:.1f}; load_trace {1e3 * (t1 - t0):.1f} ms for {len(text) / 1e6:.0f} MB, {n} records", flush=True)
