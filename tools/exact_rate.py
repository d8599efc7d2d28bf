"""Throughput of the exact (sort-based) path, force_path=2, on generated traces (GPU box)."""
import ctypes as C
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2110_10401_b200 import _lib  # noqa: E402

ctx = _lib.context(0)
lib = ctx.lib
for kind, nc, n in ((4, 1, 100_000_000), (3, 3, 100_000_000), (2, 1, 100_000_000)):
    n = lib.ct_generate_boundary(kind, n)
    buf = torch.empty(n * 32, dtype=torch.uint8, device="cuda")
    assert lib.ct_generate(ctx.handle, kind, 7, 0, n, C.c_void_p(buf.data_ptr()), None) == 0
    for force in (1, 2):
        cfg = _lib.make_config(dev_hint=8, n_comms=nc, force_path=force)
        s = _lib.CtSummary()
        for it in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            rc = lib.ct_analyze(ctx.handle, C.c_void_p(buf.data_ptr()), n, 1, C.byref(cfg), C.byref(s), None)
            t1 = time.perf_counter()
        print(f"C{kind} n={n} force_path={force} rc={rc} path={s.path} ms_total={s.ms_total:.2f} "
              f"wall={1e3 * (t1 - t0):.2f} ms -> {n / (s.ms_total / 1e3) / 1e9:.2f} G rec/s")
    del buf
    torch.cuda.empty_cache()
