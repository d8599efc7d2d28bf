"""Diagnostic: fraction of fast-kernel windows taking the steady (deferred) path per workload."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

os.environ["CT_DEBUG_MODE"] = "24"
from paper_2110_10401_b200 import _lib  # noqa: E402

ctx = _lib.context()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 20_000_000
for kind, name in ((4, "c4"), (2, "c2"), (3, "c3"), (5, "c5")):
    n = ctx.lib.ct_generate_boundary(kind, n)
    buf = torch.empty(n * 32, dtype=torch.uint8, device="cuda")
    rc = ctx.lib.ct_generate(ctx.handle, kind, C.c_uint64(7), C.c_uint64(0), C.c_uint64(n), C.c_void_p(buf.data_ptr()), None)
    ctx.check(rc, "gen")
    cfg = _lib.make_config(d=8, dev_hint=8, n_comms=8)
    s = _lib.CtSummary()
    rc = ctx.lib.ct_analyze(ctx.handle, C.c_void_p(buf.data_ptr()), n, 1, C.byref(cfg), C.byref(s), None)
    ctx.check(rc, "analyze")
    print(name, "path", s.path, "status", s.status, "steady windows", s.reserved, "~windows", n // 30,
          "frac", round(s.reserved / (n / 30), 3), "why", hex(s.err_aux[3]), "slowest warp", s.err_aux[2] & 0xFFFFFF, "cycles", s.err_aux[2] >> 24)
