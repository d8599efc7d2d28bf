"""Per-rank step cost at the N=8 shard size on one GPU: ct_analyze on 125M C4 records,
ct_partial_export, and ct_partial_merge of 8 copies of the partial (the all-gather is
NCCL over NVLink, ~15 KB per rank, not included)."""
import ctypes as C
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2110_10401_b200 import _lib  # noqa: E402

ctx = _lib.context(0)
lib = ctx.lib
n = lib.ct_generate_boundary(4, 125_000_000)
buf = torch.empty(n * 32, dtype=torch.uint8, device="cuda")
assert lib.ct_generate(ctx.handle, 4, 2, 0, n, C.c_void_p(buf.data_ptr()), None) == 0
cfg = _lib.make_config(dev_hint=8, n_comms=1)
s, m = _lib.CtSummary(), _lib.CtSummary()
words = C.c_uint64()
st = torch.cuda.current_stream()
for it in range(6):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    assert lib.ct_analyze(ctx.handle, C.c_void_p(buf.data_ptr()), n, 1, C.byref(cfg), C.byref(s),
                          C.c_void_p(st.cuda_stream)) == 0
    t1 = time.perf_counter()
    lib.ct_partial_size(ctx.handle, C.byref(words))
    p = torch.empty(words.value * 8, dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    assert lib.ct_partial_export(ctx.handle, C.c_void_p(p.data_ptr()), words.value, C.c_void_p(st.cuda_stream)) == 0
    torch.cuda.synchronize()
    te = time.perf_counter()
    for k in range(1, 8):
        p[k * words.value:(k + 1) * words.value].copy_(p[:words.value])
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    # 8 copies of one shard fail the cross-shard seq-order check (status 22): timing only
    rc = lib.ct_partial_merge(ctx.handle, C.c_void_p(p.data_ptr()), 8, words.value, C.byref(m),
                              C.c_void_p(st.cuda_stream))
    t3 = time.perf_counter()
    print(f"analyze {1e3 * (t1 - t0):.3f} ms (kernel {s.ms_kernel:.3f}, total {s.ms_total:.3f})  "
          f"export {1e3 * (te - t1):.3f} ms  merge {1e3 * (t3 - t2):.3f} ms (rc {rc})")
