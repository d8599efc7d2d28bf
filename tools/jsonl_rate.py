"""GPU box: device JSONL loader throughput vs the host reader on a generated C3 text.

Usage: python tools/jsonl_rate.py [records_per_block] [repeats]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2110_10401_b200.events import parse_trace  # noqa: E402
from paper_2110_10401_b200.loader import load_trace  # noqa: E402
from paper_2110_10401_b200.packed import pack_events  # noqa: E402
from tests.test_gpu_loader import _generated_text  # noqa: E402

blk = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
rep = int(sys.argv[2]) if len(sys.argv) > 2 else 200
block = _generated_text(3, blk, seed=7)
if len(sys.argv) > 3 and sys.argv[3] == "bigts":  # nanosecond wall-clock timestamps, as the shim writes
    import re
    base = 1_760_000_000_000_000_000
    block = re.sub(rb'"ts":(\d+)', lambda m: b'"ts":%d' % (base + 1000 * int(m.group(1))), block)
t0 = time.perf_counter()
ref = pack_events(parse_trace(block))
t_host = time.perf_counter() - t0
text = block * rep
n = blk * rep
load_trace(block)  # warm-up (context, allocator)
for _ in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    tr = load_trace(text)
    torch.cuda.synchronize()
    t_e2e = time.perf_counter() - t0
ms = tr.load_info["ms_device"]
assert len(tr) == n and tr.load_info["deferred"] == 0
assert tr.records[:blk].cpu().numpy().tobytes() == ref.records.tobytes()
print(f"text {len(text) / 1e9:.3f} GB, {n / 1e6:.1f} M records ({len(text) / n:.0f} B/record)")
print("load_info", {k: v for k, v in tr.load_info.items()})
print(f"device parse {ms:.2f} ms -> {n / ms / 1e6:.2f} G rec/s, {len(text) / ms / 1e6:.1f} GB/s of JSONL")
print(f"load_trace end to end (host bytes -> HBM records) {t_e2e * 1e3:.1f} ms -> {n / t_e2e / 1e6:.1f} M rec/s")
print(f"host reader parse_trace+pack_events on {blk} records: {blk / t_host / 1e3:.1f} K rec/s (1 core)")
