"""The interposer on the real NCCL (torch-bundled) on a B200: torch.distributed NCCL
collectives in a preloaded child process -> trace -> device loader -> analysis."""

import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHIM = os.path.join(ROOT, "paper_2110_10401_b200", "libcomscribe_shim.so")

pytestmark = pytest.mark.gpu

CHILD = r"""
import os, torch, torch.distributed as dist
dist.init_process_group("nccl", init_method="tcp://127.0.0.1:%s" % os.environ["PORT"], rank=0, world_size=1,
                        device_id=torch.device("cuda:0"))
x = torch.ones(1024, device="cuda")
dist.all_reduce(x)                                           # float32, 1024
dist.broadcast(torch.ones(300, dtype=torch.bfloat16, device="cuda"), src=0)
dist.reduce(torch.ones(64, dtype=torch.float64, device="cuda"), dst=0)
dist.all_gather_into_tensor(torch.empty(32, device="cuda"), torch.ones(32, device="cuda"))
dist.reduce_scatter_tensor(torch.empty(16, device="cuda"), torch.ones(16, device="cuda"))
torch.cuda.synchronize()
dist.destroy_process_group()
print("child ok")
"""


def test_real_nccl_trace_loads_and_analyses(tmp_path):
    if not os.path.exists(SHIM):
        pytest.fail("shim not built")
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = tmp_path / "trace.jsonl"
    env = dict(os.environ, LD_PRELOAD=SHIM, COMSCRIBE_OUT=str(out), PORT=str(port))
    p = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True, timeout=300)
    assert p.returncode == 0 and "child ok" in p.stdout, p.stderr[-2000:]
    text = out.read_text()
    objs = [json.loads(l) for l in text.splitlines()]
    got = [(o["coll"], o["count"], o["dtype"]) for o in objs if o["kind"] == "collective"]
    # (with one rank torch does reduce_scatter_tensor as a local copy: no NCCL call)
    for want in [("allreduce", 1024, "float32"), ("broadcast", 300, "bfloat16"), ("reduce", 64, "float64"),
                 ("allgather", 32, "float32")]:
        assert want in got, (want, got)
    assert all(o["nranks"] == 1 and o["rank"] == 0 and o["dev"] == 0 for o in objs)
    main = [o for o in objs if o["comm"] == objs[0]["comm"]]
    assert [o["seq"] for o in main] == list(range(len(main)))

    from paper_2110_10401_b200 import analyze_packed, load_trace, pack_events
    from paper_2110_10401_b200.events import parse_trace
    tr = load_trace(text.encode())
    assert tr.load_info["deferred"] == 0
    ref = pack_events(parse_trace(text))
    assert tr.records.cpu().numpy().tobytes() == ref.records.tobytes()
    res = analyze_packed(tr)
    assert res.stats.instances == sum(1 for o in objs if o["kind"] == "collective")
