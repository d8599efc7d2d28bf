#!/usr/bin/env python
"""Headline benchmark: trace records/s -> communication matrices on B200.

Workload (BASELINE.json configs[3]): a ResNet-50 data-parallel
training trace — ring allreduce over 25 MiB gradient buckets, init broadcasts,
per-iteration h2d copies, 8 ranks — synthesised on the device, 1B records total,
sharded by record range across N GPUs (strong scaling).  One step = the whole
analysis path over every record: layout check, group/match, expansion, byte +
frequency matrices and per-primitive statistics (ct_analyze), plus the NCCL
all-gather + merge of the per-GPU partials when N > 1.

    python bench.py [--gpus N --steps K --warmup W --impl b200|reference]

``value`` is device-timed with inputs resident in HBM; ``e2e`` repeats the step
through the public C ABI from pinned host buffers (H2D inside the timed region).
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {  # name -> (generator kind, n_comms, description)
    "c2": (2, 1, "C2 8-rank mixed collectives (5 kinds, 10 dtypes, count log-uniform [1,2^28))"),
    "c3": (3, 3, "C3 collectives + send/recv pairs + memcpy/um/zerocopy incl. host"),
    "c4": (4, 1, "C4 ResNet-50 DP training: 25 MiB bucketed ring allreduce, n=8"),
    "c5": (5, 7, "C5 ring vs tree allreduce sweep, n in 2..8, 1 KiB-1 GiB"),
    "c4i": (6, 1, "C4 in the capture layout of an LD_PRELOAD interposer (ranks interleaved, per-rank order kept)"),
}
RECORD_BYTES = 32
# one metric string for both arms (the driver divides b200 by reference only when they match)
METRIC = "trace records/sec -> comm matrix"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="c4", choices=sorted(WORKLOADS))
    ap.add_argument("--records", type=int, default=1_000_000_000)
    ap.add_argument("--seed", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-loader", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--no-object-api", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=64_000_000)
    ap.add_argument("--ref-sample", type=int, default=2_000_000)
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_traffic(workload, records):
    """dram bytes/launch of the fast kernel: dram__bytes_read.sum + dram__bytes_write.sum per
    record from the committed ``ncu --set full`` capture (profiles/ncu_traffic.json, taken
    at the capture's own record count), EXTRAPOLATED linearly to this launch; the source
    is reported next to it (``traffic_source``).  None when no capture exists."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as fh:
            e = json.load(fh).get(workload)
        if e is None:
            return None, None
        src = (f"extrapolated from profiles/ncu_traffic.json ({e.get('records_captured', '?')} records, "
               f"{e['bytes_per_record']:.3f} B/record)")
        return e["bytes_per_record"] * records, src
    except Exception:
        return None, None


class ClockSampler:
    """SM clocks / throttle reasons sampled during the timed region (NVML, else nvidia-smi)."""

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _nvml(self):
        """NVML reader (≈1 ms per sample) or None; same fields as the nvidia-smi query."""
        try:
            import pynvml as N
            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.index)
            reasons = getattr(N, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                N.nvmlDeviceGetCurrentClocksThrottleReasons
            bits = (0x8, 0x40, 0x20, 0x4)  # hw_slowdown, hw_thermal, sw_thermal, sw_power_cap

            def read():
                r = reasons(h)
                return [str(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)),
                        str(N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM))] + \
                    ["Active" if r & b else "Not Active" for b in bits]
            read()
            return read
        except Exception:
            return None

    def _run(self):
        read = self._nvml()
        if read is not None:
            while not self._stop.is_set():
                try:
                    self.samples.append(read())
                except Exception:
                    pass
                self._stop.wait(0.005)
            return
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.02)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for s in self.samples for k in range(4) if s[2 + k] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# --------------------------------------------------------------------------- CPU side

def _jsonl(evs) -> str:
    """The reference wire format (write_trace, events.py:262-291 key order) of host events."""
    lines = []
    for e in evs:
        o = {"seq": e.seq, "ts": e.ts_ns, "kind": e.kind.value, "comm": e.comm, "nranks": e.n_ranks,
             "rank": e.rank, "dev": e.device}
        if e.kind.value == "collective":
            o.update(coll=e.collective.value, algo=e.algorithm.value, count=e.count, dtype=e.dtype.value)
            if e.root is not None:
                o["root"] = e.root
        else:
            o.update(ckind=e.copy_kind.value, src={"kind": e.copy_src.kind.value, "idx": e.copy_src.index},
                     dst={"kind": e.copy_dst.kind.value, "idx": e.copy_dst.index}, bytes=e.bytes)
        lines.append(json.dumps(o, separators=(",", ":")))
    return "\n".join(lines) + "\n"


def _cpu_worker(args):
    from oracle import commtrace_oracle as O
    from oracle import workload_oracle as W

    lo, hi, parse = args
    evs = W.c4_events(hi, 8, lo)
    if parse:  # the reference's whole CPU path: parse_trace + analyze_events
        text = _jsonl(evs).encode()
        del evs
        t0 = time.perf_counter()
        res = O.analyze_flat(O.parse_jsonl(text))
    else:      # analyze_events on already-parsed events (the drop-in boundary, matrix.py:316)
        t0 = time.perf_counter()
        res = O.analyze(evs)
    return time.perf_counter() - t0, hi - lo, res["result"]["instances"]


def cpu_reference(sample: int, procs: int, parse: bool = False):
    """The reference algorithm (CPU oracle restatement, oracle/commtrace_oracle.py) on
    instance-aligned shards of the first ``sample`` C4 records, one process per core.
    Returns (records/s, busy seconds, records)."""
    import multiprocessing as mp

    step = (sample // procs) // 8 * 8
    shards = [(k * step, (k + 1) * step, parse) for k in range(procs)]
    # events (and their JSONL text) are built inside each worker, untimed; the path is timed
    with mp.get_context("fork").Pool(procs) as pool:
        out = pool.map(_cpu_worker, shards)
    busy = max(t for t, _, _ in out)
    n = sum(k for _, k, _ in out)
    return n / busy, busy, n


def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    procs = os.cpu_count() or 1
    sample = a.ref_sample
    for _ in range(max(a.warmup, 0) and 1):
        cpu_reference(min(sample, 80_000), procs)
    rates = []
    t_all = time.perf_counter()
    for _ in range(a.steps):
        r, _, n = cpu_reference(sample, procs)
        rates.append(r)
        if time.perf_counter() - t_all > 240:
            break
    v = statistics.median(rates)
    psample = max(procs * 8, min(sample, a.ref_sample // 4))
    prate, pbusy, pn = cpu_reference(psample, procs, parse=True)
    line = {
        "impl": "reference", "metric": METRIC, "value": v,
        "unit": "records/s", "n_gpus": a.gpus, "steps": len(rates), "warmup": a.warmup,
        "ms_per_step": 1e3 * sample / v, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": {"workload": WORKLOADS[a.workload][2], "records_sample": sample,
                   "timed": "analyze_events on parsed events (group + decompose + accumulate); "
                            "parse_trace excluded -- it is timed separately in parse_analyze"},
        "cpu_baseline": {"value": v, "unit": "records/s", "cores": procs, "kind": "port",
                         "sample": f"first {sample} C4 records (host-built, oracle/workload_oracle.py), "
                                   f"instance-aligned shards over {procs} processes; analysis timed"},
        "e2e": {"value": v, "unit": "records/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "parse_analyze": {"value": prate, "unit": "records/s", "records": pn, "busy_s": pbusy, "cores": procs,
                          "sample": f"first {psample} C4 records as JSONL (reference wire format); "
                                    "parse_trace + analyze_events restated (oracle parse_jsonl + analyze_flat)"},
    }
    print(json.dumps(line))


# --------------------------------------------------------------------------- GPU side

def main():
    a = parse()
    if a.impl == "reference":
        run_reference(a)
        return
    import torch
    import torch.distributed as dist

    from paper_2110_10401_b200 import _lib
    from paper_2110_10401_b200.dist import gather_partials

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    device = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(device)
    backend = os.environ.get("CT_DIST_BACKEND", "nccl")  # gloo: plumbing tests with ranks sharing a GPU
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", device))
        else:
            dist.init_process_group(backend)
    kind, n_comms, desc = WORKLOADS[a.workload]
    ctx = _lib.context(device)
    lib = ctx.lib
    total = lib.ct_generate_boundary(kind, a.records)
    # capture layouts (kind 6) shard by plain record ranges and route records to the rank
    # owning their canonical position (dist.route_any_layout); canonical ones cut at
    # element boundaries and need no exchange beyond the partials
    any_layout = kind == 6 and world > 1
    if any_layout:
        lo, hi = total * rank // world, total * (rank + 1) // world
    else:
        lo = lib.ct_generate_boundary(kind, total * rank // world)
        hi = lib.ct_generate_boundary(kind, total * (rank + 1) // world) if rank + 1 < world else total
    n = hi - lo
    buf = torch.empty(max(n, 1) * RECORD_BYTES, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()
    rc = lib.ct_generate(ctx.handle, kind, a.seed, lo, n, C.c_void_p(buf.data_ptr()), C.c_void_p(stream.cuda_stream))
    assert rc == 0, ctx.error()
    torch.cuda.synchronize()
    cfg = _lib.make_config(d=None, dev_hint=8, n_comms=n_comms, force_path=_lib.FORCE_FAST if any_layout else 0)
    summ = _lib.CtSummary()
    merged = _lib.CtSummary()

    pbuf = None

    dev_shard = None

    def step(ptr, on_device):
        """One pass of the path over this rank's shard (+ the partial exchange)."""
        nonlocal pbuf, dev_shard
        n_step = n
        if any_layout:  # global grouping: two small all-gathers + one all-to-all, then a canonical slice
            from paper_2110_10401_b200.dist import route_any_layout
            if on_device:
                src = buf
            else:  # host shard: H2D inside the step
                if dev_shard is None:
                    dev_shard = torch.empty(max(n, 1) * RECORD_BYTES, dtype=torch.uint8, device="cuda")
                dev_shard.copy_(host_shard, non_blocking=True)
                src = dev_shard
            part = route_any_layout(src[: n * RECORD_BYTES], n_comms, stream=stream.cuda_stream)
            ptr, on_device, n_step = part.data_ptr(), 1, part.shape[0]
        rc = lib.ct_analyze(ctx.handle, C.c_void_p(ptr), n_step, on_device, C.byref(cfg), C.byref(summ),
                            C.c_void_p(stream.cuda_stream))
        if rc != 0:
            raise RuntimeError(f"ct_analyze status {rc}: {ctx.error()}")
        ms_k = summ.ms_kernel
        launches = summ.n_launches
        if world > 1:
            words = C.c_uint64()
            lib.ct_partial_size(ctx.handle, C.byref(words))
            if pbuf is None:
                pbuf = torch.empty(words.value, dtype=torch.int64, device="cuda")
            rc = lib.ct_partial_export(ctx.handle, C.c_void_p(pbuf.data_ptr()), words.value,
                                       C.c_void_p(stream.cuda_stream))
            assert rc == 0, ctx.error()
            launches += 2
            if backend == "nccl":
                gbuf = gather_partials(pbuf)
            else:
                torch.cuda.synchronize()
                gbuf = gather_partials(pbuf.cpu()).cuda()
            rc = lib.ct_partial_merge(ctx.handle, C.c_void_p(gbuf.data_ptr()), world, words.value,
                                      C.byref(merged), C.c_void_p(stream.cuda_stream))
            if rc != 0:
                raise RuntimeError(f"ct_partial_merge status {rc}: {ctx.error()}")
            launches += merged.n_launches
        return ms_k, launches

    def timed(ptr, on_device, steps):
        for _ in range(a.warmup):
            step(ptr, on_device)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        kms, launches = [], 0
        with ClockSampler(device) as clk:
            e0.record(stream)
            for _ in range(steps):
                k, l = step(ptr, on_device)
                kms.append(k)
                launches += l
            e1.record(stream)
            torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ms = e0.elapsed_time(e1) / steps
        t = torch.tensor([ms], device="cuda" if backend == "nccl" else "cpu")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item()), statistics.mean(kms), launches, clk.summary()

    ms, kms, launches, clocks = timed(buf.data_ptr(), 1, a.steps)
    value = total / (ms / 1e3)
    peak, peak_kind = peaks()
    achieved = n * RECORD_BYTES / (kms / 1e3) / 1e9 if kms else None
    result = merged if world > 1 else summ
    check = {"instances": int(sum(result.calls[t] for t in range(5))), "diagnostics": int(sum(result.diag)),
             "d": int(result.d), "path": int(summ.path)}

    timed_cells = None
    if world == 1 and not a.no_parity:  # the timed step's own result, checked below
        import numpy as np
        g2 = summ.g_cap + 2
        timed_cells = (np.zeros(9 * g2 * g2, np.uint64), np.zeros(9 * g2 * g2, np.uint64))
        assert lib.ct_result_cells(ctx.handle, timed_cells[0].ctypes.data, timed_cells[1].ctypes.data,
                                   timed_cells[0].size) == 0, ctx.error()
        timed_summ = _lib.CtSummary.from_buffer_copy(summ)

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu:
        cpu = cpu_baseline_c(buf, min(n, a.cpu_sample), kind, lib)

    host = None
    if not a.no_e2e or timed_cells is not None:
        host = torch.empty(max(n, 1) * RECORD_BYTES, dtype=torch.uint8, pin_memory=True)
        host.copy_(buf)
    e2e = None
    host_shard = host
    if not a.no_e2e:
        if not any_layout:
            del buf
            torch.cuda.empty_cache()
        e_steps = max(1, min(a.steps, 5))
        ems, _, _, _ = timed(host.data_ptr(), 0, e_steps)
        d2h = (2 * 9 * 10 * 10 * 8 + 6 * n_comms * 8 + 512) * world
        e2e = {"value": total / (ems / 1e3), "unit": "records/s", "h2d_bytes_per_step": total * RECORD_BYTES,
               "d2h_bytes_per_step": d2h, "ms_per_step": ems, "steps": e_steps,
               "source": "pinned host buffers through ct_analyze (H2D inside the timed region)"}

    parity = None
    if timed_cells is not None:
        parity = parity_check(host, n, kind, lib, timed_summ, timed_cells)
    del host

    loader = None
    if rank == 0 and world == 1 and not a.no_loader:
        loader = loader_measure(ctx)
    object_api = None
    if rank == 0 and world == 1 and not a.no_object_api:
        object_api = object_api_measure(ctx)

    traffic, traffic_src = ncu_traffic(a.workload, n)
    if rank == 0:
        line = {
            "metric": METRIC,
            "value": value, "unit": "records/s", "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "int64", "data": "synthetic",
            "config": {"workload": desc, "records": total, "record_bytes": RECORD_BYTES,
                       "sharding": "record range, element-aligned", "l2": "inputs larger than L2 (32 GB at 1B records)",
                       "seed": a.seed},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak if achieved else None, "traffic": traffic,
                         "traffic_source": traffic_src,
                         "kernel": "ct::fast_kernel", "kernel_ms": kms, "peak_source": peak_kind,
                         "algorithmic_bytes_per_launch": n * RECORD_BYTES},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clocks,
            "result_check": check,
            "parity": parity,
            "loader": loader,
            "object_api": object_api,
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def loader_measure(ctx, blk=20_000, reps=200):
    """Device JSONL loader (``load_trace``) on a generated C3 text: ``blk``
    records written with the reference wire format (write_trace), repeated ``reps``
    times, passed as host bytes.  Reported beside the headline, not part of it."""
    try:
        import numpy as np
        import torch
        from paper_2110_10401_b200.events import parse_trace, write_trace
        from paper_2110_10401_b200.loader import load_trace
        from paper_2110_10401_b200.packed import PackedTrace, RECORD_DTYPE, pack_events, unpack

        buf = torch.empty(blk * RECORD_BYTES, dtype=torch.uint8, device="cuda")
        rc = ctx.lib.ct_generate(ctx.handle, 3, 11, 0, blk, C.c_void_p(buf.data_ptr()), None)
        assert rc == 0, ctx.error()
        torch.cuda.synchronize()
        rec = np.frombuffer(buf.cpu().numpy().tobytes(), dtype=RECORD_DTYPE).copy()
        names = [f"comm{i}" for i in range(int(rec["comm"].max()) + 1)]
        block = write_trace(unpack(PackedTrace(rec, names, list(range(blk)), None)))
        text = block * reps
        load_trace(text)  # warm-up at full size (device pool, pinned staging slots)
        dev_ms, e2e_s = [], []
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            tr = load_trace(text)
            torch.cuda.synchronize()
            e2e_s.append(time.perf_counter() - t0)
            dev_ms.append(tr.load_info["ms_device"])
        n = len(tr)
        assert n == blk * reps and tr.load_info["deferred"] == 0
        want = pack_events(parse_trace(block))  # host reader on one block (comm ids in first-seen order)
        assert tr.records[:blk].cpu().numpy().tobytes() == want.records.tobytes() and tr.comms == want.comms
        ms, dt = statistics.median(dev_ms), statistics.median(e2e_s)
        return {"records_per_s_device": n / (ms / 1e3), "jsonl_gb_per_s_device": len(text) / (ms / 1e3) / 1e9,
                "hbm_frac_device": len(text) / (ms / 1e3) / 1e9 / peaks()[0],
                "pipeline": "single-pass" if tr.load_info.get("fused") else "multi-pass",
                "ms_device": ms, "e2e_records_per_s": n / dt, "e2e_ms": dt * 1e3,
                "e2e_ms_runs": [round(x * 1e3, 1) for x in e2e_s], "lines": n, "bytes": len(text),
                "sample": f"C3 {blk} records x {reps} as JSONL, host bytes; median of 3",
                "api": "load_trace (JSONL -> records in HBM; device time = CUDA events around ct_jsonl_parse)"}
    except Exception as exc:  # reported, never fatal for the headline line
        return {"error": repr(exc)[:300]}


def parity_check(host, n, kind, lib, summ, cells):
    """The timed step's result (cells, frequencies, calls, 128-bit payloads, diagnostics,
    d) against oracle/ct_oracle.c over the WHOLE trace, outside the timed region (all
    host threads over element-aligned shards, merged exactly)."""
    import numpy as np
    from oracle import c_oracle as CO
    from paper_2110_10401_b200.packed import RECORD_DTYPE

    recs = host.numpy().view(RECORD_DTYPE)[:n]
    threads = os.cpu_count() or 1
    k = max(threads, 64)
    bounds = sorted({0, n} | {lib.ct_generate_boundary(kind, n * j // k) for j in range(1, k)})
    t0 = time.perf_counter()
    want = CO.analyze_threads(recs, bounds, threads, gcap=summ.g_cap)
    dt = time.perf_counter() - t0
    cb, cf = cells
    checks = {
        "status": want["status"] == 0,
        "d": int(summ.d) == int(want["d"]),
        "cells": bool(np.array_equal(cb.astype(object), np.asarray(want["cells"], dtype=object))),
        "freq": bool(np.array_equal(cf, want["freq"])),
        "calls": [int(x) for x in summ.calls] == [int(x) for x in want["calls"]],
        "payload": [int(summ.payload_lo[t]) + (int(summ.payload_hi[t]) << 64) for t in range(9)] == want["payload"],
        "diag": [int(x) for x in summ.diag] == [int(x) for x in want["diag"]],
    }
    return {"ok": all(checks.values()), "checks": checks, "records": n, "oracle": "oracle/ct_oracle.c",
            "oracle_s": round(dt, 2), "threads": threads}


def object_api_measure(ctx, n=1_000_000, ref_sample=100_000):
    """The drop-in object API end to end: ``analyze_events(list[TraceEvent])`` (native
    packer -> H2D -> ct_analyze -> result objects) on C1 (the reference's own training
    trace, tests/golden) and on a 1M-event C3 trace, next to the reference algorithm's
    CPU port (oracle/commtrace_oracle.analyze, one process) on the same event objects."""
    try:
        import numpy as np
        import torch
        from oracle import commtrace_oracle as O
        from paper_2110_10401_b200.events import parse_trace
        from paper_2110_10401_b200.matrix import analyze_events
        from paper_2110_10401_b200.packed import PackedTrace, RECORD_DTYPE, unpack
        from tests.golden_loader import load_case

        out = {}
        c1 = parse_trace(load_case("C1")["jsonl"])
        buf = torch.empty(n * RECORD_BYTES, dtype=torch.uint8, device="cuda")
        rc = ctx.lib.ct_generate(ctx.handle, 3, 13, 0, n, C.c_void_p(buf.data_ptr()), None)
        assert rc == 0, ctx.error()
        torch.cuda.synchronize()
        rec = np.frombuffer(buf.cpu().numpy().tobytes(), dtype=RECORD_DTYPE).copy()
        del buf
        names = [f"comm{i}" for i in range(int(rec["comm"].max()) + 1)]
        big = unpack(PackedTrace(rec, names, list(range(n)), None))  # TraceEvent objects (untimed)
        for name, evs in (("C1", c1), ("C3_1M", big)):
            analyze_events(evs[: min(len(evs), 10_000)])  # warm-up
            ts = []
            for _ in range(3):
                t0 = time.perf_counter()
                res = analyze_events(evs)
                ts.append(time.perf_counter() - t0)
            dt = statistics.median(ts)
            k = min(len(evs), ref_sample)
            t0 = time.perf_counter()
            want = O.analyze(evs[:k])
            rdt = time.perf_counter() - t0
            out[name] = {"events": len(evs), "records_per_s": len(evs) / dt, "ms": dt * 1e3,
                         "ref_port_records_per_s": k / rdt, "ref_port_sample": k, "ref_port_cores": 1,
                         "instances": res.stats.instances, "ref_instances_in_sample": want["result"]["instances"]}
        # the literal drop-in path on a JSONL text: parse_trace (device loader + native
        # unpack) then analyze_events, against the reference's own CPU path restated
        # (oracle parse_jsonl + analyze_flat, one process) on a sample of the same text
        import paper_2110_10401_b200 as P
        from paper_2110_10401_b200.events import write_trace

        text = write_trace(big)
        lines = text.splitlines(keepends=True)
        P.analyze_events(P.parse_trace(b"".join(lines[:20_000])))  # warm-up
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            res = P.analyze_events(P.parse_trace(text))
            ts.append(time.perf_counter() - t0)
        dt = statistics.median(ts)
        sample = b"".join(lines[:ref_sample])
        t0 = time.perf_counter()
        O.analyze_flat(O.parse_jsonl(sample))
        rdt = time.perf_counter() - t0
        out["parse_analyze_C3_1M"] = {"lines": n, "bytes": len(text), "lines_per_s": n / dt, "ms": dt * 1e3,
                                      "ref_port_lines_per_s": ref_sample / rdt, "ref_port_sample": ref_sample,
                                      "instances": res.stats.instances,
                                      "api": "parse_trace(jsonl) + analyze_events (drop-in top-level API)"}
        out["api"] = ("analyze_events(list[TraceEvent]) end to end (native packer, pinned-less H2D, device "
                      "analysis, result objects); ref_port = reference algorithm CPU port on the same events")
        return out
    except Exception as exc:  # reported, never fatal for the headline line
        return {"error": repr(exc)[:300]}


def cpu_baseline_c(buf, sample, kind, lib):
    """C restatement of the reference path (oracle/ct_oracle.c) on all host cores over
    element-aligned shards of the first ``sample`` records of the same trace."""
    from oracle import c_oracle as CO
    from paper_2110_10401_b200.packed import RECORD_DTYPE

    sample = lib.ct_generate_boundary(kind, sample)
    recs = buf[: sample * RECORD_BYTES].cpu().numpy().view(RECORD_DTYPE)
    threads = os.cpu_count() or 1
    bounds = sorted({0, sample} | {lib.ct_generate_boundary(kind, sample * k // threads) for k in range(1, threads)})
    CO.analyze_threads(recs[: min(sample, 1 << 20)], [0, min(sample, 1 << 20)], 1, gcap=8)  # warm-up
    t0 = time.perf_counter()
    CO.analyze_threads(recs, bounds, threads, gcap=8)
    dt = time.perf_counter() - t0
    return {"value": sample / dt, "unit": "records/s", "cores": threads, "kind": "port",
            "sample": f"first {sample} records of the same trace, oracle/ct_oracle.c (C restatement of the "
                      f"reference path) on {threads} host threads over element-aligned shards, {dt:.2f}s"}


if __name__ == "__main__":
    main()
