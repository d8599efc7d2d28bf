"""CPU ORACLE — test infrastructure only (tests/, smoke(), bench.py CPU legs).

ctypes wrapper of ``oracle/ct_oracle.c`` (the C restatement of the reference path).
``analyze_records`` returns the result in the kernels' internal cell layout plus a
reference-layout view; ``analyze_threads`` runs instance-aligned shards on host threads
(ctypes releases the GIL) and merges them exactly, the way SURVEY §8(d) prescribes for
the CPU baseline.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_build", "libct_oracle.so")
TYPES = ("allreduce", "broadcast", "reduce", "reducescatter", "allgather",
         "sendrecv", "explicit_transfer", "unified_memory", "zero_copy")
_lib = None


def load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            subprocess.run(["make", "-s", "-C", HERE], check=True)
        lib = C.CDLL(LIB)
        lib.cto_analyze.restype = C.c_int
        lib.cto_analyze.argtypes = [C.c_void_p, C.c_uint64, C.c_int64, C.c_uint64, C.c_void_p, C.c_int, C.c_int,
                                    C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                    C.POINTER(C.c_int64), C.POINTER(C.c_int)]
        _lib = lib
    return _lib


def analyze_records(records: np.ndarray, d=None, tree_threshold=1 << 20, ring_order=None, gcap=16):
    """Analyze a packed record array; returns a dict of numpy arrays / ints."""
    lib = load()
    recs = np.ascontiguousarray(records)
    g2 = gcap + 2
    ncell = 9 * g2 * g2
    cells = np.zeros(ncell, np.uint64)
    freq = np.zeros(ncell, np.uint64)
    calls = np.zeros(9, np.uint64)
    plo = np.zeros(9, np.uint64)
    phi = np.zeros(9, np.uint64)
    diag = np.zeros(6, np.uint64)
    ring = None if ring_order is None else np.array(ring_order, np.uint16)
    d_out, ovf = C.c_int64(), C.c_int()
    st = lib.cto_analyze(recs.ctypes.data, recs.shape[0], -1 if d is None else int(d), int(tree_threshold),
                         None if ring is None else ring.ctypes.data, 0 if ring is None else len(ring), gcap,
                         cells.ctypes.data, freq.ctypes.data, calls.ctypes.data, plo.ctypes.data,
                         phi.ctypes.data, diag.ctypes.data, C.byref(d_out), C.byref(ovf))
    return {"status": st, "d": d_out.value, "gcap": gcap, "cells": cells, "freq": freq, "calls": calls,
            "payload": [int(a) + (int(b) << 64) for a, b in zip(plo, phi)], "diag": diag,
            "overflow": bool(ovf.value)}


def merge(results):
    """Exact merge of shard results (matrix.py:164-178 semantics; counters summed)."""
    out = dict(results[0])
    out["cells"] = sum(r["cells"].astype(object) for r in results)
    out["freq"] = sum(r["freq"].astype(np.uint64) for r in results)
    out["calls"] = sum(r["calls"] for r in results)
    out["payload"] = [sum(r["payload"][t] for r in results) for t in range(9)]
    out["diag"] = sum(r["diag"] for r in results)
    out["d"] = max(r["d"] for r in results)
    out["status"] = next((r["status"] for r in results if r["status"]), 0)
    return out


def analyze_threads(records: np.ndarray, bounds, threads: int, **kw):
    """Analyze [bounds[i], bounds[i+1]) shards on ``threads`` host threads and merge."""
    shards = [records[a:b] for a, b in zip(bounds[:-1], bounds[1:])]
    with ThreadPoolExecutor(max_workers=threads) as ex:
        parts = list(ex.map(lambda r: analyze_records(r, **kw), shards))
    return merge(parts)


def reference_layout(cells: np.ndarray, t: int, g2: int, d: int, agg: bool):
    """Internal [src][dst] (host 0, net 1, gpu g + 2) -> reference rows (host, gpu0.., net)."""
    idx = [0] + [g + 2 for g in range(d)] + ([1] if agg else [])
    block = cells[t * g2 * g2:(t + 1) * g2 * g2].reshape(g2, g2)
    return [[int(block[i, j]) for j in idx] for i in idx]
