"""ctypes binding of ``libcommtrace_b200.so`` (C ABI in include/commtrace_b200.h).

There is deliberately no fallback: if the library is missing or no CUDA device is
usable, every analysis entry point raises ``NativeLibraryMissing`` /
``RuntimeError`` instead of computing on the host.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

from .errors import NativeLibraryMissing

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libcommtrace_b200.so")
NTYPES = 9
NDIAG = 6

CT_OK = 0
CT_ERR_INVARIANT = 1
CT_ERR_INVALID_CONFIG = 2
CT_ERR_ENDPOINT_RANGE = 3
CT_ERR_OVERFLOW = 4
CT_ERR_WRONG_ALGORITHM = 5
CT_ERR_MISSING_ROOT = 6
CT_ERR_ARGUMENT = 20
CT_ERR_CUDA = 21
CT_ERR_NOT_CANONICAL = 22
CT_ERR_CAPACITY = 23

FORCE_AUTO, FORCE_FAST, FORCE_EXACT, FORCE_COUNT = 0, 1, 2, 3


class CtConfig(C.Structure):
    _fields_ = [
        ("d", C.c_int64),
        ("tree_threshold", C.c_uint64),
        ("ring_len", C.c_int32),
        ("force_path", C.c_int32),
        ("ring_order", C.POINTER(C.c_uint16)),
        ("dev_hint", C.c_int32),
        ("n_comms", C.c_int32),
    ]


class CtSummary(C.Structure):
    _fields_ = [
        ("status", C.c_int32),
        ("path", C.c_int32),
        ("d", C.c_int64),
        ("g_cap", C.c_int32),
        ("net_used", C.c_int32),
        ("calls", C.c_uint64 * NTYPES),
        ("payload_lo", C.c_uint64 * NTYPES),
        ("payload_hi", C.c_uint64 * NTYPES),
        ("diag", C.c_uint64 * NDIAG),
        ("type_first", C.c_uint64 * NTYPES),
        ("n_records", C.c_uint64),
        ("err_index", C.c_uint64),
        ("err_aux", C.c_uint64 * 4),
        ("ms_total", C.c_float),
        ("ms_kernel", C.c_float),
        ("n_launches", C.c_uint32),
        ("reserved", C.c_uint32),
    ]


_lib = None
_lock = threading.Lock()
_contexts: dict[int, "Context"] = {}

_SIGNATURES = {
    "ct_context_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    "ct_context_destroy": (C.c_int, [C.c_void_p]),
    "ct_last_error": (C.c_char_p, [C.c_void_p]),
    "ct_analyze": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_int, C.POINTER(CtConfig),
                             C.POINTER(CtSummary), C.c_void_p]),
    "ct_result_cells": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64]),
    "ct_result_groups": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64,
                                   C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    "ct_result_p2p_diags": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.POINTER(C.c_uint64)]),
    "ct_materialize": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_int, C.c_int32,
                                 C.POINTER(CtSummary)]),
    "ct_infer_device_count": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_int,
                                        C.POINTER(C.c_int64)]),
    "ct_emit_transfers": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_int, C.POINTER(CtConfig),
                                    C.c_void_p, C.c_uint64, C.POINTER(C.c_uint64)]),
    "ct_generate": (C.c_int, [C.c_void_p, C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, C.c_void_p,
                              C.c_void_p]),
    "ct_generate_boundary": (C.c_uint64, [C.c_int, C.c_uint64]),
    "ct_c4_shape": (None, [C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.c_void_p]),
    "ct_partial_size": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint64)]),
    "ct_partial_export": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p]),
    "ct_partial_merge": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_uint64, C.POINTER(CtSummary),
                                   C.c_void_p]),
    "ct_shard_words": (C.c_int, [C.c_int32, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    "ct_shard_meta": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_int32, C.c_void_p, C.c_void_p]),
    "ct_shard_count": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_int32, C.c_void_p, C.c_int, C.c_void_p,
                                 C.c_void_p]),
    "ct_shard_route": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_void_p,
                                 C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                                 C.c_void_p]),
    "ct_shard_assemble": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p]),
    "ct_element_boundary": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_int, C.c_uint64,
                                      C.POINTER(C.c_uint64)]),
    "ct_jsonl_parse": (C.c_int, [C.c_int, C.c_void_p, C.c_uint64, C.c_int, C.POINTER(C.c_void_p),
                                 C.c_void_p]),
    "ct_jsonl_records": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "ct_jsonl_deferred": (C.c_int, [C.c_void_p, C.c_void_p]),
    "ct_jsonl_comms": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "ct_jsonl_error": (C.c_char_p, [C.c_void_p]),
    "ct_jsonl_free": (None, [C.c_void_p]),
}


class CtJsonlInfo(C.Structure):
    """ct_jsonl_info (include/commtrace_b200.h)."""

    _fields_ = [
        ("n_lines", C.c_uint64),
        ("n_records", C.c_uint64),
        ("n_deferred", C.c_uint64),
        ("n_comms", C.c_uint64),
        ("comm_bytes", C.c_uint64),
        ("non_ascii", C.c_uint32),
        ("ms_device", C.c_float),
        ("fused", C.c_uint32),
        ("n_slow", C.c_uint64),
    ]


def load():
    """Load the shared library (no CUDA calls)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise NativeLibraryMissing(
                f"{LIB_PATH} is not built; run `python -m paper_2110_10401_b200.build` "
                "(there is no CPU fallback for the analysis path)")
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


class Context:
    """One ct_context per CUDA device (owns its stream and scratch)."""

    def __init__(self, device: int = 0):
        lib = load()
        handle = C.c_void_p()
        rc = lib.ct_context_create(device, C.byref(handle))
        if rc != CT_OK:
            raise RuntimeError(f"ct_context_create(device={device}) failed with status {rc}: "
                               "no usable CUDA device (the analysis path has no CPU fallback)")
        self.lib = lib
        self.handle = handle
        self.device = device

    def error(self) -> str:
        msg = self.lib.ct_last_error(self.handle)
        return msg.decode() if msg else ""

    def check(self, rc: int, what: str):
        if rc in (CT_ERR_ARGUMENT, CT_ERR_CUDA, CT_ERR_NOT_CANONICAL, CT_ERR_CAPACITY):
            raise RuntimeError(f"{what}: status {rc}: {self.error()}")

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                self.lib.ct_context_destroy(self.handle)
        except Exception:
            pass


def context(device: int | None = None) -> Context:
    if device is None:
        if os.environ.get("CT_DEVICE") is not None:
            device = int(os.environ["CT_DEVICE"])
        else:  # torch's current device (set_device per rank), else LOCAL_RANK
            device = int(os.environ.get("LOCAL_RANK", "0"))
            try:
                import torch
                if torch.cuda.is_available():
                    device = torch.cuda.current_device()
            except Exception:  # noqa: BLE001 - torch is optional for the C-ABI user
                pass
    with _lock:
        ctx = _contexts.get(device)
    if ctx is None:
        ctx = Context(device)
        with _lock:
            _contexts[device] = ctx
    return ctx


def make_config(d=None, tree_threshold=1 << 20, ring_order=None, force_path=FORCE_AUTO,
                dev_hint=0, n_comms=1):
    cfg = CtConfig()
    cfg.d = -1 if d is None else int(d)
    cfg.tree_threshold = int(tree_threshold) if tree_threshold >= 0 else 0
    keep = None
    if ring_order is not None and len(ring_order) > 0:
        vals = [int(v) for v in ring_order]
        if any(v < 0 or v > 0xFFFF for v in vals):
            # out-of-range entries can never form a permutation; keep them invalid
            vals = [0xFFFF if (v < 0 or v > 0xFFFF) else v for v in vals]
        keep = np.array(vals, dtype=np.uint16)
        cfg.ring_len = len(vals)
        cfg.ring_order = keep.ctypes.data_as(C.POINTER(C.c_uint16))
    cfg.force_path = force_path
    cfg.dev_hint = int(dev_hint)
    cfg.n_comms = max(int(n_comms), 1)
    cfg._keep = keep  # keep the ring array alive with the struct
    return cfg


def records_pointer(records) -> tuple[int, int, int]:
    """(pointer, n, on_device) for a numpy record array or a CUDA torch tensor."""
    if isinstance(records, np.ndarray):
        arr = np.ascontiguousarray(records)
        return arr.ctypes.data, arr.shape[0], 0
    # torch tensor of uint8 / int64 holding packed records on a CUDA device
    if hasattr(records, "data_ptr") and getattr(records, "is_cuda", False):
        nbytes = records.numel() * records.element_size()
        return records.data_ptr(), nbytes // 32, 1
    raise TypeError("records must be a numpy RECORD_DTYPE array or a CUDA tensor of packed records")


def torch_stream(tensor):
    """torch's current stream on ``tensor``'s device as a ctypes handle: the library then
    runs after every torch kernel already queued there (the records' producers)."""
    import torch

    return C.c_void_p(torch.cuda.current_stream(tensor.device).cuda_stream)
