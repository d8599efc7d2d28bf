"""Device JSONL loader: reference wire text -> PackedTrace with records in HBM.

Drop-in for ``parse_trace`` followed by ``pack_events`` (reference
``pkg/src/commtrace/events.py:352-384``): the same records, comm ids
(first-seen order), timestamps and the same exceptions (class, message, first
offending line) as ``pack_events(parse_trace(text))``.

The sm_100a library splits lines (``str.splitlines`` terminators), parses, checks and
packs every line it can prove the reference accepts unchanged, and interns comm names
(``csrc/ct_jsonl.cu``), non-ASCII text and ``\\`` / ``\\uXXXX`` escapes included (names
decoded on the device).  The remaining "deferred" lines (raw control characters,
floats / bools / huge integers in consulted keys, escaped comm names longer than 256
bytes, and every malformed or invalid line) are read here with the reference-mirroring
line reader
(``events._parse_line``): for a well-formed trace that is normally none of them; for
a broken one it is where the reference's exception is raised.  Device-accepted lines
can never raise, so the first exception is the reference's.  There is no CPU path for
the bulk of the text: without the library this module raises NativeLibraryMissing.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .events import _parse_line
from .packed import RECORD_BYTES, PackedTrace, pack_events

_I64_MIN, _I64_MAX = -(1 << 63), (1 << 63) - 1


def _as_bytes(source) -> bytes:
    if isinstance(source, str):
        return source.encode("utf-8", "surrogatepass")
    data = source if isinstance(source, (bytes, bytearray, memoryview)) else source.read()
    return bytes(data) if not isinstance(data, str) else data.encode("utf-8", "surrogatepass")


def load_trace(source, device: int | None = None) -> PackedTrace:
    """JSONL (bytes / str / binary file / 1-D CUDA uint8 tensor) -> PackedTrace whose ``records`` is a CUDA
    uint8 tensor of shape (n, 32) on ``device``; ``ts`` is an int64 numpy array (a
    list when a timestamp does not fit int64); ``comms`` lists names by comm id."""
    import torch

    dev_text = None
    if isinstance(source, str):
        text_str = source
        data = source.encode("utf-8", "surrogatepass")
    elif isinstance(source, torch.Tensor):  # text already in device memory (uint8, 1-D)
        if not source.is_cuda or source.dtype != torch.uint8 or source.dim() != 1:
            raise TypeError("device text must be a 1-D CUDA uint8 tensor")
        text_str, data, dev_text = None, None, source.contiguous()
        if device is None:
            device = dev_text.device.index
    else:
        text_str = None
        data = _as_bytes(source)
    lib = _lib.load()
    if device is None:
        device = _lib.context().device
    handle = C.c_void_p()
    info = _lib.CtJsonlInfo()
    if dev_text is not None:
        torch.cuda.current_stream(dev_text.device).synchronize()  # the library uses its own stream
        rc = lib.ct_jsonl_parse(device, C.c_void_p(dev_text.data_ptr() if dev_text.numel() else 0),
                                dev_text.numel(), 1, C.byref(handle), C.byref(info))
    else:
        # the bytes object's own buffer (no copy); the library copies it to the device
        ptr = C.cast(C.c_char_p(data), C.c_void_p) if data else None
        rc = lib.ct_jsonl_parse(device, ptr, len(data), 0, C.byref(handle), C.byref(info))
    try:
        if rc != _lib.CT_OK:
            msg = lib.ct_jsonl_error(handle)
            raise RuntimeError(f"ct_jsonl_parse: status {rc}: {msg.decode() if msg else ''}")
        n = int(info.n_records)
        recs = torch.empty((n, RECORD_BYTES), dtype=torch.uint8, device=f"cuda:{device}")
        ts = np.empty(n, dtype=np.int64)
        _check(lib, handle, lib.ct_jsonl_records(handle, C.c_void_p(recs.data_ptr() if n else 0),
                                                 ts.ctypes.data if n else None), "ct_jsonl_records")
        nd, nc = int(info.n_deferred), int(info.n_comms)
        drows = np.zeros((max(nd, 1), 4), dtype=np.uint64)
        _check(lib, handle, lib.ct_jsonl_deferred(handle, drows.ctypes.data), "ct_jsonl_deferred")
        crows = np.zeros((max(nc, 1), 3), dtype=np.uint64)
        names = C.create_string_buffer(max(int(info.comm_bytes), 1))
        _check(lib, handle, lib.ct_jsonl_comms(handle, crows.ctypes.data, names), "ct_jsonl_comms")
        name_bytes = names.raw
    finally:
        lib.ct_jsonl_free(handle)

    if dev_text is not None and (nd or info.non_ascii):
        data = dev_text.cpu().numpy().tobytes()  # host copy only for deferred lines / UTF-8 check
    # the reference decodes the whole text before reading any line (UnicodeDecodeError first)
    if info.non_ascii and text_str is None:
        data.decode("utf-8")
    comm_first = {}
    for cid in range(nc):
        first, off, ln = (int(x) for x in crows[cid])
        # raw UTF-8 or decoded escapes (lone surrogates as in "surrogatepass")
        comm_first[name_bytes[off:off + ln].decode("utf-8", "surrogatepass")] = (first, cid)
    load_info = {"lines": int(info.n_lines), "deferred": nd, "device_comms": nc,
                 "ms_device": float(info.ms_device), "fused": bool(info.fused),
                 "slow": int(info.n_slow)}
    if nd == 0:
        names_out = [None] * nc
        for name, (_, cid) in comm_first.items():
            names_out[cid] = name
        out = PackedTrace(recs, names_out, ts, None)
    else:
        out = _finish_deferred(data, text_str, recs, ts, drows[:nd], comm_first)
    out.load_info = load_info
    return out


def _check(lib, handle, rc, what):
    if rc != _lib.CT_OK:
        msg = lib.ct_jsonl_error(handle)
        raise RuntimeError(f"{what}: status {rc}: {msg.decode() if msg else ''}")


def _finish_deferred(data, text_str, recs, ts, drows, comm_first) -> PackedTrace:
    """Read the deferred lines in line order (raising the reference's first error),
    pack them, merge their comm names into first-seen order and patch the records."""
    import torch

    events, slots, blank = [], [], []
    for line_no, slot, off, ln in (tuple(int(x) for x in r) for r in drows):
        raw = data[off:off + ln]
        line = raw.decode("utf-8", "surrogatepass") if text_str is not None else raw.decode("utf-8")
        ev = _parse_line(line, line_no)
        if ev is None:
            blank.append(slot)
        else:
            events.append(ev)
            slots.append(slot)
    # comm ids in first-seen record order over device and deferred lines
    first = {name: f for name, (f, _) in comm_first.items()}
    for ev, slot in zip(events, slots):
        if ev.comm not in first or slot < first[ev.comm]:
            first[ev.comm] = slot
    order = sorted(first, key=first.__getitem__)
    new_id = {name: i for i, name in enumerate(order)}
    part = pack_events(events, comms=new_id)  # packed-range errors, in record order
    dev = recs.device
    if comm_first:
        remap = torch.tensor([new_id[name] for name, _ in sorted(comm_first.items(), key=lambda kv: kv[1][1])],
                             dtype=torch.int32, device=dev)
        if not torch.equal(remap, torch.arange(len(comm_first), dtype=torch.int32, device=dev)):
            comm = recs.view(torch.int32)[:, 4]  # deferred / blank slots are rewritten below
            comm.copy_(remap[comm.long()])
    if slots:
        idx = torch.tensor(slots, dtype=torch.long, device=dev)
        rows = torch.from_numpy(part.records.view(np.uint8).reshape(-1, RECORD_BYTES)).to(dev)
        recs[idx] = rows
        big = [t for t in part.ts if not _I64_MIN <= t <= _I64_MAX]
        if big:
            ts = [int(t) for t in ts]
            for slot, t in zip(slots, part.ts):
                ts[slot] = t
        else:
            ts[np.array(slots, dtype=np.int64)] = np.array(part.ts, dtype=np.int64)
    if blank:
        keep = torch.ones(recs.shape[0], dtype=torch.bool, device=dev)
        keep[torch.tensor(blank, dtype=torch.long, device=dev)] = False
        recs = recs[keep].contiguous()
        keep_h = np.ones(len(ts), dtype=bool)
        keep_h[blank] = False
        ts = ts[keep_h] if isinstance(ts, np.ndarray) else [t for t, k in zip(ts, keep_h) if k]
    return PackedTrace(recs, order, ts, None)


def load_trace_file(path, device: int | None = None) -> PackedTrace:
    with open(path, "rb") as fh:
        return load_trace(fh.read(), device=device)


#: texts at least this large are read by the device loader in ``parse_trace``
DEVICE_PARSE_MIN_BYTES = 1 << 20


def _device_ready() -> bool:
    try:
        import torch

        if not torch.cuda.is_available():
            return False
        _lib.load()
        return True
    except Exception:
        return False


def parse_trace(source) -> list:
    """``parse_trace`` of the drop-in API (reference events.py:352-384): the same
    TraceEvent list and the same exceptions.  A text of 1 MB or more goes through the
    device loader (``load_trace``) and the native unpacker; a smaller one through the
    reference-mirroring host reader (``events.parse_trace``), whose per-call cost is lower
    than a device round trip."""
    from .events import parse_trace as host_parse
    from .packed import unpack

    data = source if isinstance(source, (str, bytes, bytearray, memoryview)) else source.read()
    if len(data) >= DEVICE_PARSE_MIN_BYTES and _device_ready():
        return unpack(load_trace(data))
    return host_parse(data)


def parse_trace_file(path) -> list:
    with open(path, "rb") as fh:
        return parse_trace(fh.read())


__all__ = ["load_trace", "load_trace_file", "parse_trace", "parse_trace_file"]
