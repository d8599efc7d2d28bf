"""``analyze`` command: trace files -> matrix / stats / diagnostics files.

Drop-in for the reference CLI's ``analyze`` subcommand (``pkg/src/commtrace/cli.py``:
emitters :53-115, ``cmd_analyze`` :123-187, options :368-380): same options, same
output file names and bytes, same stdout / stderr lines and exit codes (0 ok, 1 I/O
error, 2 invalid trace; an ``OverflowError`` escapes as in the reference).  The
difference is underneath: each file goes through the device JSONL loader
(``load_trace``) and the records never leave HBM before ``analyze_packed``.

Not provided: ``--heatmap`` SVG rendering (``heatmap.py:71-111``, formatting only —
rejected with exit 2), and the ``gen`` / ``verify`` / ``render`` subcommands.

    python -m paper_2110_10401_b200.cli analyze trace.jsonl -o out --split-per-primitive
"""

from __future__ import annotations

import argparse
import csv
import hashlib
import io
import json
import os
import sys
from pathlib import Path

from .decompose import DEFAULT_TREE_THRESHOLD
from .errors import TraceError
from .matrix import ALL_TYPES, CommMatrix, ModelConfig, analyze_packed

OUT_DIR_ENV = "COMSCRIBE_OUT"
EXIT_OK, EXIT_IO, EXIT_INVALID = 0, 1, 2


def _csv(rows) -> str:
    buf = io.StringIO()
    csv.writer(buf, lineterminator="\n").writerows(rows)
    return buf.getvalue()


def _json(obj) -> str:
    return json.dumps(obj, sort_keys=True, indent=2) + "\n"


def matrix_to_csv(m: CommMatrix) -> str:
    """Header row of endpoint labels, then one labelled row per source (cli.py:53-60)."""
    labels = m.labels()
    return _csv([[""] + labels] + [[lab] + row for lab, row in zip(labels, m.rows())])


def matrix_to_json(m: CommMatrix, meta: dict | None = None) -> str:
    """cli.py:71-80: d, aggregator flag, labels, cells (+ run metadata)."""
    return _json({"d": m.d, "aggregator": m.with_aggregator, "labels": m.labels(), "cells": m.rows(),
                  **(meta or {})})


def stats_to_json(result, meta: dict) -> str:
    """cli.py:88-102."""
    types = {key: {"calls": st.call_count, "payload_bytes": st.payload_bytes, "wire_bytes": st.wire_bytes}
             for key, st in result.stats.types.items()}
    return _json({"types": types, "instances": result.stats.instances,
                  "diagnostics": result.stats.diagnostics, **meta})


def stats_to_csv(result) -> str:
    """cli.py:105-114: one row per type in ALL_TYPES order."""
    rows = [["type", "calls", "payload_bytes", "wire_bytes"]]
    for key in ALL_TYPES:
        st = result.stats.types[key]
        rows.append([key, st.call_count, st.payload_bytes, st.wire_bytes])
    return _csv(rows)


def _concat(traces):
    """PackedTraces of several files -> one, comm ids in first-seen order over the
    concatenated events (what parse_trace(file1) + parse_trace(file2) gives)."""
    import numpy as np
    import torch

    from .packed import PackedTrace

    if len(traces) == 1:
        return traces[0]
    names, ids, parts, ts = [], {}, [], []
    for tr in traces:
        remap = []
        for name in tr.comms:
            if name not in ids:
                ids[name] = len(names)
                names.append(name)
            remap.append(ids[name])
        recs = tr.records.clone()
        if len(tr) and remap != list(range(len(remap))):
            comm = recs.view(torch.int32)[:, 4]
            comm.copy_(torch.tensor(remap, dtype=torch.int32, device=recs.device)[comm.long()])
        parts.append(recs)
        ts.append(tr.ts)
    recs = torch.cat(parts) if parts else traces[0].records
    if all(isinstance(t, np.ndarray) for t in ts):
        ts_all = np.concatenate(ts)
    else:
        ts_all = [int(x) for t in ts for x in t]
    return PackedTrace(recs, names, ts_all, None)


def _ring(text):
    return tuple(int(x) for x in text.split(",")) if text else None


def cmd_analyze(args) -> int:
    from .loader import load_trace

    if args.heatmap:
        print("error: --heatmap (SVG rendering) is not provided by this package", file=sys.stderr)
        return EXIT_INVALID
    out_dir = Path(args.out or os.environ.get(OUT_DIR_ENV) or ".")
    config = ModelConfig(ring_order=_ring(args.ring_perm), tree_threshold=args.tree_threshold)
    digest = hashlib.sha256()
    try:
        traces = []
        for path in args.trace:
            raw = Path(path).read_bytes()
            digest.update(raw)
            traces.append(load_trace(raw))
        trace = _concat(traces)
        result = analyze_packed(trace, d=args.gpus, config=config)
    except OSError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_IO
    except TraceError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_INVALID

    meta = {"trace_digest": f"sha256:{digest.hexdigest()}", "symmetrized": args.symmetrize}
    matrices = {"combined": result.combined}
    if args.split_per_primitive:
        matrices.update(result.per_primitive)
    if args.symmetrize:
        matrices = {k: m.symmetrized() for k, m in matrices.items()}
    diags = result.diagnostics
    try:
        out_dir.mkdir(parents=True, exist_ok=True)
        for name, m in matrices.items():
            if args.format in ("csv", "both"):
                (out_dir / f"matrix_{name}.csv").write_text(matrix_to_csv(m))
            if args.format in ("json", "both"):
                (out_dir / f"matrix_{name}.json").write_text(matrix_to_json(m, meta))
        (out_dir / "stats.json").write_text(stats_to_json(result, meta))
        if args.format in ("csv", "both"):
            (out_dir / "stats.csv").write_text(stats_to_csv(result))
        (out_dir / "diagnostics.json").write_text(
            _json([{"reason": g.reason, "comm": g.comm, "ordinal": g.ordinal, "detail": g.detail} for g in diags]))
    except OSError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_IO
    print(f"analyzed {len(trace)} events -> {result.stats.instances} instances, "
          f"{result.stats.diagnostics} diagnostics, d={result.d}")
    for g in diags:
        print(f"warning: {g}", file=sys.stderr)
    return EXIT_OK


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(
        prog="commtrace", description="Analyze inter-GPU communication traces into matrices and stats.")
    sub = parser.add_subparsers(dest="command", required=True)
    p = sub.add_parser("analyze", help="trace file(s) -> matrices, stats")
    p.add_argument("trace", nargs="+", help="JSONL trace file(s)")
    p.add_argument("-o", "--out", help=f"output directory (default ${OUT_DIR_ENV} or .)")
    p.add_argument("--gpus", type=int, default=None, help="device count (default: inferred)")
    p.add_argument("--split-per-primitive", action="store_true")
    p.add_argument("--symmetrize", action="store_true", help="emit undirected matrices (M + M^T)")
    p.add_argument("--ring-perm", help="comma-separated ring order, e.g. 0,2,1,3")
    p.add_argument("--tree-threshold", type=int, default=DEFAULT_TREE_THRESHOLD,
                   help="auto algorithm: tree below this payload size")
    p.add_argument("--format", choices=("csv", "json", "both"), default="both")
    p.add_argument("--heatmap", action="store_true", help="not provided (exit 2)")
    p.add_argument("--scale", choices=("log", "linear"), default="log")
    p.set_defaults(func=cmd_analyze)
    return parser


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    return args.func(args)


if __name__ == "__main__":
    sys.exit(main())
