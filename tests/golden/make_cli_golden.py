"""Freeze the reference CLI's ``analyze`` output files as fixtures.

    python tests/golden/make_cli_golden.py

Runs the REAL reference (``/root/reference/pkg/src``, read-only, this container only)
``commtrace.cli.main(["analyze", ...])`` on golden traces with several flag sets
and records, per run: exit code, stdout, stderr and every file written (name ->
text).  ``tests/test_gpu_cli.py`` replays the same runs through
``paper_2110_10401_b200.cli`` and compares byte for byte.  Writes
``tests/golden/cli.json.gz``.
"""

from __future__ import annotations

import contextlib
import gzip
import io
import json
import os
import sys
import tempfile

sys.path.insert(0, "/root/reference/pkg/src")

from commtrace.cli import main as ref_main  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

TRACES = ["C1", "gnmt_d4_s42", "algos_n5", "algos_n5_ring", "algos_n5_thresh", "algos_n5_d7",
          "bad_ring", "empty", "dup_seq", "nranks", "overflow", "rand0_canonical", "rand1_rankmajor",
          "rand2_shuffled", "rand5_shuffled", "rand8_shuffled"]

FLAGS = [
    [],
    ["--split-per-primitive"],
    ["--split-per-primitive", "--symmetrize", "--format", "json"],
    ["--format", "csv", "--gpus", "8"],
    ["--split-per-primitive", "--ring-perm", "0,2,1,3,4", "--tree-threshold", "4096"],
]


def run(argv):
    out, err = io.StringIO(), io.StringIO()
    with contextlib.redirect_stdout(out), contextlib.redirect_stderr(err):
        try:
            code = ref_main(argv)
        except SystemExit as exc:  # argparse
            code = exc.code
        except Exception as exc:  # escapes the reference CLI (e.g. OverflowError)
            code = {"exception": type(exc).__name__, "message": str(exc)}
    return code, out.getvalue(), err.getvalue()


def main():
    with gzip.open(os.path.join(HERE, "traces.json.gz"), "rt", encoding="utf-8") as fh:
        cases = {c["name"]: c for c in json.load(fh)}
    runs = []
    for name in TRACES:
        text = cases[name]["jsonl"]
        for flags in FLAGS:
            with tempfile.TemporaryDirectory() as tmp:
                trace = os.path.join(tmp, "trace.jsonl")
                with open(trace, "w", encoding="utf-8") as fh:
                    fh.write(text)
                out_dir = os.path.join(tmp, "out")
                code, out, err = run(["analyze", trace, "-o", out_dir, *flags])
                files = {}
                if os.path.isdir(out_dir):
                    for f in sorted(os.listdir(out_dir)):
                        with open(os.path.join(out_dir, f), encoding="utf-8") as fh:
                            files[f] = fh.read()
            runs.append({"trace": name, "flags": flags, "code": code, "stdout": out, "stderr": err,
                         "files": files})
    # two files in one run (events concatenated across files, one digest over both)
    with tempfile.TemporaryDirectory() as tmp:
        paths = []
        for k, name in enumerate(["algos_n5", "gnmt_d4_s42"]):
            paths.append(os.path.join(tmp, f"t{k}.jsonl"))
            with open(paths[-1], "w", encoding="utf-8") as fh:
                fh.write(cases[name]["jsonl"])
        out_dir = os.path.join(tmp, "out")
        code, out, err = run(["analyze", *paths, "-o", out_dir, "--split-per-primitive"])
        files = {f: open(os.path.join(out_dir, f), encoding="utf-8").read() for f in sorted(os.listdir(out_dir))}
        runs.append({"trace": ["algos_n5", "gnmt_d4_s42"], "flags": ["--split-per-primitive"], "code": code,
                     "stdout": out, "stderr": err, "files": files})
    with gzip.open(os.path.join(HERE, "cli.json.gz"), "wt", encoding="utf-8") as fh:
        json.dump(runs, fh)
    print(len(runs), "runs,", sum(len(r["files"]) for r in runs), "files")


if __name__ == "__main__":
    main()
