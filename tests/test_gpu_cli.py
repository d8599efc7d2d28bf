"""``analyze`` command against the reference CLI's frozen outputs.

``tests/golden/make_cli_golden.py`` ran the reference ``commtrace analyze`` on golden
traces with several flag sets; every run is replayed here through
``paper_2110_10401_b200.cli`` (device loader + device analysis) and must reproduce
the exit code (or escaping exception), stdout, stderr and every output file byte for
byte — the reference's own determinism contract (test_acceptance.py:246-270).
"""

import contextlib
import gzip
import io
import json
import os

import pytest

from paper_2110_10401_b200.cli import main as cli_main
from tests.conftest import GOLDEN, load_golden

pytestmark = pytest.mark.gpu


def _run(argv):
    out, err = io.StringIO(), io.StringIO()
    with contextlib.redirect_stdout(out), contextlib.redirect_stderr(err):
        try:
            code = cli_main(argv)
        except SystemExit as exc:
            code = exc.code
        except Exception as exc:
            code = {"exception": type(exc).__name__, "message": str(exc)}
    return code, out.getvalue(), err.getvalue()


def test_analyze_matches_reference_cli(tmp_path):
    cases = {c["name"]: c for c in load_golden("traces.json.gz")}
    runs = load_golden("cli.json.gz")
    assert len(runs) >= 80
    for k, run in enumerate(runs):
        names = run["trace"] if isinstance(run["trace"], list) else [run["trace"]]
        paths = []
        for j, name in enumerate(names):
            p = tmp_path / f"r{k}_{j}.jsonl"
            with open(p, "w", encoding="utf-8") as fh:
                fh.write(cases[name]["jsonl"])
            paths.append(str(p))
        out_dir = tmp_path / f"out{k}"
        code, out, err = _run(["analyze", *paths, "-o", str(out_dir), *run["flags"]])
        where = (run["trace"], run["flags"])
        assert code == run["code"], where
        assert out == run["stdout"], where
        assert err == run["stderr"], where
        files = {}
        if out_dir.is_dir():
            for f in sorted(os.listdir(out_dir)):
                files[f] = (out_dir / f).read_text(encoding="utf-8")
        assert sorted(files) == sorted(run["files"]), where
        for f, text in run["files"].items():
            assert files[f] == text, (where, f)
