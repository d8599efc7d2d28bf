"""GPU parity: the sm_100a path against the reference's golden outputs.

Every fixture was produced by running the real reference (tests/golden/make_golden.py);
the CPU oracle is pinned to the same fixtures (test_oracle_golden.py).  Integer
results must be bit-exact.
"""

import pytest

from tests.helpers import run_case

pytestmark = pytest.mark.gpu


def _analyze(force):
    from paper_2110_10401_b200 import matrix
    from paper_2110_10401_b200.packed import pack_events

    def go(events, d, cfg):
        return matrix.analyze_packed(pack_events(events), d=d, config=cfg, force_path=force)
    return go


@pytest.mark.parametrize("force", [0, 2], ids=["auto", "exact"])
def test_golden_traces(golden_traces, force):
    bad = []
    for case in golden_traces:
        got, _ = run_case(case, _analyze(force))
        want = {k: case[k] for k in ("error", "result") if k in case}
        if got != want:
            bad.append(case["name"])
    assert not bad, bad


def test_golden_traces_counting_canonicaliser(golden_traces):
    """force_path=3: the counting canonicaliser (capture layout) on every golden trace it
    accepts -- rank-major files keep per-(comm, rank) order and must go through it; a
    trace outside its scope (file order != seq order) is refused, never misanalysed."""
    bad, taken = [], 0
    for case in golden_traces:
        try:
            got, _ = run_case(case, _analyze(3))
        except RuntimeError as exc:
            assert "status 22" in str(exc), exc
            continue
        taken += 1
        want = {k: case[k] for k in ("error", "result") if k in case}
        if got != want:
            bad.append(case["name"])
    assert not bad, bad
    assert taken > 100, taken


def test_fast_path_taken_on_canonical(golden_traces):
    from paper_2110_10401_b200 import matrix
    from paper_2110_10401_b200.events import parse_trace
    from paper_2110_10401_b200.packed import pack_events

    c1 = next(c for c in golden_traces if c["name"] == "C1")
    res = matrix.analyze_packed(pack_events(parse_trace(c1["jsonl"])), force_path=1)
    assert res.path == 1
    assert res.combined.rows()[1][2] == 104980480
