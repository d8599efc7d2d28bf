"""CPU: the analyze emitters (cli.py:53-115 formats) on the reference's expected
matrices reproduce the reference CLI's files byte for byte (no GPU needed)."""

from paper_2110_10401_b200.cli import matrix_to_csv, matrix_to_json
from paper_2110_10401_b200.decompose import DEFAULT_TREE_THRESHOLD
from paper_2110_10401_b200.matrix import CommMatrix
from tests.conftest import load_golden


def test_combined_matrix_files_from_expected_results():
    cases = {c["name"]: c for c in load_golden("traces.json.gz")}
    checked = 0
    for run in load_golden("cli.json.gz"):
        if run["flags"] != [] or run["code"] != 0 or isinstance(run["trace"], list):
            continue
        case = cases[run["trace"]]
        if case["ring_order"] or case["d"] is not None or case["tree_threshold"] != DEFAULT_TREE_THRESHOLD:
            continue  # expected result computed under a non-default config
        res = case["result"]
        m = CommMatrix.from_rows(res["d"], res["combined"], res["combined_agg"])
        assert matrix_to_csv(m) == run["files"]["matrix_combined.csv"], run["trace"]
        meta = {k: v for k, v in __import__("json").loads(run["files"]["matrix_combined.json"]).items()
                if k in ("trace_digest", "symmetrized")}
        assert matrix_to_json(m, meta) == run["files"]["matrix_combined.json"], run["trace"]
        checked += 1
    assert checked >= 8
