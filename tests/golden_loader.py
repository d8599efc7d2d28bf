"""Load a named golden case (used by __graft_entry__.smoke and tests)."""

import gzip
import json
import os

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_case(name):
    with gzip.open(os.path.join(GOLDEN, "traces.json.gz"), "rt", encoding="utf-8") as fh:
        for case in json.load(fh):
            if case["name"] == name:
                return case
    raise KeyError(name)
