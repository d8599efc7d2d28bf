"""Debug helper: analyze golden cases on the GPU and print differing cells per type."""
import sys

sys.path.insert(0, ".")
from tests.conftest import load_golden  # noqa: E402
from tests.helpers import run_case  # noqa: E402
from paper_2110_10401_b200 import matrix  # noqa: E402
from paper_2110_10401_b200.packed import pack_events  # noqa: E402

force = int(sys.argv[1]) if len(sys.argv) > 1 else 0
names = set(sys.argv[2:])
cases = load_golden("traces.json.gz")
shown = 0
paths = {}


def analyze(ev, d, cfg):
    r = matrix.analyze_packed(pack_events(ev), d=d, config=cfg, force_path=force)
    paths["last"] = r.path
    return r


for case in cases:
    if names and case["name"] not in names:
        continue
    got, _ = run_case(case, analyze)
    want = {k: case[k] for k in ("error", "result") if k in case}
    if got == want:
        continue
    print("==", case["name"], "path", paths.get("last"))
    if "result" in got and "result" in want:
        g, w = got["result"], want["result"]
        for k in w:
            if k == "per_primitive":
                gp = {x[0]: x for x in g[k]}
                for x in w[k]:
                    y = gp.get(x[0])
                    if y is None or y[1:] != x[1:]:
                        cells = [(i, j, y[1][i][j] if y else None, x[1][i][j]) for i in range(len(x[1]))
                                 for j in range(len(x[1])) if not y or y[1][i][j] != x[1][i][j]]
                        print("  type", x[0], "cells(got,want)", cells[:8])
            elif g.get(k) != w[k] and k not in ("combined", "combined_freq"):
                print("  field", k, "got", str(g.get(k))[:300], "want", str(w[k])[:300])
    else:
        print("  got ", str(got)[:300])
        print("  want", str(want)[:300])
    shown += 1
    if shown >= 8:
        break
print("done")
