"""Debug helper: analyze golden cases on the GPU and print the first differing fields."""
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
for case in cases:
    if names and case["name"] not in names:
        continue
    got, _ = run_case(case, lambda ev, d, cfg: matrix.analyze_packed(pack_events(ev), d=d, config=cfg, force_path=force))
    want = {k: case[k] for k in ("error", "result") if k in case}
    if got == want:
        continue
    print("==", case["name"])
    if "result" in got and "result" in want:
        for k in want["result"]:
            if got["result"].get(k) != want["result"][k]:
                print("  field", k)
                print("   got ", str(got["result"].get(k))[:600])
                print("   want", str(want["result"][k])[:600])
    else:
        print("  got ", str(got)[:300])
        print("  want", str(want)[:300])
    shown += 1
    if shown >= 6:
        break
print("done")
