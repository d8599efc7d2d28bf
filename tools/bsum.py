"""Print a one-line summary of a bench.py JSON line read from stdin: tools/bsum.py <label>."""
import json
import sys

label = " ".join(sys.argv[1:])
for line in sys.stdin:
    line = line.strip()
    if not line.startswith("{"):
        continue
    d = json.loads(line)
    rf = d.get("roofline") or {}
    print(label, d["config"]["workload"][:3], f"{d['value'] / 1e9:.2f} Grec/s", f"frac={rf.get('frac', 0):.3f}",
          f"kernel_ms={rf.get('kernel_ms', 0):.2f}", f"path={d.get('path')}")
