"""Sum an ncu --metrics gpu__time_duration.sum CSV launch list per kernel: tools/launchsum.py file.csv [calls]"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
calls = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
h, agg, cnt = None, defaultdict(float), defaultdict(int)
for r in rows:
    if "Kernel Name" in r:
        h = r
        continue
    if h and len(r) == len(h) and r[h.index("Metric Name")] == "gpu__time_duration.sum":
        k = r[h.index("Kernel Name")][:70]
        agg[k] += float(r[h.index("Metric Value")].replace(",", ""))
        cnt[k] += 1
tot = sum(agg.values())
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:20]:
    print(f"{v / 1e3 / calls:9.1f} us/call  x{cnt[k]:4d}  {100 * v / tot:5.1f}%  {k}")
