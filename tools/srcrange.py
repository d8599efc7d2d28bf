"""Instructions per 32-record window by source-line range of ct_fast.cu and by other file:
python tools/srcrange.py page.csv records lo-hi[:name] ..."""
import csv
import sys
from collections import defaultdict

path, records = sys.argv[1], int(sys.argv[2])
ranges = []
for a in sys.argv[3:]:
    span, _, name = a.partition(":")
    lo, hi = map(int, span.split("-"))
    ranges.append((lo, hi, name or span))
inst = defaultdict(int)
cur = None
hdr = None
for r in csv.reader(open(path)):
    if len(r) == 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) < 8 or not r[0].isdigit():
        continue
    try:
        inst[(cur, int(r[0]))] += int(float(r[hdr.index("Instructions Executed")] or 0))
    except ValueError:
        pass
win = records / 32
tot = sum(inst.values())
print(f"total {tot / win:.1f} inst/window")
other = defaultdict(int)
for (f, ln), v in inst.items():
    if f != "ct_fast.cu":
        other[f] += v
for f, v in sorted(other.items(), key=lambda x: -x[1]):
    print(f"  {f:<28} {v / win:6.1f}")
for lo, hi, name in ranges:
    v = sum(x for (f, ln), x in inst.items() if f == "ct_fast.cu" and lo <= ln <= hi)
    print(f"  {name:<28} {v / win:6.1f}")
top = sorted(((v, k) for k, v in inst.items()), reverse=True)[:25]
for v, k in top:
    print(f"    {k[0]}:{k[1]} {v / win:6.1f}")
