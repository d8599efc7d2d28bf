"""Instruction counts per kernel region (per 32-record window) from an ncu source CSV.
python tools/regions.py page.csv records"""
import csv
import re
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
win = int(sys.argv[2]) / 32
inst = defaultdict(int); cur = None; hdr = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur = r[1].split('/')[-1]; continue
    if r and r[0] == "Line No":
        hdr = r; continue
    if not hdr or len(r) < 8 or not r[0].isdigit():
        continue
    try:
        inst[(cur, int(r[0]))] += int(float(r[hdr.index("Instructions Executed")] or 0))
    except ValueError:
        pass
src = open('paper_2110_10401_b200/csrc/ct_fast.cu').read().split('\n')
marks = [(i + 1, m.group(1)) for i, l in enumerate(src) for m in [re.search(r'// REGION (\w+)', l)] if m]
fast = {k[1]: v for k, v in inst.items() if k[0] == 'ct_fast.cu'}
print(f"total {sum(inst.values()) / win:.1f}  other files {sum(v for k, v in inst.items() if k[0] != 'ct_fast.cu') / win:.1f}")
for (a, name), nxt in zip(marks, marks[1:] + [(10 ** 9, 'end')]):
    print(f"{name:16s} {a:5d} {sum(v for l, v in fast.items() if a <= l < nxt[0]) / win:7.1f}")
