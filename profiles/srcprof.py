"""Summarise an ncu source page (cuda,sass CSV) by CUDA source line: instructions
executed and warp-stall samples.  Usage: python profiles/srcprof.py page.csv [top]"""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
inst = defaultdict(int)
samp = defaultdict(int)
text = {}
cur_file = None
with open(path) as fh:
    rows = list(csv.reader(fh))
hdr = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) < 8 or not r[0].isdigit():
        continue
    key = (cur_file, int(r[0]))
    text[key] = r[1][:90]
    try:
        inst[key] += int(float(r[hdr.index("Instructions Executed")] or 0))
        samp[key] += int(float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0))
    except ValueError:
        pass
tot_i = sum(inst.values()) or 1
tot_s = sum(samp.values()) or 1
print(f"total inst {tot_i:.3e}  samples {tot_s}")
for key in sorted(samp, key=lambda k: -samp[k])[:top]:
    print(f"{key[0]:>14}:{key[1]:<4} samp {100*samp[key]/tot_s:5.1f}%  inst {100*inst[key]/tot_i:5.1f}%  {text[key]}")
