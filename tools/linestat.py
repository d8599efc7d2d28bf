"""Per-source-line executed instructions and stall samples from an ncu source page CSV,
normalised per 32-record window.  python tools/linestat.py page.csv records [top]"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
win = int(sys.argv[2]) / 32
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
inst = defaultdict(int); samp = defaultdict(int); txt = {}; cur = None; hdr = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur = r[1].split('/')[-1]; continue
    if r and r[0] == "Line No":
        hdr = r; continue
    if not hdr or len(r) < 8 or not r[0].isdigit():
        continue
    k = (cur, int(r[0])); txt[k] = r[1][:90]
    try:
        inst[k] += int(float(r[hdr.index("Instructions Executed")] or 0))
        samp[k] += int(float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0))
    except ValueError:
        pass
ti = sum(inst.values()); ts = sum(samp.values())
print(f"inst/window {ti / win:.1f}")
for k in sorted(samp, key=lambda k: -samp[k])[:top]:
    print(f"{k[0][:12]:>12}:{k[1]:<4} samp {100 * samp[k] / ts:5.1f}% inst/win {inst[k] / win:6.1f}  {txt[k]}")
