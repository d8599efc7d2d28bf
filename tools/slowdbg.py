import os, sys
sys.path.insert(0, os.getcwd())
from tests.test_gpu_loader import _generated_text
from paper_2110_10401_b200.loader import load_trace
block = _generated_text(3, 20000, seed=7)
tr = load_trace(block)
print(tr.load_info)
lines = block.splitlines()
import re
for n in (1, 2, 3):
    print(repr(lines[n - 1]))
for a in sys.argv[1:]:
    print(a, repr(lines[int(a) - 1]))
