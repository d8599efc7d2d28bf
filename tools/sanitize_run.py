"""Small mixed traces through the fast kernel, for compute-sanitizer runs (GPU box):
    compute-sanitizer --tool racecheck python tools/sanitize_run.py"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests.test_gpu_paths import Gen, _gpu  # noqa: E402

for seed, n_comms, pool in ((0, 6, 8), (1, 7, 8), (2, 4, 70)):
    g = Gen(np.random.default_rng(seed), n_comms=n_comms, dev_pool=pool, diag=0.02, dev_change=0.02).mixed(60_000)
    s, cells, freq = _gpu(g.array(), n_comms)
    print("seed", seed, "status", s.status, "path", s.path, "calls", list(s.calls)[:5])
