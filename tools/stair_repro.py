"""Minimal repro of one tests/test_stair.py case (for compute-sanitizer).
usage: stair_repro.py DIM WINDOW TYPES STAIR(0|1)"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
import test_stair  # noqa: E402
fw = test_stair.fw

dim, window, types, stair = (int(a) for a in sys.argv[1:5])
n_neg = 5
rng = np.random.default_rng(dim * 100 + window * 10 + types)
n_sent, band = 24, 600
V = n_sent * band
counts = (10 + V - np.arange(V)).astype(np.uint64)
launches = []
for _ in range(3):
    lens = rng.integers(1, 90, n_sent)
    lens[:4] = [1, 2, 3, 2 * window + 3][:4]
    launches.append(test_stair._disjoint_launch(rng, n_sent, band, lens, n_neg, types))
inp = ((rng.random((V, dim)) - 0.5) / dim).astype(np.float32)
out = ((rng.random((V, dim)) - 0.5) * 0.5).astype(np.float32)
cfg = fw.TrainConfig(dim=dim, window=window, negatives=n_neg, workers=4, deterministic=0, reuse_mode="lifetime",
                     fast_sigmoid=True, delta_writeback=2, l1_refresh_log2=0, hot_rows=0)
test_stair._run(bool(stair), cfg, counts, inp, out, launches)
print("ok")
