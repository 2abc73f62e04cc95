"""Profiling aid: K7 fitness sweep time (model pass + norm pass are launched per call; the call
also forms the norm once).  Usage: python tools/runs/fitness_time.py [c2|c4]"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2007_10798_b200 as rocp  # noqa: E402

CFG = {"c2": ([1000, 1000, 100], 20), "c4": ([4000, 4000, 50], 50), "c1": ([200, 200, 50], 10)}
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
dims, R = CFG[name]
g = np.random.default_rng(0)
dev = rocp.Device(0)
X = dev.tensor(dims)
F = [np.asfortranarray(g.standard_normal((d, R))) for d in dims]
X.generate(F, snr_db=20.0, noise_seed=1)
for _ in range(3):
    f = rocp.model_fitness(dev, X, F)
dev.synchronize()
n = 20
dev.timer_record(0)
for _ in range(n):
    f = rocp.model_fitness(dev, X, F)
dev.timer_record(1)
dev.synchronize()
ms = dev.timer_elapsed_ms(0, 1) / n
gb = np.prod(dims) * 8 / 1e9
print(f"{name}: fitness {f:.6f}; {ms:.4f} ms per call ({gb:.2f} GB tensor; includes factor upload and the launches of one call)")
