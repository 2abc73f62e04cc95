import sys, time
import os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import bench
import paper_2007_10798_b200 as rocp
cfg = bench.CONFIGS[sys.argv[1]]
dims, R, t_init = cfg["dims"], cfg["rank"], cfg["t_init"]
dev = rocp.Device(0)
g = np.random.default_rng(1000)
X = dev.tensor(dims)
X.generate(bench.make_factors(dims, R, cfg["family"], g), snr_db=cfg["snr_db"], noise_seed=2000)
dev.synchronize()
for k in range(3):
    t0 = time.perf_counter()
    init = rocp.cprand_decompose(dev, X.slab(0, t_init), R, bench.init_factors(cfg, 0), seed=3000, tol=cfg["tol"], max_iters=cfg["max_iters"])
    print(sys.argv[1], "cprand", k, round(time.perf_counter() - t0, 4), "s", init.iterations, "sweeps", dev.kernel_launches, "launches")
