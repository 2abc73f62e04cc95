"""Profiling aid: configs[1] step time with the residual pass on/off (device-timed, 10 steps)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2007_10798_b200 as rocp
from bench import CONFIGS, auto_s, make_factors

cfg = CONFIGS["c2"]
dims, R, t_init, B = cfg["dims"], cfg["rank"], cfg["t_init"], cfg["batch"]
S = auto_s(R)
g = np.random.default_rng(1000)
dev = rocp.Device(0)
X = dev.tensor(dims)
X.generate(make_factors(dims, R, cfg["family"], g), snr_db=cfg["snr_db"], noise_seed=2000)
init = rocp.cprand_decompose(dev, X.slab(0, t_init), R, [np.asfortranarray(g.standard_normal((d, R))) for d in dims[:-1] + [t_init]],
                             seed=3000, tol=cfg["tol"], max_iters=cfg["max_iters"])
st = rocp.RocpStream(dev, init, S, t_capacity=dims[-1] + 8)
st.checkpoint()
nb = (dims[-1] - t_init) // B
for level in (1, 0, 1):
    st.set_residual_tracking(level)
    for w in range(3):
        st.restore()
        st.consume_range(X, t_init, B, nb, 100 + w, 1)
    dev.synchronize()
    dev.timer_record(0)
    for k in range(10):
        st.restore()
        st.consume_range(X, t_init, B, nb, 200 + k, 1)
    dev.timer_record(1)
    ms = dev.timer_elapsed_ms(0, 1) / 10
    print(f"resid_level={level}: {ms:.3f} ms/step ({nb * B / ms * 1e3:.0f} slices/s)")
