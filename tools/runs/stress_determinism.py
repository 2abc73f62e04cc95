"""Stress check of the cross-block / cross-kernel synchronisation (overlapped gather, chunk
arrival counters): the same configs[1] window replayed many times, with several gather-SM splits,
must give bit-identical factors every time (and equal the serial-gather result)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2007_10798_b200 as rocp
from bench import CONFIGS, auto_s, make_factors

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
cfg = CONFIGS[name]
dims, R, t_init, B = cfg["dims"], cfg["rank"], cfg["t_init"], cfg["batch"]
S = auto_s(R)
g = np.random.default_rng(7)
dev = rocp.Device(0)
X = dev.tensor(dims)
X.generate(make_factors(dims, R, cfg["family"], g), snr_db=cfg["snr_db"], noise_seed=11)
init = rocp.cprand_decompose(dev, X.slab(0, t_init), R,
                             [np.asfortranarray(g.standard_normal((d, R))) for d in dims[:-1] + [t_init]], seed=13,
                             tol=cfg["tol"], max_iters=cfg["max_iters"])
st = rocp.RocpStream(dev, init, S, t_capacity=dims[-1] + 8)
st.checkpoint()
nb = (dims[-1] - t_init) // B


def run(sms):
    dev.set_gather_sms(sms)
    st.restore()
    st.consume_range(X, t_init, B, nb, 4321, 1)
    out = [st.factor(n).copy() for n in range(1, len(dims))] + [st.temporal().copy(), st.last_residuals().copy()]
    return [a.view(np.uint64) for a in out]


ref = run(0)
bad = 0
for sms in (8, 12, 20, 32, -1):
    for k in range(reps):
        got = run(sms)
        if not all(np.array_equal(a, b) for a, b in zip(ref, got)):
            bad += 1
            print(f"MISMATCH sms={sms} rep={k}", flush=True)
print(f"{name}: {5 * reps} replays, {bad} mismatches")
sys.exit(1 if bad else 0)
