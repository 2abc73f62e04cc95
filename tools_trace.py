"""Profiling aid: per-phase timeline of the persistent chain kernel (globaltimer stamps)."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import paper_2007_10798_b200 as rocp

dims, R, t_init, B = [1000, 1000, 1000], 20, 100, 25
if len(sys.argv) > 1:
    cfg = json.loads(sys.argv[1])
    dims, R, t_init, B = cfg["dims"], cfg["R"], cfg["t_init"], cfg["B"]
S = max(R, int(np.ceil(10 * R * np.log(R))))
g = np.random.default_rng(0)
dev = rocp.Device(0)
X = dev.tensor(dims)
X.generate([np.asfortranarray(g.standard_normal((d, R))) for d in dims], snr_db=20.0, noise_seed=1)
init = rocp.cprand_decompose(dev, X.slab(0, t_init), R,
                             [np.asfortranarray(g.standard_normal((d, R))) for d in dims[:-1] + [t_init]], seed=3)
st = rocp.RocpStream(dev, init, S, t_capacity=dims[-1] + 8)
st.checkpoint()
nb = (dims[-1] - t_init) // B
for k in range(3):
    st.restore()
    st.consume_range(X, t_init, B, nb, 100 + k, 1)
st.chain_trace(True, fetch=False)
st.restore()
st.consume_range(X, t_init, B, nb, 200, 1)
tr = st.chain_trace(False).astype(np.int64)
N = len(dims)


def med(a):
    a = a[np.isfinite(a)]
    return np.median(a) / 1e3 if a.size else float("nan")


for stg in range(N):
    t = tr[stg::N].astype(float)
    t[t == 0] = np.nan
    z = lambda k: t[:, k] - t[:, 0]
    print(f"stage {stg}: z(block0)={med(t[:,14]-t[:,0]):.2f} chunk-gram={med(t[:,15]-t[:,14]):.2f} p0+sync={med(z(1)):.2f} | item0 ready={med(t[:,8]-t[:,1]):.2f} compute={med(t[:,9]-t[:,8]):.2f} | "
          f"gram->factor start={med(t[:,3]-t[:,1]):.2f} combine={med(t[:,10]-t[:,3]):.2f} prologue={med(t[:,12]-t[:,10]):.2f} "
          f"ldlt={med(t[:,13]-t[:,12]):.2f} check={med(t[:,11]-t[:,13]):.2f} publish={med(t[:,4]-t[:,11]):.2f} | "
          f"tma-wait={med(t[:,18]-t[:,3]):.2f} | sync1 done={med(z(5)):.2f} LD ready={med(t[:,16]-t[:,5]):.2f} row loop={med(t[:,17]-t[:,16]):.2f} rows={med(t[:,6]-t[:,5]):.2f} sync2={med(t[:,7]-t[:,6]):.2f} | total={med(t[:,7]-t[:,0]):.2f} us")
if tr.shape[1] > 23 and tr[:, 20:24].any():
    for stg in range(N):
        t = tr[stg::N].astype(float)
        print(f"stage {stg}: streamed items, cycles per ring step: warp 0 data wait {np.median(t[:,20]):.0f}, block wait {np.median(t[:,21]):.0f}, "
              f"MMA section {np.median(t[:,22]):.0f}; warp 4 (issuer) MMA section {np.median(t[:,23]):.0f}")
print("whole window us:", (tr[-1, 7] - tr[0, 0]) / 1e3)
print("residual of last batch:", st.last_residuals()[0])
