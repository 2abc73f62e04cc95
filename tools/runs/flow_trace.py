"""Profiling aid: per-stage timeline of k_flow (globaltimer stamps, traced build).
Usage: python tools/runs/flow_trace.py [c1|c2|c3|c5]  (env ROCP_GATHER_SMS to fix the split)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2007_10798_b200 as rocp  # noqa: E402

CFG = {"c1": ([200, 200, 500], 10, 50, 10), "c2": ([1000, 1000, 1000], 20, 100, 25),
       "c3": ([200, 200, 200, 200], 10, 20, 10), "c5": ([60, 60, 60, 60, 300], 16, 10, 10),
       "c4": ([4000, 4000, 500], 50, 50, 50)}
dims, R, t_init, B = CFG[sys.argv[1] if len(sys.argv) > 1 else "c2"]
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
tr_i = st.chain_trace(False).astype(np.int64)
base = tr_i[tr_i > 0].min()
tr = np.where(tr_i > 0, tr_i - base, -1).astype(float)
tr[tr < 0] = np.nan
N = len(dims)
pub = tr[:, 4]
prev = np.concatenate([[np.nan], pub[:-1]])  # previous stage's publish


def med(a):
    a = a[np.isfinite(a)]
    return np.median(a) / 1e3 if a.size else float("nan")


print(f"gather SMs {st.last_gather_sms}")
for stg in range(N):
    t = tr[stg::N]
    p0 = prev[stg::N]
    print(f"stage {stg}: chunk start={med(t[:,0]-p0):.2f} chunk pub={med(t[:,1]-t[:,0]):.2f} (od={med(t[:,12]-t[:,0]):.2f} [ginv staged {med(t[:,15]-t[:,0]):.2f} w in {med(t[:,16]-t[:,0]):.2f}] z={med(t[:,14]-t[:,12]):.2f}) | "
          f"fin wait done={med(t[:,3]-t[:,1]):.2f} combine={med(t[:,10]-t[:,3]):.2f} solve={med(t[:,11]-t[:,10]):.2f} publish={med(t[:,4]-t[:,11]):.2f} | stage={med(t[:,4]-p0):.2f} | "
          f"mat0 done={med(t[:,5]-p0):.2f} item0 gather ok={med(t[:,7]-p0):.2f} item0 start={med(t[:,8]-p0):.2f} "
          f"computed={med(t[:,19]-p0):.2f} end={med(t[:,9]-p0):.2f} last tsum={med(t[:,6]-p0):.2f} us")
print("whole window us:", (np.nanmax(tr[:, 4]) - np.nanmin(tr[:, 1])) / 1e3)
