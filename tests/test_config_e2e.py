"""End-to-end config-size parity: the bench's exact path against the oracle.

For BASELINE.json configs[1], [2], [4] the tensor is built
by bench.synth_host (the bytes bench.py streams, and the reference arm too), then:
  * cprand_decompose runs at full size on the GPU and in the oracle
    (orc_cprand) from the same initial model and counter seed -- every factor,
    the Z_best rebuild, the fitness, the sweep count and the flag agree bit for bit;
  * the whole post-init stream runs through exactly the bench's call
    (RocpStream::consume_range over the full window, one persistent chain, the
    overlapped gather on the SMs the model chooses) and through the oracle's
    RocpStream::consume batch by batch -- every factor, P, Q, temporal row, flag
    and the last batch's sampled residuals agree bit for bit.
configs[3] (C4, 4000 x 4000 x 500, R = 50, 64 GB): the first cprand sweep at full
size is compared bit for bit (max_iters = 1: the oracle's full-fit sweeps over the
6.4 GB init slab are the expensive part), then the full 9-batch window from that
init on both sides.
The reference's own recursion check (acceptance.cpp:80-124) and SURVEY Appendix A
(C5 is chaotic: any rounding difference grows to O(1)) are why this is bitwise.
"""
import ctypes as C
import gc

import numpy as np
import pytest

import bench
import paper_2007_10798_b200 as rocp
from oracle import oracle as orc

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def bitwise(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


def _cprand_pair(dev, cfg, x, X, max_iters=None):
    dims, R, t_init = cfg["dims"], cfg["rank"], cfg["t_init"]
    slice_ = int(np.prod(dims[:-1]))
    it = cfg["max_iters"] if max_iters is None else max_iters
    init0 = bench.init_factors(cfg, 0)
    a = rocp.cprand_decompose(dev, X.slab(0, t_init), R, init0, seed=3000, tol=cfg["tol"], max_iters=it)
    b = orc.cprand_decompose(x[:t_init * slice_], dims[:-1] + [t_init], R, init0, seed=3000, tol=cfg["tol"],
                             max_iters=it)
    assert a.iterations == b.iterations and a.regularized == b.regularized
    assert bitwise(np.float64(a.best_fitness), np.float64(b.best_fitness))
    assert bitwise(a.fit_trace, b.fit_trace)
    for n in range(len(dims)):
        assert bitwise(a.model[n], b.model[n]), f"cprand U{n + 1}"
    for n in range(len(dims) - 1):
        assert bitwise(a.best_sampled_kr[n], b.best_sampled_kr[n]), f"cprand Z_best{n + 1}"
    return a, b


def _window_pair(dev, cfg, x, X, a, b, seed=10000):
    dims, R, t_init, B = cfg["dims"], cfg["rank"], cfg["t_init"], cfg["batch"]
    nb = (dims[-1] - t_init) // B
    S = bench.auto_s(R)
    slice_ = int(np.prod(dims[:-1]))
    st = rocp.RocpStream(dev, a, S, t_capacity=dims[-1] + 8)
    st.consume_range(X, t_init, B, nb, seed, 1)  # the bench step (bench.py step())
    ob = orc.Stream(b.model, t_init, b.best_sampled_kr, S, regularized=b.regularized)
    for k in range(nb):
        t0 = t_init + k * B
        ob.consume(x[t0 * slice_:(t0 + B) * slice_], B, seed, k + 1)
    for n in range(1, len(dims)):
        assert bitwise(st.factor(n), ob.factor(n)), f"U{n}"
        assert bitwise(st.p(n), ob.p(n)), f"P{n}"
        assert bitwise(st.q(n), ob.q(n)), f"Q{n}"
    assert bitwise(st.temporal(), ob.temporal()), "temporal"
    assert st.t_len == ob.t_len == t_init + nb * B
    assert st.regularized == ob.regularized
    ra = st.last_residuals()
    rb = np.zeros(len(dims))
    orc.lib().orc_stream_last_residuals(ob._h, rb.ctypes.data_as(C.POINTER(C.c_double)))
    assert bitwise(ra, rb)
    return st.last_gather_sms, nb


@pytest.mark.parametrize("key", ["c2", "c3", "c5"])
def test_config_cprand_and_full_window_bitwise(dev, key):
    cfg = bench.CONFIGS[key]
    x = bench.synth_host(cfg, 0)
    X = dev.tensor(cfg["dims"], x)
    dev.decision_stats(reset=True)
    a, b = _cprand_pair(dev, cfg, x, X)
    gsms, nb = _window_pair(dev, cfg, x, X, a, b)
    stats = dev.decision_stats(reset=True)
    print(f"{key}: cprand {a.iterations} sweeps fit {a.best_fitness:.6f}; {nb} batches through consume_range, "
          f"gather on {gsms} SMs; gram decisions {stats}; bitwise equal to the oracle")
    del X
    gc.collect()


def test_config_c4_sweep_and_window_bitwise(dev):
    cfg = bench.CONFIGS["c4"]
    x = bench.synth_host(cfg, 0)
    X = dev.tensor(cfg["dims"], x)
    a, b = _cprand_pair(dev, cfg, x, X, max_iters=1)
    gsms, nb = _window_pair(dev, cfg, x, X, a, b)
    print(f"c4: first cprand sweep + {nb}-batch window (gather on {gsms} SMs) bitwise equal to the oracle")
    del X
    gc.collect()
