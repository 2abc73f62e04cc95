"""Config-size GPU checks (BASELINE.json configs[1..4] = SURVEY.md C2..C5).

At full size the oracle cannot replay cprand or a whole stream in seconds, so:
  * the data is generated on the device (gen_synthetic semantics,
    synthetic.cpp:8-31) from seeded factors of each config's family;
  * cprand runs on the GPU at full size; its reported best fitness must equal
    an independent model_fitness launch on the returned model, bit for bit;
  * the stream consumes WARM batches on the GPU, then one more batch is
    TEACHER-FORCED: the oracle stream is loaded with the GPU state (factors,
    P, Q, temporal, flag) and both consume the same slab with the same
    counter key -- every factor, P, Q, temporal row, flag and the sampled
    residuals must agree bit for bit;
  * size-independent properties: old temporal rows frozen (test_rocp.cpp:243-256),
    Q symmetric and PSD (test_rocp.cpp:217-232), the streamed batch fitted close to
    its noise floor.
"""
import gc

import numpy as np
import pytest

import paper_2007_10798_b200 as rocp
from oracle import oracle as orc
from tests import helpers as H

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

# name, dims, R, t_init, B, snr_db, factor family, warm batches before the forced one
CONFIGS = [
    ("C2", [1000, 1000, 1000], 20, 100, 25, 20.0, "normal", 3),
    ("C3", [200, 200, 200, 200], 10, 20, 10, 30.0, "uniform", 3),
    ("C4", [4000, 4000, 500], 50, 50, 50, 20.0, "normal", 2),
    ("C5", [60, 60, 60, 60, 300], 16, 10, 10, 10.0, "congruent", 3),
]


def bitwise(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


def _factors(dims, R, family, g):
    if family == "uniform":
        return [np.asfortranarray(g.random((d, R))) for d in dims]
    if family == "congruent":
        return H.congruent_factors(dims, R, 0.9, g)
    return H.random_model(dims, R, g)


@pytest.mark.parametrize("name,dims,R,t_init,B,snr,family,warm", CONFIGS, ids=[c[0] for c in CONFIGS])
def test_config_size_stream(dev, name, dims, R, t_init, B, snr, family, warm):
    g = H.rng(7000 + R)
    truth = _factors(dims, R, family, g)
    X = dev.tensor(dims)
    X.generate(truth, snr_db=snr, noise_seed=11)
    head = dims[:-1]
    ideal = 1.0 - 10.0 ** (-snr / 20.0)  # fit of the noise-free model

    # ---- init (cprand.cpp:12-69), full size on the GPU
    X0 = X.slab(0, t_init)
    init0 = H.random_model(head + [t_init], R, H.rng(5))
    init = rocp.cprand_decompose(dev, X0, R, init0, seed=31)
    assert init.iterations >= 1
    fit0 = rocp.model_fitness(dev, X0, init.model)
    assert bitwise(np.float64(fit0), np.float64(init.best_fitness)), (fit0, init.best_fitness)
    assert init.best_fitness > 0.5 * ideal, (name, init.best_fitness, ideal)

    s = init.samples
    assert s == rocp.auto_sample_count(R)
    st = rocp.RocpStream(dev, init, s, t_capacity=dims[-1])
    seed = 424242
    for k in range(warm):
        st.consume(X.slab(t_init + k * B, B), seed, k + 1)

    # ---- teacher-forced batch: oracle loaded with the GPU state
    t0 = t_init + warm * B
    old_temporal = st.temporal()
    orc_st = orc.Stream([st.factor(n) for n in range(1, len(dims))] + [old_temporal], st.t_len,
                        [np.zeros((s, R), order="F") for _ in range(len(dims) - 1)], s,
                        regularized=st.regularized)
    for n in range(1, len(dims)):
        orc_st.set(1, n, st.p(n))
        orc_st.set(2, n, st.q(n))
    slab = X.slab(t0, B)
    st.consume(slab, seed, warm + 1)
    orc_st.consume(slab.download(), B, seed, warm + 1)
    for n in range(1, len(dims)):
        assert bitwise(st.factor(n), orc_st.factor(n)), f"{name} U{n}"
        assert bitwise(st.p(n), orc_st.p(n)), f"{name} P{n}"
        assert bitwise(st.q(n), orc_st.q(n)), f"{name} Q{n}"
    new_temporal = st.temporal()
    assert bitwise(new_temporal, orc_st.temporal()), f"{name} temporal"
    assert st.regularized == orc_st.regularized
    ra = st.last_residuals()
    rb = np.zeros(len(dims))
    import ctypes as C
    orc.lib().orc_stream_last_residuals(orc_st._h, rb.ctypes.data_as(C.POINTER(C.c_double)))
    assert bitwise(ra, rb), (ra, rb)

    # ---- properties
    assert bitwise(new_temporal[:old_temporal.shape[0]], old_temporal)  # frozen rows
    for n in range(1, len(dims)):
        q = st.q(n)
        assert bitwise(q, q.T), f"{name} Q{n} symmetric"
        ev = np.linalg.eigvalsh(q)
        assert ev.min() >= -1e-10 * max(1.0, abs(ev).max()), f"{name} Q{n} PSD"
    model = [st.factor(n) for n in range(1, len(dims))] + [new_temporal[-B:]]
    fit_batch = rocp.model_fitness(dev, slab, model)
    floor = 0.5 if family == "congruent" else 0.9
    assert fit_batch > floor * ideal, (name, fit_batch, ideal)
    print(f"{name}: init fit {init.best_fitness:.6f} ({init.iterations} sweeps), "
          f"batch fit {fit_batch:.6f}, ideal {ideal:.6f}, residuals {ra}")
    del st, slab, X0, X
    gc.collect()
