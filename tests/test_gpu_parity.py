"""GPU parity: the CUDA path (librocp_b200.so via the C ABI) against the CPU
oracle on the same seeded inputs.  Integer/index work and every fp64 result
are compared BIT-FOR-BIT (canonical operation order);
tolerance-based reference properties are re-checked on the GPU results.
"""
import json
import os

import numpy as np
import pytest

import paper_2007_10798_b200 as rocp
from oracle import oracle as orc
from tests import helpers as H

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")
KAT = json.load(open(os.path.join(GOLD, "reference_kat.json")))
TOL = {k: v[0] for k, v in KAT["tolerances"].items()}


def bitwise(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64) if a.dtype == np.float64 else a,
                                                  b.view(np.uint64) if b.dtype == np.float64 else b)


# ---- K1 draws -----------------------------------------------------------------
@pytest.mark.parametrize("dims,mode", [([200, 200, 500], 3), ([200, 200, 10], 1), ([200, 200, 10], 2),
                                       ([60, 60, 60, 60, 10], 3), ([4000, 4000, 50], 1),
                                       ([1, 1, 5], 3), ([2, 10], 1)])
def test_draw_bitwise(dev, dims, mode):
    for (seed, batch, it) in [(0, 0, 1), (12345678901234, 7, 0), (2**64 - 1, 2**32 - 1, 2**32 - 1)]:
        r_gpu, d_gpu = rocp.draw_samples(dev, dims, mode, 1957, seed, batch, it)
        r_orc, d_orc = orc.draw_samples(dims, mode, 1957, seed, batch, it)
        assert bitwise(r_gpu, r_orc) and bitwise(d_gpu, d_orc)


def test_draw_reference_pins(dev):
    c = KAT["draw_codomain_one"]
    rows, _ = rocp.draw_samples(dev, c["dims"], c["mode"], c["s"], 1, 0, 0)
    assert rows.tolist() == c["rows"]
    with pytest.raises(rocp.DomainError):
        rocp.draw_samples(dev, [2, 2], 1, 0, 1)
    for cc in KAT["decode_index"]:
        dec = rocp.decode_rows(dev, cc["dims"], cc["mode"], [cc["j"]])
        assert dec[0].tolist() == cc["multi"]
    with pytest.raises(rocp.DomainError):
        rocp.decode_rows(dev, [2, 3, 4], 1, [13])


# ---- K2 gather ------------------------------------------------------------------
@pytest.mark.parametrize("dims", [[3, 4, 5], [20, 30, 7], [6, 5, 4, 3, 2], [200, 200, 10]])
def test_gather_bitwise(dev, dims):
    g = H.rng(55)
    t = g.standard_normal(int(np.prod(dims)))
    T = dev.tensor(dims, t)
    for mode in range(1, len(dims) + 1):
        rows, dec = orc.draw_samples(dims, mode, 231, 9, 1, 0)
        assert bitwise(rocp.sample_unfolding(dev, T, mode, rows), orc.sample_unfolding(t, dims, mode, dec))


def test_gather_reference_pins(dev):
    dims = [3, 4, 5]
    t = H.rng(55).standard_normal(60)
    T = dev.tensor(dims, t)
    for mode in (1, 2, 3):  # all columns in order == unfold (test_factor_model.cpp:145-150)
        co = orc.codomain_size(dims, mode)
        allr = np.arange(1, co + 1)
        assert bitwise(rocp.sample_unfolding(dev, T, mode, allr),
                       orc.sample_unfolding(t, dims, mode, orc.from_rows(dims, mode, allr)))
    dup = rocp.sample_unfolding(dev, T, 1, [4, 4])
    assert bitwise(dup[:, 0], dup[:, 1])
    c = KAT["unfold_mode1_2x2"]
    T2 = dev.tensor(c["dims"], np.array(c["data"], float))
    assert rocp.sample_unfolding(dev, T2, 1, [1, 2]).tolist() == c["matrix_rowwise"]
    with pytest.raises(rocp.DomainError):  # index set drawn against other dims (:164-167)
        rocp.sample_unfolding(dev, T, 1, [21])


# ---- K3 sampled Khatri-Rao ------------------------------------------------------------
@pytest.mark.parametrize("dims,rank", [([3, 4, 5], 3), ([2, 3, 4, 5], 1), ([3, 3, 3, 3], 4),
                                       ([60, 50, 40, 30, 10], 16), ([200, 200, 50], 50)])
def test_skr_bitwise(dev, dims, rank):
    model = H.random_model(dims, rank, H.rng(73))
    for mode in range(1, len(dims) + 1):
        fs = orc.factors_excluding(model, mode)
        _, dec = orc.draw_samples(dims, mode, 300, 5, 0, 1)
        assert bitwise(rocp.sampled_khatri_rao(dev, dec, fs), orc.sampled_khatri_rao(dec, fs))


def test_skr_exhaustive_equals_full_kr(dev):
    for dims in ([3, 3], [2, 3, 4], [3, 3, 3, 3]):
        for rank in (1, 4):
            model = H.random_model(dims, rank, H.rng(73))
            for mode in range(1, len(dims) + 1):
                fs = orc.factors_excluding(model, mode)
                co = orc.codomain_size(dims, mode)
                z = rocp.sampled_khatri_rao(dev, orc.from_rows(dims, mode, np.arange(1, co + 1)), fs)
                assert bitwise(z, orc.khatri_rao_list(fs))
    model = H.random_model([2, 3], 2, H.rng(79))
    with pytest.raises(rocp.DomainError):
        rocp.sampled_khatri_rao(dev, orc.from_rows([5, 3], 2, [4]), orc.factors_excluding(model, 2))


# ---- K4 contraction + Gram ---------------------------------------------------------------
@pytest.mark.parametrize("I,s,R", [(10, 231, 10), (200, 231, 10), (1000, 600, 20), (60, 444, 16),
                                   (333, 1957, 50), (7, 33, 3), (5, 1, 1), (130, 65, 7)])
def test_contract_gram_bitwise(dev, I, s, R):
    g = H.rng(I * 7 + s)
    x = H.random_matrix(I, s, g)
    z = H.random_matrix(s, R, g)
    assert bitwise(rocp.gram(dev, z), orc.gram(z))
    assert bitwise(rocp.contract(dev, x, z), orc.contract(x, z))


# ---- K5 solve ------------------------------------------------------------------------------
@pytest.mark.parametrize("R,rows", [(1, 3), (3, 5), (10, 200), (16, 60), (20, 1000), (50, 4000),
                                    (33, 17), (64, 70)])
def test_solve_gram_bitwise(dev, R, rows):
    g = H.rng(R * 1000 + rows)
    z = H.random_matrix(3 * R + 5, R, g)
    G = orc.gram(z)
    rhs = H.random_matrix(rows, R, g)
    u_gpu, reg_gpu = rocp.solve_gram(dev, G, rhs)
    u_orc, reg_orc = orc.solve_gram(G, rhs)
    assert bitwise(u_gpu, u_orc) and reg_gpu == reg_orc


def test_solve_flags_and_pins(dev):
    g = H.rng(101)
    x = H.random_matrix(5, 3, g)
    u, reg, und = rocp.solve_sampled_ls(dev, np.eye(3), x)
    assert np.abs(u - x).max() < TOL["sampled_ls_identity"] and not reg and not und
    zq, _ = np.linalg.qr(g.standard_normal((20, 3)))
    xx = H.random_matrix(6, 20, g)
    u, _, _ = rocp.solve_sampled_ls(dev, zq, xx)
    assert np.abs(u - xx @ zq).max() < TOL["sampled_ls_orthonormal"]
    u0 = H.random_matrix(6, 3, g)
    z = H.random_matrix(20, 3, g)
    u, _, _ = rocp.solve_sampled_ls(dev, z, u0 @ z.T)
    assert np.linalg.norm(u - u0) <= TOL["sampled_ls_planted"] * np.linalg.norm(u0)
    # rank-deficient sampling: underdetermined + regularized, finite (test_cprand.cpp:59-67)
    zz, xr = H.random_matrix(2, 4, g), H.random_matrix(3, 2, g)
    u, reg, und = rocp.solve_sampled_ls(dev, zz, xr)
    uo, rego, undo = orc.solve_sampled_ls(zz, xr)
    assert und and reg and np.isfinite(u).all() and bitwise(u, uo) and rego
    # zero sampling matrix: zero solution + flag (:69-74)
    u, reg, _ = rocp.solve_sampled_ls(dev, np.zeros((5, 2)), H.random_matrix(3, 5, g))
    assert reg and (u == 0).all()
    with pytest.raises(rocp.DomainError):
        rocp.solve_sampled_ls(dev, np.zeros((5, 2)), np.zeros((3, 4)))


def test_solve_sampled_ls_bitwise(dev):
    g = H.rng(11)
    z = H.random_matrix(231, 10, g)
    x = H.random_matrix(200, 231, g)
    a = rocp.solve_sampled_ls(dev, z, x)
    b = orc.solve_sampled_ls(z, x)
    assert bitwise(a[0], b[0]) and a[1:] == b[1:]


# ---- K7 fitness -------------------------------------------------------------------------------
@pytest.mark.parametrize("dims,R", [([3, 4, 5], 2), ([200, 200, 20], 10), ([60, 20, 20, 10], 16),
                                    ([37, 5, 3, 2, 2], 7), ([1, 1, 1], 1), ([70, 300, 40], 50)])
def test_fitness_bitwise(dev, dims, R):
    g = H.rng(23)
    model = H.random_model(dims, R, g)
    x = H.reconstruct(model, dims) + 0.3 * g.standard_normal(int(np.prod(dims)))
    T = dev.tensor(dims, x)
    f_gpu = rocp.model_fitness(dev, T, model)
    f_orc = orc.model_fitness(x, dims, model)
    assert bitwise(np.float64(f_gpu), np.float64(f_orc))


def test_fitness_pins(dev):
    c = KAT["fitness_single_entry"]
    one = np.ones((1, 1))
    T = dev.tensor([1, 1, 1], [c["x"]])
    assert rocp.model_fitness(dev, T, [one * c["x_hat"], one, one]) == pytest.approx(c["fitness"], rel=1e-15)
    with pytest.raises(rocp.DomainError):
        rocp.model_fitness(dev, dev.tensor([3, 4]), [np.zeros((3, 1)), np.zeros((4, 1))])


# ---- E1 cprand ------------------------------------------------------------------------------------
def _cmp_init(a, b):
    assert a.iterations == b.iterations
    assert bitwise(np.float64(a.best_fitness), np.float64(b.best_fitness))
    assert a.regularized == b.regularized
    for n in range(len(a.model)):
        assert bitwise(a.model[n], b.model[n]), f"factor {n}"
    for n in range(len(a.best_sampled_kr)):
        assert bitwise(a.best_sampled_kr[n], b.best_sampled_kr[n]), f"Z_best {n}"
    assert bitwise(a.fit_trace, b.fit_trace)


@pytest.mark.parametrize("dims,R,snr,kw", [
    ([30, 30, 30], 5, None, {}),
    ([200, 200, 50], 10, 20.0, dict(tol=1e-6, max_iters=20)),       # configs[0] init slab
    ([40, 40, 40, 20], 10, 30.0, {}),                               # configs[2]-like, 4-way
    ([12, 12, 12, 12, 10], 16, 10.0, dict(max_iters=15)),          # configs[4]-like, 5-way
    ([6, 7, 8, 9], 2, None, dict(samples=13, max_iters=5)),
])
def test_cprand_bitwise(dev, dims, R, snr, kw):
    g = H.rng(sum(dims) + R)
    if len(dims) == 5:
        truth = H.congruent_factors(dims, R, 0.9, g)
        x, _ = H.gen_synthetic(dims, R, snr, g, factors=truth)
    else:
        x, _ = H.gen_synthetic(dims, R, snr, g)
    init = H.random_model(dims, R, H.rng(17))
    T = dev.tensor(dims, x)
    a = rocp.cprand_decompose(dev, T, R, init, seed=17, **kw)
    b = orc.cprand_decompose(x, dims, R, init, seed=17, **kw)
    _cmp_init(a, b)


def test_cprand_errors(dev):
    with pytest.raises(rocp.DomainError):
        rocp.cprand_decompose(dev, dev.tensor([3, 3]), 1, H.random_model([3, 3], 1, H.rng(1)), seed=1)
    x = np.zeros(27)
    x[0] = np.inf
    with pytest.raises(rocp.NumericalError) as e:
        rocp.cprand_decompose(dev, dev.tensor([3, 3, 3], x), 2, H.random_model([3, 3, 3], 2, H.rng(1)), seed=1)
    assert e.value.sweep == 1
    with pytest.raises(rocp.DomainError):
        rocp.cprand_decompose(dev, dev.tensor([3, 3, 3], np.ones(27)), 2,
                              H.random_model([3, 3, 3], 2, H.rng(1)), seed=1, max_iters=0)


# ---- E3 online stream -----------------------------------------------------------------------------
def _run_pair(dev, dims, R, snr, t_init, B, seed=29, congruence=None, kw=None, nbatches=None,
              literal=False):
    g = H.rng(sum(dims) * 3 + R)
    if congruence:
        x, _ = H.gen_synthetic(dims, R, snr, g, factors=H.congruent_factors(dims, R, congruence, g))
    else:
        x, _ = H.gen_synthetic(dims, R, snr, g)
    head = dims[:-1]
    idims = head + [t_init]
    xi = H.slab(x, dims, 0, t_init)
    init0 = H.random_model(idims, R, H.rng(seed))
    kw = kw or {}
    a_init = rocp.cprand_decompose(dev, dev.tensor(idims, xi), R, init0, seed=seed, **kw)
    b_init = orc.cprand_decompose(xi, idims, R, init0, seed=seed, **kw)
    _cmp_init(a_init, b_init)
    s = a_init.samples
    a = rocp.RocpStream(dev, a_init, s, literal_init=literal, t_capacity=dims[-1])
    b = orc.Stream(b_init.model, t_init, b_init.best_sampled_kr, s, literal_init=literal,
                   regularized=b_init.regularized)
    X = dev.tensor(dims, x)
    nb = (dims[-1] - t_init) // B if nbatches is None else nbatches
    return x, X, a, b, s, nb


def _cmp_stream(a, b, order):
    for n in range(1, order):
        assert bitwise(a.factor(n), b.factor(n)), f"U{n}"
        assert bitwise(a.p(n), b.p(n)), f"P{n}"
        assert bitwise(a.q(n), b.q(n)), f"Q{n}"
    assert bitwise(a.temporal(), b.temporal())
    assert a.t_len == b.t_len
    assert a.regularized == b.regularized


@pytest.mark.parametrize("name,dims,R,snr,t_init,B,cong,kw,nbat", [
    ("c1", [200, 200, 500], 10, 20.0, 50, 10, None, dict(tol=1e-6, max_iters=20), 12),
    ("c3-like", [40, 40, 40, 60], 10, 30.0, 20, 10, None, {}, None),
    ("c5-like", [12, 12, 12, 12, 60], 16, 10.0, 10, 10, 0.9, dict(max_iters=15), None),
    ("2-way", [50, 120], 4, 20.0, 30, 7, None, {}, 12),
    ("batch1", [20, 20, 80], 5, None, 16, 1, None, {}, 30),
])
def test_stream_consume_bitwise(dev, name, dims, R, snr, t_init, B, cong, kw, nbat):
    x, X, a, b, s, nb = _run_pair(dev, dims, R, snr, t_init, B, congruence=cong, kw=kw, nbatches=nbat)
    seed = 4242
    for k in range(nb):
        t0 = t_init + k * B
        a.consume(X.slab(t0, B), seed, k + 1)
        b.consume(H.slab(x, dims, t0, B), B, seed, k + 1)
        if k < 2 or k == nb - 1:
            _cmp_stream(a, b, len(dims))
            ra = a.last_residuals()
            rb = np.zeros(len(dims))
            import ctypes as C
            orc.lib().orc_stream_last_residuals(b._h, rb.ctypes.data_as(C.POINTER(C.c_double)))
            assert bitwise(ra, rb)
    _cmp_stream(a, b, len(dims))


def test_stream_host_slab_and_range_graph(dev):
    dims, R, t_init, B = [60, 50, 130], 6, 30, 10
    x, X, a, b, s, nb = _run_pair(dev, dims, R, 20.0, t_init, B)
    a.checkpoint()
    # (1) host slabs through the reference-facing call
    for k in range(nb):
        a.consume(H.slab(x, dims, t_init + k * B, B), 77, k + 1)
        b.consume(H.slab(x, dims, t_init + k * B, B), B, 77, k + 1)
    _cmp_stream(a, b, 3)
    ref = [a.factor(1), a.factor(2), a.temporal()]
    # (2) restore + the whole range as one persistent-kernel window, twice (replay)
    for _ in range(2):
        a.restore()
        a.consume_range(X, t_init, B, nb, 77, 1)
        assert bitwise(a.factor(1), ref[0]) and bitwise(a.factor(2), ref[1])
        assert bitwise(a.temporal(), ref[2])
    # (3) restore + the whole range from HOST slabs (host gather of sampled fibres only)
    for threads in (1, 0):
        a.restore()
        a.consume_range_host(H.slab(x, dims, t_init, B * nb), B, nb, 77, 1, threads=threads)
        assert bitwise(a.factor(1), ref[0]) and bitwise(a.factor(2), ref[1])
        assert bitwise(a.temporal(), ref[2])
    # (4) the same range in a registered huge-page buffer (rocp_host_alloc): the GPU reads
    # the mode-1 fibres in place, host threads gather the strided stages
    slab = H.slab(x, dims, t_init, B * nb)
    hb = rocp.HostBuffer(slab.size)
    hb.array[:] = slab
    for _ in range(2):
        a.restore()
        a.consume_range_host(hb.array, B, nb, 77, 1)
        assert bitwise(a.factor(1), ref[0]) and bitwise(a.factor(2), ref[1])
        assert bitwise(a.temporal(), ref[2])
    hb.free()


def test_stream_replay_seams_and_pins(dev):
    head, dims = [5, 6], [5, 6, 10]
    truth = H.random_model(dims, 2, H.rng(331))
    init = H.init_from_model(truth, dims, 16, seed=337)
    init.samples = 16
    a = rocp.RocpStream(dev, init, 16, t_capacity=64)
    b = orc.Stream(init.model, 10, init.best_sampled_kr, 16)
    g = H.rng(347)
    for k in range(4):
        slab, _ = H.planted_slab(truth, head, 2, g)
        S = dev.tensor(head + [2], slab)
        rows, _ = orc.draw_samples(head + [2], 3, 16, 347, k + 1, 0)
        ua, za, ra = a.update_last_mode_with(S, rows)
        ub, zb, rb = b.update_last_mode_with(slab, 2, rows)
        assert bitwise(ua, ub) and bitwise(za, zb) and ra == rb
        a.append_temporal(ua)
        b.append_temporal(ub)
        for n in (1, 2):
            r, _ = orc.draw_samples(head + [2], n, 16, 347, k + 1, 0)
            z1, x1, f1 = a.update_mode_with(S, ua, n, r)
            z2, x2, f2 = b.update_mode_with(slab, 2, ub, n, r)
            assert bitwise(z1, z2) and bitwise(x1, x2) and f1 == f2
        a.finish_batch(2)
        b.finish_batch(2)
    _cmp_stream(a, b, 3)
    # zero batch -> zero temporal rows (test_rocp.cpp:127-133)
    rows, _ = orc.draw_samples(head + [2], 3, 16, 1, 99, 0)
    u, _, _ = a.update_last_mode_with(dev.tensor(head + [2]), rows)
    assert (u == 0).all()
    with pytest.raises(rocp.DomainError):  # head mismatch (test_rocp.cpp:152-156)
        a.consume(dev.tensor([5, 7, 1]), 1, 1)
    with pytest.raises(rocp.DomainError):
        a.update_mode_with(S, ua, 3, r)
    # literal init keeps P = U (test_rocp.cpp:100-110)
    lit = rocp.RocpStream(dev, init, 16, literal_init=True, t_capacity=20)
    assert bitwise(lit.p(1), init.model[0]) and bitwise(lit.p(2), init.model[1])
    with pytest.raises(rocp.DomainError):
        rocp.RocpStream(dev, init, 17, t_capacity=20)


def test_stream_state_properties(dev):
    dims, head = [7, 6, 200], [7, 6]
    truth = H.random_model(dims, 2, H.rng(353))
    init = H.init_from_model(truth, dims[:2] + [12], 14, seed=359)
    init.model[-1] = H.random_matrix(12, 2, H.rng(1))
    init.samples = 14
    a = rocp.RocpStream(dev, init, 14, t_capacity=12 + 2 * 90)
    g = H.rng(361)
    before = a.temporal()
    for k in range(90):
        slab, _ = H.planted_slab(truth, head, 2, g)
        a.consume(slab, 361, k + 1)
        if k % 10 == 0:
            now = a.temporal()
            assert np.array_equal(now[: before.shape[0]], before)
            before = now
    assert a.t_len == 12 + 180
    for n in (1, 2):
        q = a.q(n)
        scale = np.abs(q).max()
        assert np.abs(q - q.T).max() <= TOL["q_symmetric"] * scale
        assert np.linalg.eigvalsh(q).min() >= -TOL["q_psd"] * scale


# ---- mode-1 sharded stream, one rank of world 1 -------------------------------
@pytest.mark.parametrize("dims,R,t_init,B,V", [([24, 10, 60], 4, 20, 8, 8), ([16, 6, 5, 30], 3, 10, 5, 4),
                                               ([40, 30, 50], 6, 20, 10, 1), ([200, 200, 120], 10, 50, 10, 8)])
def test_sharded_stream_bitwise(dev, dims, R, t_init, B, V):
    x, X, a, b, s, nb = _run_pair(dev, dims, R, 20.0, t_init, B)
    unsharded = None
    if V == 1:
        x2, X2, unsharded, _, _, _ = _run_pair(dev, dims, R, 20.0, t_init, B)
    r0, r1 = a.shard(V)
    assert (r0, r1) == (0, dims[0])
    XL = X.rows(r0, r1)
    for k in range(nb):
        t0 = t_init + k * B
        if k % 2 == 0:
            a.consume(XL.slab(t0, B), 515, k + 1)
        else:
            a.consume_range(XL, t0, B, 1, 515, k + 1)
        b.consume_sharded(H.slab(x, dims, t0, B), B, 515, k + 1, V)
        if unsharded is not None:
            unsharded.consume(X.slab(t0, B), 515, k + 1)
        if k < 2 or k == nb - 1:
            _cmp_stream(a, b, len(dims))
            assert bitwise(a.last_residuals(), b.last_residuals())
    if unsharded is not None:  # V = 1: the unsharded stream
        for n in range(1, len(dims)):
            assert bitwise(a.factor(n), unsharded.factor(n))
        assert bitwise(a.temporal(), unsharded.temporal())


def test_sharded_stream_window_and_errors(dev):
    dims, R, t_init, B = [32, 12, 90], 5, 30, 10
    x, X, a, b, s, nb = _run_pair(dev, dims, R, 20.0, t_init, B)
    a.shard(8)
    with pytest.raises(rocp.DomainError):
        a.shard(8)
    XL = X.rows(0, dims[0])
    a.consume_range(XL, t_init, B, nb, 616, 1)  # one window of every batch
    for k in range(nb):
        b.consume_sharded(H.slab(x, dims, t_init + k * B, B), B, 616, k + 1, 8)
    _cmp_stream(a, b, 3)
    with pytest.raises(rocp.DomainError):
        a.consume_range_host(H.slab(x, dims, t_init, B), B, 1, 1, 1)
    with pytest.raises(rocp.DomainError):
        a.set_residual_tracking(2)
        a.consume(XL.slab(t_init, B), 1, 1)
    a.set_residual_tracking(1)
    c = rocp.RocpStream(dev, rocp.InitResult([np.asfortranarray(m) for m in H.random_model([6, 5, 4], 2, H.rng(2))],
                                             [np.zeros((8, 2), order="F")] * 2, 0.0, 0, False, [], 8), 8)
    with pytest.raises(rocp.DomainError):
        c.shard(7)  # more shards than rows


def test_exhaustive_sampling_equals_full_update_on_device(dev):
    """SURVEY 8f-1 / acceptance.cpp:128-170 on the GPU: sampling every column once
    through the replay seams equals the exact online update (baselines.cpp:161-195)
    within the reference tolerance."""
    dims, R, t_init = [5, 6, 30], 2, 12
    g = H.rng(3001)
    x, _ = H.gen_synthetic(dims, R, 20.0, g)
    xi = H.slab(x, dims, 0, t_init)
    model = orc.cprand_decompose(xi, [5, 6, t_init], R, H.random_model([5, 6, t_init], R, H.rng(3002)),
                                 seed=3002, tol=1e-10, max_iters=60).model
    p, q = orc.online_full_init(xi, [5, 6, t_init], model)
    batch = H.slab(x, dims, t_init, 2)
    bd = [5, 6, 2]
    fh = [np.array(m, order="F", copy=True) for m in model[:-1]]
    pf = [np.array(m, order="F", copy=True) for m in p]
    qf = [np.array(m, order="F", copy=True) for m in q]
    u_full = orc.online_full_update(batch, bd, fh, pf, qf)

    def stream_with(s):
        init = rocp.InitResult([np.asfortranarray(m) for m in model], [np.zeros((s, R), order="F")] * 2,
                               0.0, 0, False, [], s)
        st = rocp.RocpStream(dev, init, s, literal_init=True, t_capacity=64)
        for n in (1, 2):
            st.set(1, n, p[n - 1])
            st.set(2, n, q[n - 1])
        return st

    Xb = dev.tensor(bd, batch)
    st = stream_with(30)
    u, _, _ = st.update_last_mode_with(Xb, np.arange(1, 31))
    worst = np.linalg.norm(u - u_full) / np.linalg.norm(u_full)
    state_u = [model[0], model[1]]
    state_p, state_q = list(p), list(q)
    for n in (1, 2):
        co = orc.codomain_size(bd, n)
        sn = stream_with(co)
        for k in (1, 2):
            sn.set(0, k, state_u[k - 1])
            sn.set(1, k, state_p[k - 1])
            sn.set(2, k, state_q[k - 1])
        sn.update_mode_with(Xb, u, n, np.arange(1, co + 1))
        state_u[n - 1], state_p[n - 1], state_q[n - 1] = sn.factor(n), sn.p(n), sn.q(n)
        worst = max(worst, np.linalg.norm(state_p[n - 1] - pf[n - 1]) / np.linalg.norm(pf[n - 1]))
        worst = max(worst, np.linalg.norm(state_q[n - 1] - qf[n - 1]) / np.linalg.norm(qf[n - 1]))
        worst = max(worst, np.linalg.norm(state_u[n - 1] - fh[n - 1]) / np.linalg.norm(fh[n - 1]))
    assert worst <= TOL["exhaustive_equivalence"], worst


# ---- emulated multi-rank groups: the sharded product path at world 2 / 4 / 8 on one GPU ---------------
@pytest.mark.parametrize("dims,R,t_init,B,V,world", [([24, 10, 60], 4, 20, 8, 8, 2), ([24, 10, 60], 4, 20, 8, 8, 4),
                                                     ([16, 6, 5, 30], 3, 10, 5, 4, 2), ([64, 20, 70], 6, 20, 10, 8, 8),
                                                     ([9, 4, 4, 3, 20], 2, 8, 4, 4, 4), ([200, 200, 120], 10, 50, 10, 8, 8)])
def test_emulated_group_equals_oracle_sharded(dev, dims, R, t_init, B, V, world):
    """World-size runs of the product's sharded path with `world` emulated ranks on this GPU
    (rocp_create_emulated_rank + rocp_emulated_group_consume_range): k_shard_partition,
    k_seg_partials storing into every rank's landing slots and releasing every rank's counter,
    k_shard_combine / k_shard_resid_sum acquiring them, parity double-buffering across stages and
    windows.  Every rank's local U(1)/P(1) rows, the replicated factors, P, Q, the temporal factor,
    the flag and the residuals equal orc_stream_consume_sharded bit for bit."""
    g = H.rng(sum(dims) + world)
    x, _ = H.gen_synthetic(dims, R, 20.0, g)
    head = dims[:-1]
    s = orc.auto_sample_count(R)
    init = H.init_from_model(H.random_model(head + [t_init], R, H.rng(3)), head + [t_init], s, 5)
    X = dev.tensor(dims, x)
    b = orc.Stream(init.model, t_init, init.best_sampled_kr, s)
    devs = [rocp.Device(0, world, r, emulated=True) for r in range(world)]
    try:
        sts, xls, rows = [], [], []
        for r in range(world):
            st = rocp.RocpStream(devs[r], init, s, t_capacity=dims[-1])
            r0, r1 = st.shard(V)
            rows.append((r0, r1))
            sts.append(st)
            xls.append(X.rows(r0, r1))
        assert rows[0][0] == 0 and rows[-1][1] == dims[0]
        nb = (dims[-1] - t_init) // B
        windows = [1, nb - 1] if nb > 1 else [1]
        t0, bid = t_init, 1
        for w in windows:
            rocp.emulated_group_consume_range(sts, xls, t0, B, w, 616, bid)
            for k in range(w):
                b.consume_sharded(H.slab(x, dims, t0 + k * B, B), B, 616, bid + k, V)
            t0, bid = t0 + w * B, bid + w
            for r, st in enumerate(sts):
                r0, r1 = rows[r]
                assert bitwise(st.factor(1), b.factor(1)[r0:r1]), f"rank {r} U1 rows"
                assert bitwise(st.p(1), b.p(1)[r0:r1]), f"rank {r} P1 rows"
                assert bitwise(st.q(1), b.q(1)), f"rank {r} Q1"
                for n in range(2, len(dims)):
                    assert bitwise(st.factor(n), b.factor(n)), f"rank {r} U{n}"
                    assert bitwise(st.p(n), b.p(n)), f"rank {r} P{n}"
                    assert bitwise(st.q(n), b.q(n)), f"rank {r} Q{n}"
                assert bitwise(st.temporal(), b.temporal()), f"rank {r} temporal"
                assert st.t_len == b.t_len and st.regularized == b.regularized
                assert bitwise(st.last_residuals(), b.last_residuals()), f"rank {r} residuals"
        with pytest.raises(rocp.DomainError):  # a sharded member of the wrong world is rejected
            rocp.emulated_group_consume_range(sts[:1], xls[:1], t_init, B, 1, 1, 1)
    finally:
        for d in devs:
            d.close()
