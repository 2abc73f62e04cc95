"""CPU oracle pinned against the reference's own known-answer vectors and
properties (tests/golden/*.json; reference tests cited per case).

These run without a GPU.  They establish that oracle/ restates the reference
 before it is trusted as the checker of the CUDA path.
"""
import json
import os

import numpy as np
import pytest

from oracle import oracle as orc
from tests import helpers as H

GOLD = os.path.join(os.path.dirname(__file__), "golden")
KAT = json.load(open(os.path.join(GOLD, "reference_kat.json")))
TOL = {k: v[0] for k, v in KAT["tolerances"].items()}


# ---- counter RNG -------------------------------------------------------------
def test_philox_published_kat():
    kat = json.load(open(os.path.join(GOLD, "philox_kat.json")))
    for v in kat["vectors"]:
        out = orc.philox4x32_10([int(x, 16) for x in v["ctr"]], [int(x, 16) for x in v["key"]])
        assert out == [int(x, 16) for x in v["out"]]


# ---- index map (test_tensor.cpp) --------------------------------------------
def test_linear_index_kat():
    for c in KAT["linear_index"]:
        assert orc.linear_index(c["multi"], c["dims"], c["mode"]) == c["j"], c["src"]
    for c in KAT["linear_index_rejects"]:
        with pytest.raises(orc.DomainError):
            orc.linear_index(c["multi"], c["dims"], c["mode"])


def test_decode_index_kat():
    for c in KAT["decode_index"]:
        assert orc.decode_index(c["j"], c["dims"], c["mode"]) == c["multi"], c["src"]
    for c in KAT["decode_index_rejects"]:
        with pytest.raises(orc.DomainError):
            orc.decode_index(c["j"], c["dims"], c["mode"])


def enumerate_columns(dims, mode):
    """Nested-loop enumeration, lowest co-mode fastest (tests/oracles.hpp:22-39)."""
    ext = [d for k, d in enumerate(dims) if k + 1 != mode]
    out, ctr = [], [1] * len(ext)
    while True:
        out.append(list(ctr))
        k = 0
        while k < len(ext):
            ctr[k] += 1
            if ctr[k] <= ext[k]:
                break
            ctr[k] = 1
            k += 1
        if k == len(ext):
            return out


@pytest.mark.parametrize("dims", [[3, 4, 5], [2, 2], [2, 3, 4]])
def test_bijection_exhaustive(dims):  # test_tensor.cpp:84-99
    for mode in range(1, len(dims) + 1):
        cols = enumerate_columns(dims, mode)
        for p, multi in enumerate(cols):
            j = orc.linear_index(multi, dims, mode)
            assert j == p + 1
            assert orc.decode_index(j, dims, mode) == multi


def test_auto_sample_count_kat():
    for c in KAT["auto_sample_count"]:
        assert orc.auto_sample_count(c["rank"]) == c["s"], c["src"]


# ---- draws (test_factor_model.cpp:95-137) ------------------------------------
def test_draw_codomain_one():
    c = KAT["draw_codomain_one"]
    rows, _ = orc.draw_samples(c["dims"], c["mode"], c["s"], 1, 0, 0)
    assert rows.tolist() == c["rows"]


def test_draw_deterministic_and_fresh():
    a, da = orc.draw_samples([4, 5, 6], 2, 50, 99, 3, 7)
    b, db = orc.draw_samples([4, 5, 6], 2, 50, 99, 3, 7)
    assert (a == b).all() and (da == db).all()
    for key in [(100, 3, 7), (99, 4, 7), (99, 3, 8)]:  # seed / batch / iteration all matter
        c, _ = orc.draw_samples([4, 5, 6], 2, 50, *key)
        assert not (c == a).all()


def test_draw_uniform_five_sigma():  # test_factor_model.cpp:109-119
    s = 10000
    rows, _ = orc.draw_samples([2, 10], 1, s, 4242, 0, 0)
    freq = np.bincount(rows - 1, minlength=10)
    sigma = np.sqrt(s * 0.1 * 0.9)
    assert np.all(np.abs(freq - s / 10) <= 5 * sigma)


def test_draw_decoded_consistent():  # test_factor_model.cpp:124-133
    dims = [3, 4, 5]
    rows, dec = orc.draw_samples(dims, 2, 25, 7, 0, 0)
    for c in range(25):
        assert orc.decode_index(int(rows[c]), dims, 2) == dec[c].tolist()


def test_draw_rejects_nonpositive_s():
    with pytest.raises(orc.DomainError):
        orc.draw_samples([2, 2], 1, 0, 1, 0, 0)


# ---- gather (test_factor_model.cpp:141-168) ----------------------------------
def test_unfold_kat():
    c = KAT["unfold_mode1_2x2"]
    dec = orc.from_rows(c["dims"], 1, [1, 2])
    m = orc.sample_unfolding(np.array(c["data"], float), c["dims"], 1, dec)
    assert m.tolist() == c["matrix_rowwise"]


def unfold(t, dims, mode):
    co = orc.codomain_size(dims, mode)
    return orc.sample_unfolding(t, dims, mode, orc.from_rows(dims, mode, np.arange(1, co + 1)))


def test_gather_all_columns_is_unfold():
    g = H.rng(55)
    dims = [3, 4, 5]
    t = g.standard_normal(60)
    T = t.reshape(dims[::-1]).transpose()  # T[i1,i2,i3]
    for mode in (1, 2, 3):
        m = unfold(t, dims, mode)
        cols = enumerate_columns(dims, mode)
        for p, multi in enumerate(cols):
            for i in range(dims[mode - 1]):
                full = list(multi)
                full.insert(mode - 1, i + 1)
                assert m[i, p] == T[tuple(x - 1 for x in full)]


def test_gather_single_and_duplicate():
    g = H.rng(55)
    dims = [3, 4, 5]
    t = g.standard_normal(60)
    col = orc.sample_unfolding(t, dims, 2, orc.from_rows(dims, 2, [7]))
    assert (col[:, 0] == unfold(t, dims, 2)[:, 6]).all()
    cols = orc.sample_unfolding(t, dims, 1, orc.from_rows(dims, 1, [4, 4]))
    assert (cols[:, 0] == cols[:, 1]).all()


def test_from_rows_rejects_out_of_range():
    with pytest.raises(orc.DomainError):
        orc.from_rows([3, 4, 6], 1, [25])


# ---- Khatri-Rao (test_tensor.cpp:176-209, test_factor_model.cpp:172-218) -----
def test_khatri_rao_kat():
    c = KAT["khatri_rao_2x2"]
    out = orc.khatri_rao(np.array(c["a_rowwise"], float), np.array(c["b_rowwise"], float))
    assert out.tolist() == c["out_rowwise"]


@pytest.mark.parametrize("dims", [[3, 3], [2, 3, 4], [3, 3, 3, 3], [3, 4, 5], [2, 3, 4, 5]])
@pytest.mark.parametrize("rank", [1, 3, 4])
def test_skr_exhaustive_equals_full_kr_bitwise(dims, rank):
    model = H.random_model(dims, rank, H.rng(73))
    for mode in range(1, len(dims) + 1):
        fs = orc.factors_excluding(model, mode)
        full = orc.khatri_rao_list(fs)
        co = orc.codomain_size(dims, mode)
        z = orc.sampled_khatri_rao(orc.from_rows(dims, mode, np.arange(1, co + 1)), fs)
        assert np.array_equal(z, full)


def test_skr_rejects_index_beyond_rows():
    model = H.random_model([2, 3], 2, H.rng(79))
    dec = orc.from_rows([5, 3], 2, [4])
    with pytest.raises(orc.DomainError):
        orc.sampled_khatri_rao(dec, orc.factors_excluding(model, 2))


# ---- fitness (test_factor_model.cpp:73-93) -----------------------------------
def test_fitness_kat():
    c = KAT["fitness_single_entry"]
    one = np.ones((1, 1))
    fit = orc.model_fitness(np.array([c["x"]]), [1, 1, 1], [one * c["x_hat"], one, one])
    assert fit == pytest.approx(c["fitness"], rel=1e-15)


def test_frobenius_kat():
    for c in KAT["frobenius_norm"]:
        data = np.zeros(int(np.prod(c["dims"]))) if c["data"] == "zeros" else np.array(c["data"], float)
        zero = [np.zeros((d, 1)) for d in c["dims"]]
        if "value" in c and c["value"] == 0.0:
            with pytest.raises(orc.DomainError):  # zero-norm reference rejected (kruskal.cpp:75-76)
                orc.model_fitness(data, c["dims"], zero)
            continue
        # fitness against the zero model = 1 - |x|/|x| = 0 exercises |x|
        assert orc.model_fitness(data, c["dims"], zero) == 0.0


def test_fitness_matches_reconstruction():
    g = H.rng(23)
    dims = [3, 4, 5]
    model = H.random_model(dims, 2, g)
    x = H.reconstruct(model, dims) + 0.1 * g.standard_normal(60)
    fit = orc.model_fitness(x, dims, model)
    xh = H.reconstruct(model, dims)
    assert fit == pytest.approx(1 - np.linalg.norm(xh - x) / np.linalg.norm(x), rel=1e-12)
    assert orc.model_fitness(xh, dims, model) == 1.0


# ---- solve (test_cprand.cpp:25-81) --------------------------------------------
def test_sampled_ls_identity():
    g = H.rng(101)
    x = H.random_matrix(5, 3, g)
    u, reg, und = orc.solve_sampled_ls(np.eye(3), x)
    assert np.abs(u - x).max() < TOL["sampled_ls_identity"]


def test_sampled_ls_orthonormal():
    g = H.rng(102)
    z, _ = np.linalg.qr(g.standard_normal((20, 3)))
    x = H.random_matrix(6, 20, g)
    u, _, _ = orc.solve_sampled_ls(z, x)
    assert np.abs(u - x @ z).max() < TOL["sampled_ls_orthonormal"]


def test_sampled_ls_planted_and_residual():
    g = H.rng(103)
    u0 = H.random_matrix(6, 3, g)
    z = H.random_matrix(20, 3, g)
    u, _, _ = orc.solve_sampled_ls(z, u0 @ z.T)
    assert np.linalg.norm(u - u0) <= TOL["sampled_ls_planted"] * np.linalg.norm(u0)
    z = H.random_matrix(25, 4, g)
    x = H.random_matrix(7, 25, g)
    u, _, _ = orc.solve_sampled_ls(z, x)
    uref = np.linalg.lstsq(z, x.T, rcond=None)[0].T
    res = lambda uu: np.linalg.norm(z @ uu.T - x.T)
    assert res(u) <= res(uref) + TOL["sampled_ls_vs_svd_residual"]


def test_sampled_ls_flags():
    g = H.rng(104)
    u, reg, und = orc.solve_sampled_ls(H.random_matrix(2, 4, g), H.random_matrix(3, 2, g))
    assert und and reg and np.isfinite(u).all()
    u, reg, _ = orc.solve_sampled_ls(np.zeros((5, 2)), H.random_matrix(3, 5, g))
    assert reg and (u == 0).all()
    with pytest.raises(orc.DomainError):
        orc.solve_sampled_ls(np.zeros((5, 2)), np.zeros((3, 4)))


# ---- cprand (test_cprand.cpp:83-198) -------------------------------------------
def test_cprand_rank1_recovery():
    g = H.rng(7)
    truth = [np.abs(g.standard_normal((d, 1))) + 0.1 for d in (5, 6, 7)]
    x = H.reconstruct(truth, [5, 6, 7])
    res = orc.cprand_decompose(x, [5, 6, 7], 1, H.random_model([5, 6, 7], 1, H.rng(11)), seed=11)
    assert res.best_fitness >= TOL["cprand_rank1_fit"]
    assert orc.model_fitness(x, [5, 6, 7], res.model) == res.best_fitness


def test_cprand_rank5_recovery():
    dims = [30, 30, 30]
    x = H.reconstruct(H.random_model(dims, 5, H.rng(13)), dims)
    res = orc.cprand_decompose(x, dims, 5, H.random_model(dims, 5, H.rng(17)), seed=17)
    assert res.best_fitness >= TOL["cprand_rank5_fit"]


def test_cprand_same_seed_bitwise_and_shapes():
    dims = [6, 7, 8, 9]
    x = H.reconstruct(H.random_model(dims, 2, H.rng(29)), dims)
    init = H.random_model(dims, 2, H.rng(31))
    a = orc.cprand_decompose(x, dims, 2, init, seed=31, samples=13, max_iters=5)
    b = orc.cprand_decompose(x, dims, 2, init, seed=31, samples=13, max_iters=5)
    assert a.best_fitness == b.best_fitness and a.iterations == b.iterations
    for n in range(4):
        assert np.array_equal(a.model[n], b.model[n])
        assert a.model[n].shape == (dims[n], 2)
    assert len(a.best_sampled_kr) == 3
    for z in a.best_sampled_kr:
        assert z.shape == (13, 2)


def test_cprand_best_fitness_monotone_in_budget():
    dims = [10, 10, 10]
    x = H.reconstruct(H.random_model(dims, 4, H.rng(37)), dims)
    init = H.random_model(dims, 4, H.rng(41))
    prev = -1.0
    for iters in (1, 2, 3, 5, 8):
        r = orc.cprand_decompose(x, dims, 4, init, seed=41, max_iters=iters, tol=0.0)
        assert r.best_fitness >= prev
        prev = r.best_fitness


def test_cprand_errors():
    with pytest.raises(orc.DomainError):
        orc.cprand_decompose(np.zeros(9), [3, 3], 1, H.random_model([3, 3], 1, H.rng(1)), seed=1)
    x = np.zeros(27)
    x[0] = np.inf
    with pytest.raises(orc.NumericalError) as e:
        orc.cprand_decompose(x, [3, 3, 3], 2, H.random_model([3, 3, 3], 2, H.rng(1)), seed=1)
    assert e.value.sweep == 1


# ---- online state (test_rocp.cpp) -------------------------------------------------
def test_init_state_properties():
    g = H.rng(301)
    dims = [6, 7, 9]
    model = H.random_model(dims, 3, H.rng(303))
    init = H.init_from_model(model, dims, 20, seed=5)
    st = orc.Stream(init.model, dims[-1], init.best_sampled_kr, 20)
    for n in (1, 2):
        u = np.linalg.solve(st.q(n), st.p(n).T).T
        assert np.linalg.norm(u - model[n - 1]) <= TOL["init_state_pq_inverse"] * np.linalg.norm(model[n - 1])
    assert st.t_len == 9
    lit = orc.Stream(init.model, dims[-1], init.best_sampled_kr, 20, literal_init=True)
    assert np.array_equal(lit.p(1), model[0]) and np.array_equal(lit.p(2), model[1])
    with pytest.raises(orc.DomainError):
        orc.Stream(init.model, dims[-1], init.best_sampled_kr, 21)


def test_init_state_orthonormal():
    g = H.rng(302)
    model = [H.random_matrix(4, 2, g), H.random_matrix(3, 2, g), H.random_matrix(5, 2, g)]
    kr = [np.linalg.qr(g.standard_normal((12, 2)))[0] for _ in range(2)]
    st = orc.Stream(model, 5, kr, 12)
    for n in (1, 2):
        assert np.abs(st.q(n) - np.eye(2)).max() < TOL["init_state_orthonormal"]
        assert np.abs(st.p(n) - model[n - 1]).max() < TOL["init_state_orthonormal"]


def _stream_for(truth, dims, s, seed=337):
    init = H.init_from_model(truth, dims, s, seed)
    return orc.Stream(init.model, dims[-1], init.best_sampled_kr, s), init


def test_temporal_update_zero_and_planted():
    head, dims = [5, 6], [5, 6, 8]
    truth = H.random_model(dims, 3, H.rng(311))
    st, _ = _stream_for(truth, dims, 15)
    rows, _ = orc.draw_samples(head + [2], 3, 15, 313, 1, 0)
    u, z, reg = st.update_last_mode_with(np.zeros(60), 2, rows)
    assert (u == 0).all() and z.shape == (15, 3)
    slab, planted = H.planted_slab(truth, head, 4, H.rng(317))
    st2, _ = _stream_for(truth, dims, 20)
    rows, _ = orc.draw_samples(head + [4], 3, 20, 317, 1, 0)
    u, _, _ = st2.update_last_mode_with(slab, 4, rows)
    assert np.linalg.norm(u - planted) <= TOL["temporal_recovery"] * np.linalg.norm(planted)


def test_pq_recursion_matches_direct():
    dims, head = [5, 6, 10], [5, 6]
    truth = H.random_model(dims, 2, H.rng(331))
    st, _ = _stream_for(truth, dims, 16)
    p0 = [st.p(n) for n in (1, 2)]
    q0 = [st.q(n) for n in (1, 2)]
    g = H.rng(347)
    xs = {1: [], 2: []}
    zs = {1: [], 2: []}
    for k in range(5):
        slab, _ = H.planted_slab(truth, head, 1, g)
        rows, _ = orc.draw_samples(head + [1], 3, 16, 347, k + 1, 0)
        u, _, _ = st.update_last_mode_with(slab, 1, rows)
        st.append_temporal(u)
        for n in (1, 2):
            r, _ = orc.draw_samples(head + [1], n, 16, 347, k + 1, 0)
            z, x, _ = st.update_mode_with(slab, 1, u, n, r)
            xs[n].append(x)
            zs[n].append(z)
        st.finish_batch(1)
    for n in (1, 2):
        X = np.hstack(xs[n])
        Z = np.vstack(zs[n])
        pd = p0[n - 1] + X @ Z
        qd = q0[n - 1] + Z.T @ Z
        assert np.linalg.norm(st.p(n) - pd) <= TOL["pq_recursion_direct"] * np.linalg.norm(pd)
        assert np.linalg.norm(st.q(n) - qd) <= TOL["pq_recursion_direct"] * np.linalg.norm(qd)


def test_q_symmetric_psd_and_frozen_rows():
    dims, head = [7, 6, 12], [7, 6]
    truth = H.random_model(dims, 2, H.rng(353))
    st, init = _stream_for(truth, dims, 14)
    g = H.rng(349)
    before = st.temporal()
    for k in range(40):
        slab, _ = H.planted_slab(truth, head, 2, g)
        st.consume(slab, 2, seed=349, batch_id=k + 1)
        now = st.temporal()
        assert now.shape[0] == before.shape[0] + 2
        assert np.array_equal(now[: before.shape[0]], before)  # test_rocp.cpp:243-256
        before = now
    for n in (1, 2):
        q = st.q(n)
        scale = np.abs(q).max()
        assert np.abs(q - q.T).max() <= TOL["q_symmetric"] * scale
        assert np.linalg.eigvalsh(q).min() >= -TOL["q_psd"] * scale


def test_rocp_run_planted_stream():  # test_rocp.cpp:282-294
    dims = [20, 20, 200]
    g = H.rng(383)
    x, truth = H.gen_synthetic(dims, 5, None, g)
    t_init = 40
    xi = H.slab(x, dims, 0, t_init)
    init = orc.cprand_decompose(xi, [20, 20, t_init], 5, H.random_model([20, 20, t_init], 5, H.rng(389)),
                                seed=389)
    st = orc.Stream(init.model, t_init, init.best_sampled_kr, init.best_sampled_kr[0].shape[0])
    for b in range(160):
        st.consume(H.slab(x, dims, t_init + b, 1), 1, seed=389, batch_id=b + 1)
    model = st.model()
    assert model[-1].shape[0] == 200
    assert orc.model_fitness(x, dims, model) >= TOL["rocp_run_planted_fit"]


def test_exhaustive_sampling_equals_full_update():  # acceptance.cpp:128-170
    dims = [5, 6, 30]
    g = H.rng(3001)
    x, truth = H.gen_synthetic(dims, 2, 20.0, g)
    t_init = 12
    xi = H.slab(x, dims, 0, t_init)
    model = orc.cprand_decompose(xi, [5, 6, t_init], 2, H.random_model([5, 6, t_init], 2, H.rng(3002)),
                                 seed=3002, tol=1e-10, max_iters=60).model
    p, q = orc.online_full_init(xi, [5, 6, t_init], model)
    batch = H.slab(x, dims, t_init, 2)
    bd = [5, 6, 2]
    fh = [np.array(m, order="F", copy=True) for m in model[:-1]]
    pf = [np.array(m, order="F", copy=True) for m in p]
    qf = [np.array(m, order="F", copy=True) for m in q]
    u_full = orc.online_full_update(batch, bd, fh, pf, qf)
    # sampled path with every column, same starting state
    st = orc.Stream(model, t_init, [np.zeros((1, 2))] * 2, 1, literal_init=True)
    for n in (1, 2):
        st.set(1, n, p[n - 1])
        st.set(2, n, q[n - 1])
    u, _, _ = st.update_last_mode_with(batch, 2, np.arange(1, 31))
    st.append_temporal(u)
    worst = np.linalg.norm(u - u_full) / np.linalg.norm(u_full)
    for n in (1, 2):
        co = orc.codomain_size(bd, n)
        st.update_mode_with(batch, 2, u, n, np.arange(1, co + 1))
        worst = max(worst, np.linalg.norm(st.p(n) - pf[n - 1]) / np.linalg.norm(pf[n - 1]))
        worst = max(worst, np.linalg.norm(st.q(n) - qf[n - 1]) / np.linalg.norm(qf[n - 1]))
        worst = max(worst, np.linalg.norm(st.factor(n) - fh[n - 1]) / np.linalg.norm(fh[n - 1]))
    assert worst <= TOL["exhaustive_equivalence"]


def test_residual_definition():
    g = H.rng(9)
    x = H.random_matrix(7, 30, g)
    u = H.random_matrix(7, 3, g)
    z = H.random_matrix(30, 3, g)
    import ctypes as C
    out = C.c_double(0)
    L = orc.lib()
    xf, uf, zf = (np.asfortranarray(a) for a in (x, u, z))
    L.orc_sampled_residual(xf.ctypes.data_as(C.POINTER(C.c_double)), C.c_int64(7), C.c_int64(30),
                           uf.ctypes.data_as(C.POINTER(C.c_double)),
                           zf.ctypes.data_as(C.POINTER(C.c_double)), 3, C.byref(out))
    ref = np.linalg.norm(x - u @ z.T) / np.linalg.norm(x)
    assert out.value == pytest.approx(ref, rel=1e-12)
