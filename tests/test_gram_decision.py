"""solve_gram's regularisation decision (reference solve.cpp:17-33) near the
kGramConditionLimit = 1e12 threshold (solve.hpp:15).

The reference decides from exact eigenvalues (SelfAdjointEigenSolver): zero
solution when lambda_max <= 0, G + 1e-12 tr(G) I when lambda_min <= 0 or
lambda_max / lambda_min > 1e12.  The canonical form settles it
with a rigorous certificate (LDL^T pivots and tau = tr(G^-1)) and falls back to
deterministic Jacobi eigenvalues in the band around the threshold.  These tests
build Grams whose LDL^T pivot ratio is far BELOW their condition number (the
case a pivot-ratio rule gets wrong) and check:
  * CPU: the oracle's decision equals the eigenvalue rule (numpy eigvalsh as the
    stand-in for Eigen) at kappa = 1e11, 1e12 (1 -/+ 1e-3), 1e13, singular,
    zero and indefinite Grams;
  * GPU: k_solve (every primitive, cprand, sharded stages) and the persistent
    chain's narrow (R <= 32) and wide (R > 32) finishers make the same decision
    and produce the oracle's bits.
"""
import numpy as np
import pytest

import paper_2007_10798_b200 as rocp
from oracle import oracle as orc
from tests import helpers as H

LIMIT = 1e12  # solve.hpp:15


def reference_rule(G):
    """(mode, regularized) by solve.cpp:17-33 from exact eigenvalues."""
    ev = np.linalg.eigvalsh(G)
    lo, hi = ev.min(), ev.max()
    if hi <= 0.0:
        return 0, True
    return 1, bool(lo <= 0.0 or hi / lo > LIMIT)


def conditioned_gram(R, kappa, seed):
    """Q diag(lambda) Q^T with lambda geometric in [1/kappa, 1] and a random orthogonal Q."""
    g = np.random.default_rng(seed)
    lam = np.geomspace(1.0, 1.0 / kappa, R)
    q, _ = np.linalg.qr(g.standard_normal((R, R)))
    G = (q * lam) @ q.T
    return np.asfortranarray((G + G.T) / 2.0)


def pivot_ratio(G):
    d = np.diag(np.linalg.cholesky(G)) ** 2
    return d.max() / d.min()


KAPPAS = [1e11, LIMIT * (1 - 1e-3), LIMIT * (1 + 1e-3), 1e13]
SIZES = [2, 5, 8, 20, 40]


def hidden_pair(delta, R=2):
    """[[1, 1-delta], [1-delta, 1]] (+ identity padding): kappa = (2-delta)/delta, pivot ratio ~ kappa/4."""
    G = np.eye(R)
    G[0, 1] = G[1, 0] = 1.0 - delta
    return np.asfortranarray(G)


@pytest.mark.parametrize("R", SIZES)
@pytest.mark.parametrize("kappa", KAPPAS)
def test_oracle_decision_matches_eigenvalue_rule(R, kappa):
    G = conditioned_gram(R, kappa, seed=R * 7 + int(np.log10(kappa) * 10))
    assert pivot_ratio(G) < kappa  # the pivots hide part of the conditioning
    mode, reg, path, lo, hi = orc.gram_decision(G)
    assert (mode, reg) == reference_rule(G)
    assert np.isclose(hi / lo, np.linalg.cond(G), rtol=1e-3)


@pytest.mark.parametrize("delta,expect", [(2e-12 * 1.001, False), (2e-12 * 0.999, True), (1e-12, True),
                                          (2e-10, False)])
def test_oracle_hidden_pivot_pair(delta, expect):
    for R in (2, 6, 33):
        G = hidden_pair(delta, R)
        assert pivot_ratio(G) < LIMIT  # a pivot-ratio rule never regularises these
        mode, reg, path, _, _ = orc.gram_decision(G)
        assert (mode, reg) == (1, expect) == reference_rule(G)


def test_oracle_decision_special_grams():
    assert orc.gram_decision(np.zeros((4, 4), order="F"))[:2] == (0, True)  # hi <= 0: zero solution
    assert orc.gram_decision(np.eye(7, order="F"))[:3] == (1, False, 0)    # certified without eigenvalues
    sing = np.asfortranarray(np.outer([1.0, 2.0, 3.0], [1.0, 2.0, 3.0]))  # rank 1: lambda_min = 0
    assert orc.gram_decision(sing)[:2] == (1, True)
    indef = np.asfortranarray(np.array([[0.0, 1.0], [1.0, 0.0]]))        # max diag 0, lambda_max 1
    assert orc.gram_decision(indef)[:2] == (1, True) == reference_rule(indef)
    neg = np.asfortranarray(-np.eye(3))
    assert orc.gram_decision(neg)[:2] == (0, True) == reference_rule(neg)
    # the BASELINE configs' Grams (kappa ~ 10-1e4) are settled by the certificate
    g = H.rng(3)
    for R in (10, 16, 20, 50):
        z = H.random_matrix(int(np.ceil(10 * R * np.log(R))), R, g)
        assert orc.gram_decision(orc.gram(z))[2] == 0


# ---- GPU: the same decisions and bits on the device --------------------------------------------
@pytest.mark.gpu
@pytest.mark.parametrize("R", SIZES + [64])
def test_solve_gram_decision_on_device(dev, R):
    g = H.rng(900 + R)
    rhs = H.random_matrix(37, R, g)
    cases = [conditioned_gram(R, k, seed=R + i) for i, k in enumerate(KAPPAS)]
    cases += [hidden_pair(2e-12 * 1.001, R), hidden_pair(2e-12 * 0.999, R), np.zeros((R, R), order="F")]
    for G in cases:
        u_gpu, reg_gpu = rocp.solve_gram(dev, G, rhs)
        u_orc, reg_orc = orc.solve_gram(G, rhs)
        mode, reg, _, _, _ = orc.gram_decision(G)
        assert reg_gpu == reg_orc == reg
        assert (mode, reg) == reference_rule(G)
        assert np.array_equal(u_gpu.view(np.uint64), u_orc.view(np.uint64))


@pytest.mark.gpu
@pytest.mark.parametrize("R,kappa", [(8, LIMIT * (1 + 1e-3)), (8, LIMIT * (1 - 1e-3)), (20, 1e13),
                                     (40, LIMIT * (1 + 1e-3)), (40, LIMIT * (1 - 1e-3))])
def test_chain_decision_near_threshold(dev, R, kappa):
    """The persistent chain's finisher (narrow R <= 32, wide R > 32) on a mode-1 Q(1) whose
    accumulated Gram sits at the threshold: Q(1) is replaced by c * G_kappa with c large
    enough that one batch's Z^T Z moves the spectrum by < 1e-6 relative, and P(1) = U(1) Q(1)."""
    dims, t_init, B = [24, 20, 40], 10, 5
    g = H.rng(R)
    x, _ = H.gen_synthetic(dims, R, 20.0, g)
    model = H.random_model(dims[:-1] + [t_init], R, H.rng(R + 1))
    s = orc.auto_sample_count(R)
    init = H.init_from_model(model, dims[:-1] + [t_init], s, 5)
    a = rocp.RocpStream(dev, init, s, t_capacity=dims[-1])
    b = orc.Stream(init.model, t_init, init.best_sampled_kr, s)
    Gk = np.asfortranarray(conditioned_gram(R, kappa, seed=R) * 1e24)
    Pk = np.asfortranarray(b.factor(1) @ Gk)  # keeps U(1) = P Q^-1 near its init value
    for st in (a, b):
        st.set(2, 1, Gk)
        st.set(1, 1, Pk)
    X = dev.tensor(dims, x)
    for k in range(2):
        t0 = t_init + k * B
        a.consume(X.slab(t0, B), 31, k + 1)
        b.consume(H.slab(x, dims, t0, B), B, 31, k + 1)
    for n in (1, 2):
        assert np.array_equal(a.factor(n).view(np.uint64), b.factor(n).view(np.uint64)), f"U{n}"
        assert np.array_equal(a.q(n).view(np.uint64), b.q(n).view(np.uint64)), f"Q{n}"
    # the accumulated Q(1) still straddles the threshold the same way
    assert reference_rule(b.q(1))[1] == reference_rule(Gk)[1]
