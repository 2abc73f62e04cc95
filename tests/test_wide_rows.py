"""Rows of solve_gram: u = b G^-1 against the explicit inverse that the
symmetric sweep forms, instead of an LDL^T factorisation and a 2R-step substitution per
row.  The canonical order differs from the reference's, so this pins it against
independent solves at wide ranks: the reference's solve_gram is an LDLT solve
(solve.cpp:34), and the sampled-LS properties of test_cprand.cpp:25-57 must hold with the
same tolerances."""
import json
import os

import numpy as np
import pytest

from oracle import oracle as orc
from tests import helpers as H

KAT = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_kat.json")))
TOL = {k: v[0] for k, v in KAT["tolerances"].items()}


@pytest.mark.parametrize("R", [33, 40, 50, 64])
def test_inverse_rows_match_independent_solve(R):
    g = H.rng(R)
    z = H.random_matrix(int(np.ceil(10 * R * np.log(R))), R, g)  # a sampled KR-like system, kappa ~ 10
    G = orc.gram(z)
    rhs = H.random_matrix(300, R, g)
    u, reg = orc.solve_gram(G, rhs)
    ref = np.linalg.solve(G, rhs.T).T
    assert not reg
    assert np.abs(u - ref).max() <= 1e-12 * np.abs(ref).max()


@pytest.mark.parametrize("R", [33, 50])
def test_wide_sampled_ls_properties(R):
    g = H.rng(100 + R)
    x = H.random_matrix(7, R, g)
    u, reg, und = orc.solve_sampled_ls(np.eye(R), x)  # identity -> rhs (test_cprand.cpp:28-32)
    assert np.abs(u - x).max() < TOL["sampled_ls_identity"] and not reg and not und
    zq, _ = np.linalg.qr(g.standard_normal((4 * R, R)))  # orthonormal -> projection (:34-41)
    xx = H.random_matrix(6, 4 * R, g)
    u, _, _ = orc.solve_sampled_ls(zq, xx)
    assert np.abs(u - xx @ zq).max() < TOL["sampled_ls_orthonormal"]
    u0 = H.random_matrix(6, R, g)  # plant and recover (:43-49)
    z = H.random_matrix(5 * R, R, g)
    u, _, _ = orc.solve_sampled_ls(z, u0 @ z.T)
    assert np.linalg.norm(u - u0) <= TOL["sampled_ls_planted"] * np.linalg.norm(u0)


def test_wide_ill_conditioned_still_regularises():
    R = 40
    g = H.rng(7)
    q, _ = np.linalg.qr(g.standard_normal((R, R)))
    G = np.asfortranarray((q * np.geomspace(1.0, 1e-14, R)) @ q.T)
    G = np.asfortranarray((G + G.T) / 2)
    u, reg = orc.solve_gram(G, H.random_matrix(5, R, g))
    assert reg and np.isfinite(u).all()
