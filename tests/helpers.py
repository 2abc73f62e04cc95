"""Shared test fixtures: seeded synthetic data and planted models (numpy).

Mirrors the reference's test helpers: random_matrix / init_from_model /
planted_slab (test_rocp.cpp:16-46) and gen_synthetic / split_stream
(synthetic.cpp:8-57).  numpy's Generator stands in for std::mt19937_64 +
std::normal_distribution; both the oracle and the GPU receive the same bytes.
"""
import numpy as np

from oracle import oracle as orc


def rng(seed):
    return np.random.default_rng(seed)


def random_matrix(rows, cols, g):
    return np.asfortranarray(g.standard_normal((rows, cols)))


def random_model(dims, rank, g):
    return [random_matrix(d, rank, g) for d in dims]


def reconstruct(factors, dims):
    return orc.reconstruct(factors, dims)


def gen_synthetic(dims, rank, snr_db, g, factors=None):
    """X = [[A]] + E, |E| scaled to the exact SNR (synthetic.cpp:8-31)."""
    truth = factors if factors is not None else random_model(dims, rank, g)
    x = reconstruct(truth, dims)
    if snr_db is not None:
        e = g.standard_normal(x.size)
        scale = np.linalg.norm(x) * 10.0 ** (-snr_db / 20.0) / np.linalg.norm(e)
        x = x + scale * e
    return x, truth


def slab(x, dims, t0, length):
    """Contiguous slab of the last mode (split_stream, synthetic.cpp:44-55)."""
    slice_ = int(np.prod(dims[:-1]))
    return np.ascontiguousarray(x[t0 * slice_:(t0 + length) * slice_])


def init_from_model(model, dims, s, seed):
    """InitResult assembled from a model with fresh draws (test_rocp.cpp:25-34),
    keyed like cprand's Z_best rebuild (batch 0, iteration 0)."""
    kr = []
    for n in range(1, len(model)):
        _, dec = orc.draw_samples(dims, n, s, seed, 0, 0)
        kr.append(orc.sampled_khatri_rao(dec, orc.factors_excluding(model, n)))
    return orc.InitResult([np.asfortranarray(m) for m in model], kr, 0.0, 0, False, np.zeros(0))


def planted_slab(truth, head, count, g):
    """count new slices of the planted model with fresh temporal rows (test_rocp.cpp:38-46)."""
    rows = random_matrix(count, truth[0].shape[1], g)
    model = list(truth[:-1]) + [rows]
    return reconstruct(model, list(head) + [count]), rows


def congruent_factors(dims, rank, congruence, g):
    """Factors with pairwise column congruence c (BASELINE.json configs[4]):
    G L^T with G iid N(0,1) and L = chol(c 11^T + (1-c) I)."""
    C = np.full((rank, rank), congruence) + (1.0 - congruence) * np.eye(rank)
    L = np.linalg.cholesky(C)
    return [np.asfortranarray(g.standard_normal((d, rank)) @ L.T) for d in dims]
