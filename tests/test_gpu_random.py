"""Randomised bit-exact parity sweep (GPU vs oracle) over stream shapes the
fixed cases do not pin: orders 2..6, ranks 1..40 (both chain kernel
instances, padded and unpadded R), ragged extents (row tiles, chunks and
superchunks with tails), batch sizes 1..12, explicit sample counts, plus the
host-slab range and the sharded stream on a subset."""
import numpy as np
import pytest

import paper_2007_10798_b200 as rocp
from oracle import oracle as orc
from tests import helpers as H

pytestmark = pytest.mark.gpu


def bitwise(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


def _case(k):
    g = np.random.default_rng(8800 + k)
    N = int(g.integers(2, 7))
    R = int(g.choice([1, 2, 3, 5, 8, 11, 16, 20, 24, 33, 40]))
    hi = 70 if N <= 3 else (14 if N <= 4 else 7)
    head = [int(g.integers(min(max(2, R // 3), hi - 2), hi)) for _ in range(N - 1)]
    B = int(g.integers(1, 13))
    t_init = int(g.integers(max(4, R // 2), 24))
    nb = int(g.integers(1, 5))
    s = int(g.choice([0, 7, 33, 257, 300]))
    return N, R, head, B, t_init, nb, s


@pytest.mark.parametrize("k", range(48))
def test_random_stream_bitwise(dev, k):
    N, R, head, B, t_init, nb, s_req = _case(k)
    dims = head + [t_init + nb * B]
    g = H.rng(9900 + k)
    x, _ = H.gen_synthetic(dims, R, 25.0, g)
    idims = head + [t_init]
    xi = H.slab(x, dims, 0, t_init)
    init0 = H.random_model(idims, R, H.rng(k + 1))
    kw = dict(samples=s_req, max_iters=6)
    a_init = rocp.cprand_decompose(dev, dev.tensor(idims, xi), R, init0, seed=k + 3, **kw)
    b_init = orc.cprand_decompose(xi, idims, R, init0, seed=k + 3, **kw)
    for n in range(len(dims)):
        assert bitwise(a_init.model[n], b_init.model[n]), f"cprand factor {n}"
    s = a_init.samples
    a = rocp.RocpStream(dev, a_init, s, t_capacity=dims[-1])
    b = orc.Stream(b_init.model, t_init, b_init.best_sampled_kr, s, regularized=b_init.regularized)
    X = dev.tensor(dims, x)
    if k % 2:  # host-slab range, one call
        a.consume_range_host(H.slab(x, dims, t_init, nb * B), B, nb, 61 + k, 1)
    else:      # device window, one persistent launch
        a.consume_range(X, t_init, B, nb, 61 + k, 1)
    for j in range(nb):
        b.consume(H.slab(x, dims, t_init + j * B, B), B, 61 + k, j + 1)
    for n in range(1, N):
        assert bitwise(a.factor(n), b.factor(n)), f"U{n}"
        assert bitwise(a.p(n), b.p(n)), f"P{n}"
        assert bitwise(a.q(n), b.q(n)), f"Q{n}"
    assert bitwise(a.temporal(), b.temporal())
    assert a.regularized == b.regularized
    if k % 3 == 0 and head[0] >= 4:  # the sharded stream on the same data
        V = 4 if head[0] >= 8 else 2
        c = rocp.RocpStream(dev, a_init, s, t_capacity=dims[-1])
        d = orc.Stream(b_init.model, t_init, b_init.best_sampled_kr, s, regularized=b_init.regularized)
        c.shard(V)
        XL = X.rows(0, head[0])
        c.consume_range(XL, t_init, B, nb, 77 + k, 1)
        for j in range(nb):
            d.consume_sharded(H.slab(x, dims, t_init + j * B, B), B, 77 + k, j + 1, V)
        for n in range(1, N):
            assert bitwise(c.factor(n), d.factor(n)), f"sharded U{n}"
        assert bitwise(c.temporal(), d.temporal())
