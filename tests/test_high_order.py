"""Orders 7 and 8 (kMaxOrder, the longest factor lists the kernels carry): the stream through the
dataflow chain (one window) and the per-stage path stay bit-identical to the oracle."""
import numpy as np
import pytest

import paper_2007_10798_b200 as rocp
from oracle import oracle as orc
from tests import helpers as H

pytestmark = pytest.mark.gpu


def bitwise(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


@pytest.mark.parametrize("dims,R,t_init,B,nb", [
    ([5, 4, 3, 4, 3, 3, 24], 6, 12, 4, 3),
    ([4, 3, 3, 3, 3, 3, 3, 22], 5, 10, 4, 3),
])
def test_high_order_stream_bitwise(dev, dims, R, t_init, B, nb):
    g = H.rng(sum(dims) + R)
    x, _ = H.gen_synthetic(dims, R, 25.0, g)
    head = dims[:-1]
    idims = head + [t_init]
    xi = H.slab(x, dims, 0, t_init)
    init0 = H.random_model(idims, R, H.rng(7))
    a_init = rocp.cprand_decompose(dev, dev.tensor(idims, xi), R, init0, seed=5, max_iters=6)
    b_init = orc.cprand_decompose(xi, idims, R, init0, seed=5, max_iters=6)
    for n in range(len(dims)):
        assert bitwise(a_init.model[n], b_init.model[n]), f"cprand factor {n}"
    s = a_init.samples
    a = rocp.RocpStream(dev, a_init, s, t_capacity=dims[-1])
    b = orc.Stream(b_init.model, t_init, b_init.best_sampled_kr, s, regularized=b_init.regularized)
    X = dev.tensor(dims, x)
    a.consume_range(X, t_init, B, nb, 31, 1)
    for j in range(nb):
        b.consume(H.slab(x, dims, t_init + j * B, B), B, 31, j + 1)
    N = len(dims)
    for n in range(1, N):
        assert bitwise(a.factor(n), b.factor(n)), f"U{n}"
        assert bitwise(a.p(n), b.p(n)), f"P{n}"
        assert bitwise(a.q(n), b.q(n)), f"Q{n}"
    assert bitwise(a.temporal(), b.temporal())
