"""Several independent streams on one GPU, one handle each, their persistent chains on a share of
the SMs (rocp_set_chain_sms; the reference's trial-level parallelism, bench.cpp:190-213): every
stream stays bit-identical to the oracle, whatever the share and however the calls interleave."""
import numpy as np
import pytest

import paper_2007_10798_b200 as rocp
from tests import helpers as H
from tests.test_gpu_parity import _cmp_stream, _run_pair

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dims,R,t_init,B,sms", [
    ([64, 300, 140], 6, 40, 10, 40),   # the dataflow chain on 40 blocks
    ([60, 50, 90], 20, 30, 10, 30),    # fewer free blocks than items
    ([96, 130, 60], 50, 20, 10, 36),   # the wide chain with streamed items
    ([60, 50, 90], 20, 30, 10, 16),    # too few blocks for the dataflow chain: the grid-barrier chain, two chunks per block
    ([50, 40, 60], 32, 24, 12, 16),    # the same with the chunk blocks' superchunk pre-sums
    ([96, 130, 60], 50, 20, 10, 16),   # the wide chain with one or two blocks per superchunk
])
def test_concurrent_streams_bitwise(dims, R, t_init, B, sms):
    K = 3
    devs = [rocp.Device(0) for _ in range(K)]
    try:
        pairs = []
        for i, d in enumerate(devs):
            d.set_chain_sms(sms)
            pairs.append(_run_pair(d, dims, R, 20.0, t_init, B, seed=29 + i, nbatches=3, kw=dict(max_iters=4)))
        for i, (x, X, a, b, s, nb) in enumerate(pairs):  # enqueue every stream's window, then compare
            a.consume_range(X, t_init, B, nb, 100 + i, 1)
        for i, (x, X, a, b, s, nb) in enumerate(pairs):
            for k in range(nb):
                b.consume(H.slab(x, dims, t_init + k * B, B), B, 100 + i, k + 1)
            _cmp_stream(a, b, len(dims))
    finally:
        for d in devs:
            d.close()


def test_chain_sms_domain(dev):
    with pytest.raises(ValueError):
        dev.set_chain_sms(8)
    with pytest.raises(ValueError):
        dev.set_chain_sms(100000)
    dev.set_chain_sms(0)
    assert dev.sm_count >= 16
