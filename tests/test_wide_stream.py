"""The wide chain's streamed pair items (k_chain<true>, chain_stream_items): every
padded width (RP = 40, 48, 56, 64), an odd number of row tiles (the last pair holds one tile),
stages smaller than one tile, a last superchunk that is not full, 3- and 4-way streams, serial
and overlapped gathers -- bit-identical to the oracle's stream.  A child process with
ROCP_CHAIN_STREAM=0 runs the tile-at-a-time items the streamed ones replace (the fallback when no
tensor map can be made) on the same case."""
import os
import subprocess
import sys

import numpy as np
import pytest

from tests import helpers as H
from tests.test_gpu_parity import _cmp_stream, _run_pair

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def bitwise(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


@pytest.mark.parametrize("dims,R,t_init,B,sms", [
    ([70, 45, 60], 36, 30, 10, 0),        # RP 40; 3 row tiles (odd), 2 tiles, a 10-row temporal stage
    ([100, 33, 50], 44, 20, 10, 8),       # RP 48; overlapped gather
    ([96, 130, 40], 50, 20, 10, 0),       # RP 56 (the C4 width); 5 row tiles
    ([40, 72, 48], 57, 24, 8, 8),         # RP 64, 5 ring stages
    ([30, 28, 26, 40], 64, 16, 8, 0),     # RP 64, R a multiple of 8; 4-way: every stage below one tile
    ([66, 20, 18, 30], 41, 12, 6, 12),    # RP 48; 4-way, overlapped
])
def test_streamed_wide_chain_bitwise(dev, dims, R, t_init, B, sms):
    dev.set_gather_sms(sms)
    try:
        x, X, a, b, s, nb = _run_pair(dev, dims, R, 20.0, t_init, B, nbatches=2, kw=dict(max_iters=4))
        a.consume_range(X, t_init, B, nb, 777, 1)
        for k in range(nb):
            b.consume(H.slab(x, dims, t_init + k * B, B), B, 777, k + 1)
        _cmp_stream(a, b, len(dims))
        assert bitwise(a.last_residuals(), b.last_residuals())
    finally:
        dev.set_gather_sms(-1)


def test_streamed_wide_chain_host_slabs_and_single_batches(dev):
    """The same bits through the reference-facing calls: consume() batch by batch on host slabs,
    and the whole range from host memory (sampled fibres gathered by host threads, chain per batch)."""
    import paper_2007_10798_b200 as rocp
    dims, R, t_init, B = [96, 130, 40], 50, 20, 10
    x, X, a, b, s, nb = _run_pair(dev, dims, R, 20.0, t_init, B, nbatches=2, kw=dict(max_iters=4))
    a.checkpoint()
    for k in range(nb):
        a.consume(H.slab(x, dims, t_init + k * B, B), 777, k + 1)
        b.consume(H.slab(x, dims, t_init + k * B, B), B, 777, k + 1)
    _cmp_stream(a, b, len(dims))
    ref = [a.factor(1), a.factor(2), a.temporal()]
    a.restore()
    a.consume_range_host(H.slab(x, dims, t_init, B * nb), B, nb, 777, 1)
    assert bitwise(a.factor(1), ref[0]) and bitwise(a.factor(2), ref[1]) and bitwise(a.temporal(), ref[2])
    slab = H.slab(x, dims, t_init, B * nb)
    hb = rocp.HostBuffer(slab.size)
    hb.array[:] = slab
    a.restore()
    a.consume_range_host(hb.array, B, nb, 777, 1)
    assert bitwise(a.factor(1), ref[0]) and bitwise(a.factor(2), ref[1]) and bitwise(a.temporal(), ref[2])
    hb.free()


CHILD = r'''
import numpy as np
import paper_2007_10798_b200 as rocp
from tests import helpers as H
from tests.test_gpu_parity import _cmp_stream, _run_pair
dev = rocp.Device(0)
x, X, a, b, s, nb = _run_pair(dev, [96, 130, 40], 50, 20.0, 20, 10, nbatches=2, kw=dict(max_iters=4))
a.consume_range(X, 20, 10, nb, 777, 1)
for k in range(nb):
    b.consume(H.slab(x, [96, 130, 40], 20 + k * 10, 10), 10, 777, k + 1)
_cmp_stream(a, b, 3)
print("tile items ok")
'''


def test_tile_items_fallback_bitwise():
    env = dict(os.environ, ROCP_CHAIN_STREAM="0", PYTHONPATH=ROOT)
    r = subprocess.run([sys.executable, "-c", CHILD], cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "tile items ok" in r.stdout
