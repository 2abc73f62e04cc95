"""The grid-barrier chain for R <= 32 (k_chain<false>, ROCP_CHAIN=barrier; also what a stream falls
back to when too few blocks are left for the dataflow chain): bit-identical to the oracle, with
the Gram combined by one block (few chunks) and with the superchunk pre-sums by the chunk blocks
(R = 32: more chunk partials than one block holds).  The chain kernel is picked once per process,
so the check runs in a child process with the selector set."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import numpy as np
import paper_2007_10798_b200 as rocp
from tests import helpers as H
from tests.test_gpu_parity import _cmp_stream, _run_pair
dev = rocp.Device(0)
for dims, R, t_init, B, sms in [([64, 90, 80], 6, 30, 10, 0), ([120, 70, 60], 20, 30, 10, 8),
                                ([70, 50, 60], 32, 24, 12, 0), ([40, 30, 20, 50], 32, 20, 10, 8)]:
    dev.set_gather_sms(sms)
    x, X, a, b, s, nb = _run_pair(dev, dims, R, 20.0, t_init, B, nbatches=3, kw=dict(max_iters=4))
    a.consume_range(X, t_init, B, nb, 4242, 1)
    for k in range(nb):
        b.consume(H.slab(x, dims, t_init + k * B, B), B, 4242, k + 1)
    _cmp_stream(a, b, len(dims))
    ra, rb = np.asarray(a.last_residuals()), np.asarray(b.last_residuals())
    assert np.array_equal(ra.view(np.uint64), rb.view(np.uint64))
print("barrier chain ok")
'''


def test_barrier_chain_stream_bitwise():
    env = dict(os.environ, ROCP_CHAIN="barrier", PYTHONPATH=ROOT)
    r = subprocess.run([sys.executable, "-c", CHILD], cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "barrier chain ok" in r.stdout
