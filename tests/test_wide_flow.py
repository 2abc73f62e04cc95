"""The dataflow chain's wide instances (k_flow for R in 33..64, ROCP_CHAIN=flow): bit-identical to
the oracle's stream like the default grid-barrier chain they stand in for (slower on
C4, so not the default).  The chain kernel is picked once per process, so the check runs in a
child process with the selector set."""
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
for dims, R, t_init, B, sms in [([120, 90, 80], 40, 40, 10, 8), ([96, 70, 60, 60], 36, 20, 10, 0)]:
    dev.set_gather_sms(sms)
    x, X, a, b, s, nb = _run_pair(dev, dims, R, 20.0, t_init, B, nbatches=3)
    a.consume_range(X, t_init, B, nb, 4242, 1)
    for k in range(nb):
        b.consume(H.slab(x, dims, t_init + k * B, B), B, 4242, k + 1)
    _cmp_stream(a, b, len(dims))
    ra, rb = np.asarray(a.last_residuals()), np.asarray(b.last_residuals())
    assert np.array_equal(ra.view(np.uint64), rb.view(np.uint64))
print("wide flow ok")
'''


def test_wide_flow_stream_bitwise():
    env = dict(os.environ, ROCP_CHAIN="flow", PYTHONPATH=ROOT)
    r = subprocess.run([sys.executable, "-c", CHILD], cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "wide flow ok" in r.stdout
