"""Overlapped window gather: the window's sampled-fibre gather
runs as k_gather_warps on SMs reserved beside the persistent chain kernel, which
waits per (batch, stage) on the published unit counts.  The stream must stay
bit-identical to the oracle (and to the serial gather) for every SM split and
every unit kind: TMA boxes for strided and mode-1 fibres (even I1), LSU loads
for odd I1, temporal fibres longer than one box, 4- and 5-way tensors, the wide
chain (R > 32)."""
import numpy as np
import pytest

import paper_2007_10798_b200 as rocp
from tests import helpers as H
from tests.test_gpu_parity import _cmp_stream, _run_pair

pytestmark = pytest.mark.gpu


def bitwise(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


@pytest.fixture
def gdev(dev):
    yield dev
    dev.set_gather_sms(-1)


@pytest.mark.parametrize("name,dims,R,t_init,B,nbat", [
    ("3-way even I1 (TMA units)", [64, 300, 140], 6, 40, 10, None),
    ("3-way odd I1 (LSU units)", [63, 300, 140], 6, 40, 10, None),
    ("temporal fibre > one box", [16, 12, 700], 4, 100, 300, 2),
    ("4-way", [24, 30, 20, 60], 5, 20, 8, None),
    ("5-way", [8, 10, 6, 12, 40], 4, 10, 6, None),
    ("2-way", [50, 120], 4, 30, 9, None),
    ("wide chain R=40", [120, 90, 80], 40, 40, 10, 3),
])
@pytest.mark.parametrize("sms", [8, 20])
def test_overlapped_window_bitwise(gdev, name, dims, R, t_init, B, nbat, sms):
    x, X, a, b, s, nb = _run_pair(gdev, dims, R, 20.0, t_init, B, nbatches=nbat)
    gdev.set_gather_sms(sms)
    a.checkpoint()
    a.consume_range(X, t_init, B, nb, 4242, 1)  # one window, gather overlapped
    for k in range(nb):
        b.consume(H.slab(x, dims, t_init + k * B, B), B, 4242, k + 1)
    _cmp_stream(a, b, len(dims))
    assert bitwise(a.last_residuals(), b.last_residuals())
    over = [a.factor(n) for n in range(1, len(dims))] + [a.temporal()]
    # the serial gather (every SM, before the chain) gives the same bits; so does a replay
    for g in (0, sms):
        gdev.set_gather_sms(g)
        a.restore()
        a.consume_range(X, t_init, B, nb, 4242, 1)
        again = [a.factor(n) for n in range(1, len(dims))] + [a.temporal()]
        assert all(bitwise(u, v) for u, v in zip(over, again)), f"gather_sms={g}"


def test_overlapped_single_batches(gdev):
    """consume() of one batch at a time also overlaps (stage 0's chain with the
    later stages' gathers)."""
    dims, R, t_init, B = [40, 36, 90], 5, 30, 10
    x, X, a, b, s, nb = _run_pair(gdev, dims, R, 20.0, t_init, B)
    gdev.set_gather_sms(12)
    for k in range(nb):
        t0 = t_init + k * B
        a.consume(X.slab(t0, B), 99, k + 1)
        b.consume(H.slab(x, dims, t0, B), B, 99, k + 1)
    _cmp_stream(a, b, len(dims))


def test_gather_sms_bounds(gdev):
    with pytest.raises(rocp.DomainError):
        gdev.set_gather_sms(10_000)
    gdev.set_gather_sms(-1)


def test_gather_window_profiling_entry(gdev):
    """rocp_stream_gather_window (bench.py's whole-device gather roofline) only fills the window
    scratch: the stream's model is untouched and a following window is still bit-identical."""
    dims, R, t_init, B = [64, 200, 100], 5, 30, 10
    x, X, a, b, s, nb = _run_pair(gdev, dims, R, 20.0, t_init, B)
    a.checkpoint()
    before = [a.factor(n) for n in (1, 2)] + [a.temporal()]
    for sms in (0, 8):
        ms = a.gather_window(X, t_init, B, nb, 77, 1, sms)
        assert ms > 0.0
    assert all(bitwise(u, v) for u, v in zip(before, [a.factor(n) for n in (1, 2)] + [a.temporal()]))
    gdev.set_gather_sms(8)
    a.consume_range(X, t_init, B, nb, 4243, 1)
    assert a.last_gather_sms == 8
    for k in range(nb):
        b.consume(H.slab(x, dims, t_init + k * B, B), B, 4243, k + 1)
    _cmp_stream(a, b, len(dims))
    gdev.set_gather_sms(0)
    a.restore()
    a.consume_range(X, t_init, B, nb, 4243, 1)
    assert a.last_gather_sms == 0


def test_second_handle_on_the_gpu_gathers_serially(gdev):
    """Two live handles on one GPU: the model stops overlapping (two cooperative chains and their
    spinning gathers could otherwise hold each other's SMs); results stay bitwise equal."""
    dims, R, t_init, B = [600, 600, 60], 6, 20, 10  # a gather share the model overlaps
    x, X, a, b, s, nb = _run_pair(gdev, dims, R, 20.0, t_init, B)
    gdev.set_gather_sms(-1)
    a.checkpoint()
    a.consume_range(X, t_init, B, nb, 99, 1)
    alone = a.last_gather_sms
    assert alone > 0
    ref = [a.factor(n) for n in (1, 2)] + [a.temporal()]
    other = rocp.Device(0)
    try:
        a.restore()
        a.consume_range(X, t_init, B, nb, 99, 1)
        assert a.last_gather_sms == 0
        assert all(bitwise(u, v) for u, v in zip(ref, [a.factor(n) for n in (1, 2)] + [a.temporal()]))
    finally:
        other.close()
    a.restore()
    a.consume_range(X, t_init, B, nb, 99, 1)
    assert a.last_gather_sms == alone
