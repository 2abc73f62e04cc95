"""The reference's binary records (tensor_io.cpp:12-101, rocp.cpp:180-211):
tensor files, ComplementaryState (save_state/load_state) and resumable
checkpoints of the device stream."""
import os
import struct
import tempfile

import numpy as np
import pytest

import paper_2007_10798_b200 as rocp
from oracle import oracle as orc
from tests import helpers as H


def bitwise(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


def record_bytes(arr_colmajor, dims):
    """write_tensor (tensor_io.cpp:49-56), restated for the test."""
    out = b"ROCP" + bytes([1]) + struct.pack("<I", len(dims))
    out += b"".join(struct.pack("<Q", d) for d in dims)
    return out + np.asarray(arr_colmajor, dtype="<f8").tobytes()


def test_record_layout_known_bytes():
    """2 x 2 matrix [[1, 2], [3, 4]]: column-major values after a 25-byte header."""
    m = np.array([[1.0, 2.0], [3.0, 4.0]])
    b = record_bytes(m.ravel(order="F"), [2, 2])
    assert b[:4] == b"ROCP" and b[4] == 1 and len(b) == 4 + 1 + 4 + 16 + 32
    assert struct.unpack("<I", b[5:9])[0] == 2
    assert struct.unpack("<4d", b[25:]) == (1.0, 3.0, 2.0, 4.0)
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "m.rocp")
        open(p, "wb").write(b + b + struct.pack("<Q", 7))
        recs = rocp.read_records(p)
        assert len(recs) == 2 and bitwise(recs[0], m) and bitwise(recs[1], m)


@pytest.mark.gpu
def test_tensor_file_roundtrip_and_errors(dev):
    dims = [7, 5, 3, 4]
    x = H.rng(3).standard_normal(int(np.prod(dims)))
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "t.rocp")
        dev.tensor(dims, x).write(p)
        raw = open(p, "rb").read()
        assert raw == record_bytes(x, dims)  # byte-identical to the reference writer
        q = os.path.join(d, "u.rocp")
        y = H.rng(4).standard_normal(int(np.prod(dims)))
        open(q, "wb").write(record_bytes(y, dims))
        t = dev.read_tensor(q)
        assert t.dims == dims and bitwise(t.download(), y)
        open(q, "wb").write(b"ROCX" + raw[4:])
        with pytest.raises(rocp.RecordError):
            dev.read_tensor(q)
        open(q, "wb").write(raw[:-8])
        with pytest.raises(rocp.RecordError):
            dev.read_tensor(q)
        with pytest.raises(rocp.RecordError):
            dev.read_tensor(os.path.join(d, "missing.rocp"))


def _stream_pair(dev, dims=(30, 24, 70), R=4, t_init=20):
    dims = list(dims)
    g = H.rng(11)
    x, _ = H.gen_synthetic(dims, R, 20.0, g)
    head = dims[:-1]
    init0 = H.random_model(head + [t_init], R, H.rng(12))
    init = rocp.cprand_decompose(dev, dev.tensor(head + [t_init], H.slab(x, dims, 0, t_init)), R, init0, seed=5)
    return x, dims, init


@pytest.mark.gpu
def test_state_record_matches_reference_format(dev):
    x, dims, init = _stream_pair(dev)
    st = rocp.RocpStream(dev, init, init.samples, t_capacity=dims[-1])
    X = dev.tensor(dims, x)
    for k in range(2):
        st.consume(X.slab(20 + 10 * k, 10), 71, k + 1)
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "state.rocp")
        st.write_state(p)
        recs = rocp.read_records(p)
        N = len(dims)
        assert len(recs) == 2 * (N - 1)
        for n in range(1, N):
            assert bitwise(recs[n - 1], st.p(n)) and bitwise(recs[N - 2 + n], st.q(n))
        assert struct.unpack("<Q", open(p, "rb").read()[-8:])[0] == st.t_len == 40
        # load_state into a second stream of the same shape
        other = rocp.RocpStream(dev, init, init.samples, t_capacity=dims[-1])
        other.read_state(p)
        for n in range(1, N):
            assert bitwise(other.p(n), st.p(n)) and bitwise(other.q(n), st.q(n))
        assert other.t_len == 40
        bad = os.path.join(d, "bad.rocp")
        open(bad, "wb").write(open(p, "rb").read()[:-40])
        with pytest.raises(rocp.RecordError):
            other.read_state(bad)


@pytest.mark.gpu
def test_checkpoint_resume_is_bitwise(dev):
    x, dims, init = _stream_pair(dev)
    X = dev.tensor(dims, x)
    a = rocp.RocpStream(dev, init, init.samples, t_capacity=dims[-1])
    for k in range(2):
        a.consume(X.slab(20 + 10 * k, 10), 72, k + 1)
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "ck.rocp")
        a.write_checkpoint(p)
        b = rocp.RocpStream.from_checkpoint(dev, p, t_capacity=dims[-1])
    assert b.t_len == a.t_len
    for k in range(2, 5):
        a.consume(X.slab(20 + 10 * k, 10), 72, k + 1)
        b.consume(X.slab(20 + 10 * k, 10), 72, k + 1)
    for n in range(1, len(dims)):
        assert bitwise(a.factor(n), b.factor(n)) and bitwise(a.p(n), b.p(n)) and bitwise(a.q(n), b.q(n))
    assert bitwise(a.temporal(), b.temporal()) and a.regularized == b.regularized


@pytest.mark.gpu
def test_file_backed_stream_equals_device_range(dev):
    x, dims, init = _stream_pair(dev)
    X = dev.tensor(dims, x)
    a = rocp.RocpStream(dev, init, init.samples, t_capacity=dims[-1])
    b = rocp.RocpStream(dev, init, init.samples, t_capacity=dims[-1])
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "x.rocp")
        X.write(p)
        a.consume_file(p, 20, 10, 5, 73, 1)
        with pytest.raises(rocp.DomainError):
            a.consume_file(p, 60, 10, 2, 73, 6)  # past the end of the record
    b.consume_range(X, 20, 10, 5, 73, 1)
    for n in range(1, len(dims)):
        assert bitwise(a.factor(n), b.factor(n)) and bitwise(a.p(n), b.p(n)) and bitwise(a.q(n), b.q(n))
    assert bitwise(a.temporal(), b.temporal())
