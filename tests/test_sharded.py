"""Mode-1 sharded stream on the CPU: the oracle's
sharded canonical order and the N > 1 exchange protocol over torch.distributed
(gloo, world_size 2)."""
import os
import socket
import tempfile

import numpy as np
import pytest

from oracle import oracle as orc
from tests import helpers as H
from tests import shard_protocol as SP


def bitwise(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


def _setup(dims, R, t_init, seed=5, snr=20.0):
    g = H.rng(seed)
    x, _ = H.gen_synthetic(dims, R, snr, g)
    head = dims[:-1]
    init = H.random_model(head + [t_init], R, H.rng(seed + 1))
    s = orc.auto_sample_count(R)
    kr = []
    for n in range(1, len(dims)):
        _, dec = orc.draw_samples(head + [t_init], n, s, 77, 0, 0)
        kr.append(orc.sampled_khatri_rao(dec, orc.factors_excluding(init, n)))
    return x, init, kr, s


def _stream(init, t_init, kr, s):
    return orc.Stream(init, t_init, kr, s)


CASES = [([24, 10, 60], 4, 20, 8), ([16, 6, 5, 30], 3, 10, 5), ([9, 4, 4, 3, 20], 2, 8, 4)]


@pytest.mark.parametrize("dims,R,t_init,B", CASES)
def test_one_virtual_shard_is_consume(dims, R, t_init, B):
    x, init, kr, s = _setup(dims, R, t_init)
    a, b = _stream(init, t_init, kr, s), _stream(init, t_init, kr, s)
    for k in range((dims[-1] - t_init) // B):
        xb = H.slab(x, dims, t_init + k * B, B)
        a.consume(xb, B, 91, k + 1)
        b.consume_sharded(xb, B, 91, k + 1, 1)
    for n in range(1, len(dims)):
        assert bitwise(a.factor(n), b.factor(n)) and bitwise(a.p(n), b.p(n)) and bitwise(a.q(n), b.q(n))
    assert bitwise(a.temporal(), b.temporal())
    assert bitwise(a.last_residuals(), b.last_residuals())


@pytest.mark.parametrize("dims,R,t_init,B", CASES)
def test_sharded_order_matches_unsharded_within_tolerance(dims, R, t_init, B):
    """Only the summation order of the temporal / non-owned-mode partials
    changes: the stream agrees with the unsharded one to 1e-9 (north star)."""
    x, init, kr, s = _setup(dims, R, t_init)
    a, b = _stream(init, t_init, kr, s), _stream(init, t_init, kr, s)
    V = min(8, dims[0])
    for k in range((dims[-1] - t_init) // B):
        xb = H.slab(x, dims, t_init + k * B, B)
        a.consume(xb, B, 92, k + 1)
        b.consume_sharded(xb, B, 92, k + 1, V)
    for n in range(1, len(dims)):
        ua, ub = a.factor(n), b.factor(n)
        assert np.linalg.norm(ua - ub) <= 1e-9 * np.linalg.norm(ua)
    ta, tb = a.temporal(), b.temporal()
    assert np.linalg.norm(ta - tb) <= 1e-9 * np.linalg.norm(ta)


def test_rank_rows_partition():
    for I1, V in [(4000, 8), (60, 8), (8, 8), (13, 4)]:
        for world in [w for w in (1, 2, 4, 8) if V % w == 0]:
            spans = [SP.rank_rows(world, r, I1, V)[2:] for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == I1
            assert all(spans[r][1] == spans[r + 1][0] for r in range(world - 1))
        owners = [SP.shard_of(i, I1, V) for i in range(I1)]
        assert owners == sorted(owners) and owners[0] == 0 and owners[-1] == V - 1
        for i in range(I1):
            assert SP.shard_lo(owners[i], I1, V) <= i < SP.shard_lo(owners[i] + 1, I1, V)


def _free_port():
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def _rank_main(rank, world, port, dims, R, t_init, B, V, out_path):
    import torch
    import torch.distributed as dist

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", world_size=world, rank=rank)

    def allgather(a):
        t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
        parts = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(parts, t)
        return [p.numpy() for p in parts]

    x, init, kr, s = _setup(dims, R, t_init)
    ref = _stream(init, t_init, kr, s)  # P, Q of init_state (rocp.cpp:45-69)
    st = SP.ShardedStream(init[:-1], init[-1], [ref.p(n) for n in range(1, len(dims))],
                          [ref.q(n) for n in range(1, len(dims))], s, world, rank, V, allgather)
    for k in range((dims[-1] - t_init) // B):
        xl = SP.local_rows(H.slab(x, dims, t_init + k * B, B), dims[:-1] + [B], st.r0, st.r1)
        st.consume(xl, B, 93, k + 1)
    # gather U(1) rows back in rank order
    u1 = np.concatenate(allgather(st.U[0].ravel(order="F")))
    if rank == 0:
        np.savez(out_path, u1=u1, temporal=st.temporal, **{f"u{n}": st.U[n - 1] for n in range(2, len(dims))},
                 **{f"p{n}": st.P[n - 1] for n in range(2, len(dims))}, **{f"q{n}": st.Q[n - 1] for n in range(1, len(dims))})
    dist.destroy_process_group()


@pytest.mark.parametrize("dims,R,t_init,B", CASES[:2])
def test_gloo_world2_protocol_matches_sharded_oracle(dims, R, t_init, B):
    import multiprocessing as mp

    V, world = 8 if dims[0] >= 8 else 4, 2
    out = os.path.join(tempfile.mkdtemp(), "rank0.npz")
    port = _free_port()
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, dims, R, t_init, B, V, out)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    got = np.load(out)
    x, init, kr, s = _setup(dims, R, t_init)
    ref = _stream(init, t_init, kr, s)
    for k in range((dims[-1] - t_init) // B):
        ref.consume_sharded(H.slab(x, dims, t_init + k * B, B), B, 93, k + 1, V)
    I1 = dims[0]
    u1_ref = ref.factor(1)
    rows = [SP.rank_rows(world, r, I1, V)[2:] for r in range(world)]
    u1 = np.concatenate([got["u1"][sum((b - a) * R for a, b in rows[:r]):][:(rows[r][1] - rows[r][0]) * R]
                         .reshape(rows[r][1] - rows[r][0], R, order="F") for r in range(world)])
    assert bitwise(u1, u1_ref)
    assert bitwise(got["temporal"], ref.temporal())
    for n in range(2, len(dims)):
        assert bitwise(got[f"u{n}"], ref.factor(n)) and bitwise(got[f"p{n}"], ref.p(n))
    for n in range(1, len(dims)):
        assert bitwise(got[f"q{n}"], ref.q(n))
