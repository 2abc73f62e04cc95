"""Mode-1 sharded stream protocol on the CPU oracle (TEST INFRASTRUCTURE).

A rank-local restatement of the multi-GPU stream step
that exchanges its partials through torch.distributed, so the N > 1 protocol
-- row ownership, virtual-shard partition, local fibre offsets, the exchange
layout and the fixed-order combine -- runs with world_size 2 on `gloo` here.
The GPU implementation (paper_2007_10798_b200/csrc/shard_kernels.cuh and
shard_host.inc) follows the same plan over peer memory (NCCL all-gather as the
alternative); both must reproduce orc_stream_consume_sharded bit for bit.

Rank g of G owns virtual shards [g V/G, (g+1) V/G), i.e. mode-1 rows
[lo(g V/G), lo((g+1) V/G)) with lo(v) = floor(v I_1 / V).
"""
import numpy as np

from oracle import oracle as orc


def shard_lo(v, I1, V):
    return (v * I1) // V


def shard_of(i0, I1, V):
    """Virtual shard of 0-based mode-1 row i0 (oracle shard_of)."""
    return ((i0 + 1) * V - 1) // I1


def rank_rows(world, rank, I1, V):
    assert V % world == 0
    v0, v1 = rank * V // world, (rank + 1) * V // world
    return v0, v1, shard_lo(v0, I1, V), shard_lo(v1, I1, V)


class ShardedStream:
    """One rank's share of a RocpStream: U(1) / P(1) rows [r0, r1), every other
    factor, P(n), Q(n) and the temporal factor replicated."""

    def __init__(self, factors, temporal, p, q, s, world, rank, V, allgather):
        self.head = [f.shape[0] for f in factors]
        self.N = len(factors) + 1
        self.R = factors[0].shape[1]
        self.s, self.world, self.rank, self.V = s, world, rank, V
        self.v0, self.v1, self.r0, self.r1 = rank_rows(world, rank, self.head[0], V)
        self.U = [np.asfortranarray(f) for f in factors]
        self.U[0] = np.asfortranarray(factors[0][self.r0:self.r1])
        self.P = [np.asfortranarray(m) for m in p]
        self.P[0] = np.asfortranarray(p[0][self.r0:self.r1])
        self.Q = [np.asfortranarray(m) for m in q]
        self.temporal = np.asfortranarray(temporal)
        self.allgather = allgather  # list of per-rank float64 arrays from this rank's array

    def _local_partials(self, x_local, d_local, mode, dec, factors_ex):
        """Per local virtual shard: (gram, contraction) over its samples in order."""
        I1 = self.head[0]
        v_of = np.array([shard_of(int(i) - 1, I1, self.V) for i in dec[:, 0]], dtype=np.int64)
        rows = d_local[mode - 1]
        out = []
        for v in range(self.v0, self.v1):
            sel = dec[v_of == v].copy()
            sel[:, 0] -= self.r0  # mode-1 index to this rank's rows
            if sel.shape[0]:
                z = orc.sampled_khatri_rao(sel, factors_ex)
                x = orc.sample_unfolding(x_local, d_local, mode, sel)
                out.append(np.concatenate([orc.gram(z).ravel(order="F"), orc.contract(x, z).ravel(order="F")]))
            else:
                out.append(np.zeros(self.R * self.R + rows * self.R))
        return np.concatenate(out)

    def _exchange_combine(self, local, rows):
        parts = self.allgather(local)  # rank order == shard order
        blk = self.R * self.R + rows * self.R
        allp = np.concatenate(parts).reshape(self.V, blk)
        tot = allp[0].copy()
        for v in range(1, self.V):
            tot = tot + allp[v]
        g = tot[:self.R * self.R].reshape(self.R, self.R, order="F")
        inc = tot[self.R * self.R:].reshape(rows, self.R, order="F")
        return g, inc

    def consume(self, x_local, batch, seed, batch_id):
        N, R = self.N, self.R
        d_global = self.head + [batch]
        d_local = [self.r1 - self.r0] + self.head[1:] + [batch]
        model = [self.U[0]] + self.U[1:] + [None]
        # temporal stage: shards of the head samples
        _, dec = orc.draw_samples(d_global, N, self.s, seed, batch_id, 0)
        fex = [self.U[k - 1] for k in range(N - 1, 0, -1)]
        g, rhs = self._exchange_combine(self._local_partials(x_local, d_local, N, dec, fex), batch)
        u_new, _ = orc.solve_gram(g, rhs)
        self.temporal = np.asfortranarray(np.vstack([self.temporal, u_new]))
        # modes 1..N-1
        for n in range(1, N):
            _, dec = orc.draw_samples(d_global, n, self.s, seed, batch_id, 0)
            fex = [u_new] + [self.U[k - 1] for k in range(N - 1, 0, -1) if k != n]
            if n == 1:  # owned mode: local rows, replicated Z / Q, no exchange
                z = orc.sampled_khatri_rao(dec, fex)
                x = orc.sample_unfolding(x_local, d_local, 1, dec)
                self.Q[0] = self.Q[0] + orc.gram(z)
                self.P[0] = np.asfortranarray(self.P[0] + orc.contract(x, z))
                self.U[0], _ = orc.solve_gram(self.Q[0], self.P[0])
                continue
            g, inc = self._exchange_combine(self._local_partials(x_local, d_local, n, dec, fex), self.head[n - 1])
            self.P[n - 1] = np.asfortranarray(self.P[n - 1] + inc)
            self.Q[n - 1] = self.Q[n - 1] + g
            self.U[n - 1], _ = orc.solve_gram(self.Q[n - 1], self.P[n - 1])
        del model


def local_rows(x, dims, r0, r1):
    """Rows [r0, r1) of mode 1 of a flat first-index-fastest tensor."""
    t = np.asarray(x).reshape(dims[::-1])
    return np.ascontiguousarray(t[..., r0:r1]).ravel()
