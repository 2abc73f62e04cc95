// shard_kernels.cuh -- kernels of the mode-1 sharded stream.
//
// Rank g of G owns mode-1 rows [r0, r1) = the virtual shards [v0, v1) of V
// fixed row ranges [floor(v I1 / V), floor((v+1) I1 / V)).  For the temporal
// stage and the modes n >= 2 every sample belongs to the shard of its mode-1
// index; a rank gathers, multiplies and reduces only its own shards' samples,
// each shard in its own canonical chunked order, and the per-shard partials
// are exchanged (NCCL all-gather) and summed in shard order -- the oracle's
// orc_stream_consume_sharded, identical for every G dividing V.
#pragma once

#include "kernels.cuh"

namespace rocpk {

constexpr int kMaxShards = 64;

__host__ __device__ __forceinline__ int shard_of_row(int64_t i0, int64_t I1, int V) {
    return int(((i0 + 1) * V - 1) / I1);
}

// Stable partition of one stage's samples by virtual shard (one warp per job):
// the local shards' samples, in sample order shard after shard, with the
// mode-1 index and the fibre base rebased to this rank's rows.
struct ShardPartJob {
    const int32_t* idx;   // S x n_other, global 0-based (mode-1 index first)
    const int64_t* base;  // S, offsets with local strides and the global mode-1 index
    int32_t* cidx;        // out: compacted, mode-1 index - r0
    int64_t* cbase;       // out: compacted, base - r0
    int32_t* clist;       // out: original sample index of each compacted entry
    int* counts;          // out: V per-shard sample counts (all shards)
};

struct ShardPartParams {
    const ShardPartJob* jobs;
    int S, n_other, V, v0, v1;
    int64_t I1, r0;
};

__global__ void __launch_bounds__(32) k_shard_partition(const ShardPartParams p) {
    const ShardPartJob& J = p.jobs[blockIdx.x];
    const int lane = threadIdx.x;
    __shared__ int cnt[kMaxShards], run[kMaxShards];
    for (int v = lane; v < kMaxShards; v += 32) cnt[v] = 0;
    __syncwarp();
    for (int c0 = 0; c0 < p.S; c0 += 32) {
        const int c = c0 + lane;
        if (c < p.S) atomicAdd(&cnt[shard_of_row(J.idx[int64_t(c) * p.n_other], p.I1, p.V)], 1);
    }
    __syncwarp();
    if (lane == 0) {
        int acc = 0;
        for (int v = p.v0; v < p.v1; ++v) {
            run[v] = acc;
            acc += cnt[v];
        }
    }
    for (int v = lane; v < p.V; v += 32) J.counts[v] = cnt[v];
    __syncwarp();
    const unsigned lt = (1u << lane) - 1u;
    for (int c0 = 0; c0 < p.S; c0 += 32) {
        const int c = c0 + lane;
        const int v = (c < p.S) ? shard_of_row(J.idx[int64_t(c) * p.n_other], p.I1, p.V) : -1;
        const unsigned grp = __match_any_sync(0xffffffffu, v);
        const bool mine = v >= p.v0 && v < p.v1;
        if (mine) {
            const int pos = run[v] + __popc(grp & lt);
            for (int k = 0; k < p.n_other; ++k) {
                const int32_t ik = J.idx[int64_t(c) * p.n_other + k];
                J.cidx[int64_t(pos) * p.n_other + k] = (k == 0) ? int32_t(ik - p.r0) : ik;
            }
            J.cbase[pos] = J.base[c] - p.r0;
            J.clist[pos] = c;
        }
        __syncwarp();
        if (mine && (grp & lt) == 0u) run[v] += __popc(grp);  // group leader advances
        __syncwarp();
    }
}

// Per-shard partials of one stage in ONE launch: for every local shard
// segment (its samples contiguous in the compacted order) the Gram Z_v^T Z_v
// and the contraction X_v Z_v, each output by one thread in the canonical
// chunked order over the segment (32-sample fma chains from +0.0, superchunk
// and total sums in order) -- the arithmetic of k_gram / k_contract on the
// segment.  Work item = (segment, Gram output) or (segment, row, 8 outputs).
struct SegPartParams {
    const double* Z;      // n_local x R row-major (compacted order)
    const double* X;      // rows x n_local column-major
    int64_t rows;
    int R, nseg;
    int64_t blk;          // R*R + rows*R doubles per slot
    double* slots;        // nseg slots [G_v | part_v] (local; when peers == nullptr)
    int32_t off[kMaxShards + 1];  // segment starts in the compacted order
    // fused exchange over peer memory: slot v of this rank is stored straight into
    // every rank's landing buffer at global slot slot0 + v, then every block adds 1
    // to every rank's exchange counter (release, system scope)
    double* const* peers;                       // world landing bases (device array) or nullptr
    unsigned long long* const* peer_counters;   // world exchange counters
    int world;
    int slot0;
};

__device__ __forceinline__ void red_release_sys_add(unsigned long long* p, unsigned long long v) {
    asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
// Block-wide wait until an exchange counter reaches `target` (every rank's blocks arrived).
__device__ __forceinline__ void wait_counter(const unsigned long long* c, unsigned long long target) {
    if (c && threadIdx.x == 0)
        while (ld_acquire_sys_u64(c) < target) __nanosleep(64);
    __syncthreads();
}
// Every block: its stores are made visible system-wide, then +1 on each rank's counter.
__device__ __forceinline__ void arrive_all(unsigned long long* const* counters, int world) {
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0)
        for (int g = 0; g < world; ++g) red_release_sys_add(counters[g], 1ull);
}

constexpr int kSegRG = 8;  // contraction outputs per work item

__device__ __forceinline__ void seg_dot8(const double* __restrict__ X, const double* __restrict__ Z, int64_t rows,
                                         int R, int64_t i, int r0, int nr, int c0, int n, double* out) {
    double tot[kSegRG], q[kSegRG], pk[kSegRG];
#pragma unroll
    for (int j = 0; j < kSegRG; ++j) tot[j] = q[j] = 0.0;
    for (int m0 = 0; m0 < n; m0 += kSuperSamples) {
        const int m1 = min(n, m0 + kSuperSamples);
        for (int k0 = m0; k0 < m1; k0 += kChunk) {
            const int k1 = min(m1, k0 + kChunk);
#pragma unroll
            for (int j = 0; j < kSegRG; ++j) pk[j] = 0.0;
#pragma unroll 4
            for (int c = k0; c < k1; ++c) {  // unrolled: the next samples' loads overlap this fma chain
                const double x = __ldg(X + int64_t(c0 + c) * rows + i);
                const double* z = Z + int64_t(c0 + c) * R + r0;
#pragma unroll
                for (int j = 0; j < kSegRG; ++j)
                    if (j < nr) pk[j] = __fma_rn(x, __ldg(z + j), pk[j]);
            }
#pragma unroll
            for (int j = 0; j < kSegRG; ++j) q[j] = (k0 == m0) ? pk[j] : q[j] + pk[j];
        }
#pragma unroll
        for (int j = 0; j < kSegRG; ++j) tot[j] = (m0 == 0) ? q[j] : tot[j] + q[j];
    }
#pragma unroll
    for (int j = 0; j < kSegRG; ++j) out[j] = tot[j];  // the caller stores the first nr
}

__global__ void __launch_bounds__(256) k_seg_partials(const SegPartParams p) {
    const int R = p.R;
    const int64_t RR = int64_t(R) * R;
    const int ngr = (R + kSegRG - 1) / kSegRG;
    const int64_t per_seg = RR + p.rows * ngr;  // work items per segment
    const int64_t total = per_seg * p.nseg;
    for (int64_t w = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; w < total; w += int64_t(gridDim.x) * blockDim.x) {
        const int v = int(w / per_seg);
        const int64_t t = w - int64_t(v) * per_seg;
        const int c0 = p.off[v], n = p.off[v + 1] - c0;
        double* slot = p.slots + int64_t(v) * p.blk;
        if (t < RR) {  // Gram output (r1, r2), symmetric storage like k_gram
            const int r1 = int(t % R), r2 = int(t / R);
            double tot = 0.0, q = 0.0;
            for (int m0 = 0; m0 < n; m0 += kSuperSamples) {
                const int m1 = min(n, m0 + kSuperSamples);
                for (int k0 = m0; k0 < m1; k0 += kChunk) {
                    const int k1 = min(m1, k0 + kChunk);
                    double pk = 0.0;
#pragma unroll 4
                    for (int c = k0; c < k1; ++c)
                        pk = __fma_rn(__ldg(p.Z + int64_t(c0 + c) * R + r1), __ldg(p.Z + int64_t(c0 + c) * R + r2), pk);
                    q = (k0 == m0) ? pk : q + pk;
                }
                tot = (m0 == 0) ? q : tot + q;
            }
            if (p.peers) {
                for (int gr = 0; gr < p.world; ++gr) p.peers[gr][int64_t(p.slot0 + v) * p.blk + t] = tot;
            } else {
                slot[t] = tot;
            }
        } else {  // contraction outputs (i, r0 .. r0 + 7)
            const int64_t u = t - RR;
            const int64_t i = u % p.rows;
            const int g = int(u / p.rows);
            const int r0 = g * kSegRG, nr = min(kSegRG, R - r0);
            double vals[kSegRG];
            seg_dot8(p.X, p.Z, p.rows, R, i, r0, nr, c0, n, vals);
#pragma unroll
            for (int j = 0; j < kSegRG; ++j) {
                if (j >= nr) break;
                const int64_t o = RR + i * R + r0 + j;
                if (p.peers) {
                    for (int gr = 0; gr < p.world; ++gr) p.peers[gr][int64_t(p.slot0 + v) * p.blk + o] = vals[j];
                } else {
                    slot[o] = vals[j];
                }
            }
        }
    }
    if (p.peers) arrive_all(p.peer_counters, p.world);
}

// Fixed-order combine of the V exchanged partial blocks [G_v | part_v]:
// tot = blk_0 + blk_1 + ... (shard order), then out = base + tot (P + inc,
// Q + G) or out = tot.
__global__ void __launch_bounds__(256) k_shard_combine(const double* __restrict__ parts, int V, int64_t blk, int64_t RR,
                                                       const double* base_g, double* out_g, const double* base_p,
                                                       double* out_p, const unsigned long long* counter,
                                                       unsigned long long target) {
    wait_counter(counter, target);  // fused exchange: every rank's slots have landed
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < blk; e += int64_t(gridDim.x) * blockDim.x) {
        double tot = __ldcg(parts + e);
        for (int v = 1; v < V; ++v) tot = tot + __ldcg(parts + int64_t(v) * blk + e);
        if (e < RR) out_g[e] = base_g ? base_g[e] + tot : tot;
        else out_p[e - RR] = base_p ? base_p[e - RR] + tot : tot;
    }
}

// Sampled residual columns of this rank's temporal samples (warp per compacted
// column, same per-column order as k_residual), scattered to their original
// sample positions of the 2 x S column arrays (pre-zeroed).
__global__ void __launch_bounds__(256) k_shard_resid_cols(const double* __restrict__ X, int32_t I, int32_t n,
                                                          const double* __restrict__ U, const double* __restrict__ Z,
                                                          int R, const int32_t* __restrict__ clist, int32_t S,
                                                          double* cols) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int j = blockIdx.x * (blockDim.x >> 5) + warp;
    if (j >= n) return;
    double qn = 0.0, qd = 0.0;
    const double* z = Z + int64_t(j) * R;
    for (int32_t i = lane; i < I; i += 32) {
        double uz = 0.0;
        const double* u = U + int64_t(i) * R;
        for (int r = 0; r < R; ++r) uz = __fma_rn(u[r], z[r], uz);
        const double xv = X[int64_t(j) * I + i];
        const double e = xv - uz;
        qn = __fma_rn(e, e, qn);
        qd = __fma_rn(xv, xv, qd);
    }
    qn = butterfly32(qn);
    qd = butterfly32(qd);
    if (lane == 0) {
        const int c = clist[j];
        cols[c] = qn;
        cols[S + c] = qd;
    }
}

// Sum of the ranks' scattered column arrays (each column non-zero on exactly
// one rank, so the sum is exact), then the canonical hsum of both -> out[0..1].
// Fused exchange of the residual columns: this rank's 2 x S column vector into
// slot `rank` of every rank's landing buffer, then the counters.
__global__ void __launch_bounds__(256) k_shard_resid_push(const double* __restrict__ cols, int32_t S,
                                                          double* const* peers, unsigned long long* const* counters,
                                                          int world, int rank) {
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < 2 * S; e += gridDim.x * blockDim.x) {
        const double v = cols[e];
        for (int g = 0; g < world; ++g) peers[g][int64_t(rank) * 2 * S + e] = v;
    }
    arrive_all(counters, world);
}

__global__ void __launch_bounds__(256) k_shard_resid_sum(const double* __restrict__ gathered, int world, int32_t S,
                                                         double* work, double* tmp, double* out,
                                                         const unsigned long long* counter, unsigned long long target) {
    wait_counter(counter, target);
    for (int e = threadIdx.x; e < 2 * S; e += blockDim.x) {
        double v = __ldcg(gathered + e);
        for (int g = 1; g < world; ++g) v = v + __ldcg(gathered + int64_t(g) * 2 * S + e);
        work[e] = v;
    }
    __syncthreads();
    __threadfence_block();
    block_hsum_inplace(work, S, tmp);
    block_hsum_inplace(work + S, S, tmp);
    if (threadIdx.x == 0) {
        out[0] = work[0];
        out[1] = work[S];
    }
}

}  // namespace rocpk
