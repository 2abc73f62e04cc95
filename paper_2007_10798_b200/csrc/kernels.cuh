// kernels.cuh -- sm_100a kernels of the ROCP sampled-update hot path.
//
// Every floating-point result follows the canonical operation order of
// DESIGN.md section 3 so the CPU oracle (oracle/, an independent
// implementation) reproduces it bit for bit.  Compiled with -fmad=false: the
// only fused multiply-adds are the explicit __fma_rn calls below.
//
// Device layouts:
//   tensor   float64, first index fastest (reference tensor.hpp:14-16)
//   factors, P, temporal factor, Z_s: row-major (row i's R values contiguous)
//   X_s      I_n x S column-major, column c = sampled fibre c (the reference's
//            sample_unfolding output, sampling.cpp:66-77)
//   idx      S x (N-1) int32 0-based co-mode indices, increasing mode order
//   base     S int64 flat offset of each sampled fibre's first element
#pragma once

#include <cstdint>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
#include <cstdio>

namespace rocpk {

constexpr int kMaxOrder = 8;
constexpr int kChunk = 32;       // canonical sample-reduction chunk
constexpr int kSuper = 8;        // chunks per canonical superchunk (256 samples)
constexpr int kSuperSamples = kChunk * kSuper;
constexpr int kGroup = 256;      // canonical hsum group
constexpr double kGramConditionLimit = 1e12;  // reference solve.hpp:15

__device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }

// ---------------------------------------------------------------------------
// Counter RNG: Philox4x32-10, key bumped after each round (equivalent to the
// published bump-before-rounds-1..9 schedule).
__device__ __forceinline__ void philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t lo0 = 0xD2511F53u * c[0];
        const uint32_t hi0 = __umulhi(0xD2511F53u, c[0]);
        const uint32_t lo1 = 0xCD9E8D57u * c[2];
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c[2]);
        const uint32_t n0 = hi1 ^ c[1] ^ k0;
        const uint32_t n2 = hi0 ^ c[3] ^ k1;
        c[0] = n0;
        c[1] = lo1;
        c[2] = n2;
        c[3] = lo0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
}

// ---------------------------------------------------------------------------
// K1: draw (or decode explicit rows) + Eq.(1) decode + fibre base offset.
// Replaces draw_samples / SampleIndexSet::from_rows / decode_index
// (sampling.cpp:11-55, tensor.cpp:96-109).  One launch serves any number of
// jobs (blockIdx.y = job), so every draw of a whole stream window is one
// launch: sample indices never depend on factors.
struct DrawJob {
    uint64_t seed;
    const uint64_t* seed_ptr;      // if set, the seed is read from device memory
    const uint32_t* batch_ptr;     // if set, batch = *batch_ptr + batch (window offset)
    uint32_t batch, iteration, mode;  // mode 1-based
    int n_other;
    int32_t s;
    int64_t co;                    // co-domain size
    int64_t ext[kMaxOrder];        // co-mode extents, increasing mode order
    int64_t tstride[kMaxOrder];    // tensor strides of the co-modes
    const int64_t* in_rows;        // explicit 1-based rows (replay) or nullptr (draw)
    int64_t* rows;                 // optional 1-based output
    int32_t* idx;                  // s x n_other, 0-based
    int64_t* base;                 // s
};

__global__ void __launch_bounds__(128) k_draw(const DrawJob* __restrict__ jobs) {
    const DrawJob& J = jobs[blockIdx.y];
    const uint64_t seed = J.seed_ptr ? *J.seed_ptr : J.seed;
    const uint32_t batch = J.batch_ptr ? *J.batch_ptr + J.batch : J.batch;
    for (int32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < J.s; c += gridDim.x * blockDim.x) {
        int64_t j0;
        if (J.in_rows) {
            j0 = J.in_rows[c] - 1;
        } else {
            uint32_t ctr[4] = {uint32_t(c), J.mode, J.iteration, batch};
            philox4x32_10(ctr, uint32_t(seed), uint32_t(seed >> 32));
            const uint64_t u = uint64_t(ctr[0]) | (uint64_t(ctr[1]) << 32);
            j0 = int64_t(__umul64hi(u, uint64_t(J.co)));
        }
        if (J.rows) J.rows[c] = j0 + 1;
        int64_t rem = j0, base = 0;
        for (int k = 0; k < J.n_other; ++k) {
            const int64_t e = J.ext[k];
            const int64_t q = rem / e;
            const int64_t ik = rem - q * e;
            rem = q;
            J.idx[int64_t(c) * J.n_other + k] = int32_t(ik);
            base += ik * J.tstride[k];
        }
        J.base[c] = base;
    }
}

// Window prologue in one launch: draw seed, first batch id, and (overlapped
// gather) the per-job unit counters.
__global__ void k_window_setup(uint64_t* seed_p, uint64_t seed, uint32_t* batch_p, uint32_t batch,
                               unsigned* done, int ndone) {
    if (threadIdx.x == 0) {
        *seed_p = seed;
        *batch_p = batch;
    }
    for (int i = threadIdx.x; i < ndone; i += blockDim.x) done[i] = 0u;
}
__global__ void k_set_u64(uint64_t* p, uint64_t v) { *p = v; }
__global__ void k_set_u32(uint32_t* p, uint32_t v) { *p = v; }
__global__ void k_set_i32(int* p, int n, int v) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) p[i] = v;
}

// ---------------------------------------------------------------------------
// K2: sampled-fibre gather, X_s(i, c) = T[base_c + i * ms].  Replaces
// sample_unfolding (sampling.cpp:57-79).  HBM-bound: the whole stream
// window's gathers (every batch, every stage) are one launch over a flat tile
// list, each tile kGatherTile consecutive elements of one job with i fastest:
// coalesced writes, coalesced reads along the contiguous mode-1 fibres, and
// kGatherUnroll independent loads in flight per thread for the strided modes
// (each element its own 32-B sector).
struct GatherJob {
    const double* t;
    const int64_t* base;
    int64_t ms;  // mode stride
    int32_t I;   // fibre length (I_n)
    int32_t s;
    double* out;
    int tiled;   // 0: I x s column-major; 1: row-tiled (see xs_offset)
    const int32_t* perm;  // row-tiled strided jobs: samples in fibre-base order (or nullptr)
    // overlapped gather (gather_kernel.cuh): tensor-map view + 1 of this strided job (0 = LSU
    // loads), box length along the fibre, and the job's slab offset from the window start
    int32_t tmap1;
    int32_t tlen;
    int64_t toff;
};

// Row-tiled X_s layout (stream windows): rows in tiles of 32, each tile's
// 32 x S block stored column after column, so the (32-row tile, 256-sample
// superchunk) operand of the contraction is ONE contiguous 64 KB block (a
// single TMA bulk copy).  Element (i, c) of an I x S operand:
__host__ __device__ __forceinline__ int64_t xs_offset(int64_t i, int64_t c, int64_t S) {
    return ((i >> 5) * S + c) * 32 + (i & 31);
}
__host__ __device__ __forceinline__ int64_t xs_size(int64_t I, int64_t S) { return ((I + 31) / 32) * 32 * S; }
struct GatherTile {
    int32_t job;
    uint32_t e0;
};
constexpr int kGatherThreads = 256;
constexpr int kGatherUnroll = 8;
constexpr int kGatherTile = kGatherThreads * kGatherUnroll;

// Sorted tiles (J.perm): tile.e0 = group << 16 | i-block; warp w takes the
// (8 group + w)-th sample in fibre-base order and 8 x 32 consecutive fibre
// elements, so the 8 warps of a block read neighbouring fibres at the same
// element (shared DRAM pages) while each warp writes one contiguous tiled run.
constexpr int kSortedGroup = kGatherThreads / 32;                 // samples per sorted tile
constexpr int kSortedSpan = 32 * kGatherUnroll;                   // fibre elements per sorted tile

__global__ void __launch_bounds__(kGatherThreads) k_gather(const GatherJob* __restrict__ jobs,
                                                           const GatherTile* __restrict__ tiles) {
    const GatherTile tile = tiles[blockIdx.x];
    const GatherJob& J = jobs[tile.job];
    if (J.perm) {
        const int q = int(tile.e0 >> 16) * kSortedGroup + int(threadIdx.x >> 5);
        if (q >= J.s) return;
        const int c = __ldg(J.perm + q);
        const double* a = J.t + __ldg(J.base + c);
        const int i0 = int(tile.e0 & 0xffffu) * kSortedSpan + int(threadIdx.x & 31);
        double v[kGatherUnroll];
#pragma unroll
        for (int u = 0; u < kGatherUnroll; ++u) {
            const int i = i0 + 32 * u;
            if (i < J.I) asm volatile("ld.global.cs.L2::64B.f64 %0, [%1];" : "=d"(v[u]) : "l"(a + int64_t(i) * J.ms));
        }
#pragma unroll
        for (int u = 0; u < kGatherUnroll; ++u) {
            const int i = i0 + 32 * u;
            if (i < J.I) J.out[xs_offset(i, c, J.s)] = v[u];
        }
        return;
    }
    const uint32_t total = uint32_t(J.I) * uint32_t(J.s);
    const double* __restrict__ t = J.t;
    const int64_t* __restrict__ base = J.base;
    const int64_t ms = J.ms;
    const uint32_t I = uint32_t(J.I);
    double v[kGatherUnroll];
#pragma unroll
    for (int u = 0; u < kGatherUnroll; ++u) {
        const uint32_t e = tile.e0 + u * kGatherThreads + threadIdx.x;
        if (e < total) {
            const uint32_t c = e / I;
            const uint32_t i = e - c * I;
            const double* a = t + __ldg(base + c) + int64_t(i) * ms;
            if (ms == 1) {
                v[u] = __ldcs(a);  // contiguous mode-1 fibre: full-line fetches are all useful
            } else {
                // isolated strided element: ask L2 for a 64-byte fill instead of a full
                // 128-byte line (halves DRAM bytes per element; profiles/README.md)
                asm volatile("ld.global.cs.L2::64B.f64 %0, [%1];" : "=d"(v[u]) : "l"(a));
            }
        }
    }
#pragma unroll
    for (int u = 0; u < kGatherUnroll; ++u) {
        const uint32_t e = tile.e0 + u * kGatherThreads + threadIdx.x;
        if (e < total) {
            if (J.tiled) {
                const uint32_t c = e / I;
                const uint32_t i = e - c * I;
                J.out[xs_offset(i, c, J.s)] = v[u];
            } else {
                J.out[e] = v[u];
            }
        }
    }
}

// Samples of one stage in fibre-base order (bitonic sort in shared memory,
// s <= 2048): the sorted gather's visiting order only -- results are unchanged.
struct SortJob {
    const int64_t* base;
    int32_t* perm;
    int32_t s;
};
constexpr int kSortMax = 2048;

__global__ void __launch_bounds__(1024) k_sort_by_base(const SortJob* __restrict__ jobs) {
    const SortJob J = jobs[blockIdx.x];
    __shared__ int64_t key[kSortMax];
    __shared__ int32_t val[kSortMax];
    int P = 1;
    while (P < J.s) P <<= 1;
    for (int i = threadIdx.x; i < P; i += blockDim.x) {
        key[i] = (i < J.s) ? J.base[i] : 0x7fffffffffffffffLL;
        val[i] = i;
    }
    __syncthreads();
    for (int k = 2; k <= P; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < P; i += blockDim.x) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const bool up = (i & k) == 0;
                    const bool gt = key[i] > key[ixj] || (key[i] == key[ixj] && val[i] > val[ixj]);
                    if (gt == up) {
                        const int64_t tk = key[i];
                        key[i] = key[ixj];
                        key[ixj] = tk;
                        const int32_t tv = val[i];
                        val[i] = val[ixj];
                        val[ixj] = tv;
                    }
                }
            }
            __syncthreads();
        }
    for (int i = threadIdx.x; i < J.s; i += blockDim.x) J.perm[i] = val[i];
}

// ---------------------------------------------------------------------------
// K3: sampled Khatri-Rao, Z(c, r) = 1.0 * F_0(i_0(c), r) * F_1(...) * ...
// factors in factors_excluding order (decreasing mode), left to right exactly
// as sampled_khatri_rao (sampling.cpp:90-103).  Factors row-major.
struct SkrJob {
    const int32_t* idx;
    int n_other;
    int32_t s;
    int R;
    const double* f[kMaxOrder];
    double* z;  // s x R row-major
};

__global__ void k_skr(const SkrJob J) {
    const int32_t total = J.s * J.R;
    for (int32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
        const int32_t c = e / J.R;
        const int32_t r = e - c * J.R;
        double z = 1.0;
        for (int l = 0; l < J.n_other; ++l) {
            const int k = J.n_other - 1 - l;
            const int32_t i = J.idx[int64_t(c) * J.n_other + k];
            z = z * J.f[l][int64_t(i) * J.R + r];
        }
        J.z[e] = z;
    }
}

// ---------------------------------------------------------------------------
// Last-block combine helper: returns true in exactly one block, after all
// blocks' global writes are visible.  Resets the counter for reuse (graph
// safe, one kernel at a time per counter).
__device__ __forceinline__ bool last_block_arrive(unsigned int* counter) {
    __shared__ bool is_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned int prev = atomicAdd(counter, 1u);
        is_last = (prev == gridDim.x * gridDim.y * gridDim.z - 1);
        if (is_last) *counter = 0u;
    }
    __syncthreads();
    if (is_last) __threadfence();
    return is_last;
}

// ---------------------------------------------------------------------------
// K4a: Gram G = Z^T Z (solve.cpp:41, rocp.cpp:108) in the canonical chunked
// order.  One block per 32-sample chunk writes its R x R chunk partials; the
// last block of each superchunk (8 chunks) sums them in increasing chunk order
// into the superchunk partial, and the last of those blocks sums the
// superchunk partials in order and optionally accumulates (Q + G,
// rocp.cpp:108).  Every load of a batch of outputs is issued before its sums
// (a single block combining every chunk partial with one load round trip per
// superchunk took 83 us at R = 50, S = 1957).
__device__ __forceinline__ bool last_arrive_of(unsigned int* counter, unsigned int expected);

__global__ void __launch_bounds__(256) k_gram(const double* __restrict__ Z, int32_t s, int R,
                                              double* __restrict__ partial, double* __restrict__ spart,
                                              unsigned int* counter, unsigned int* sc_counters,
                                              const double* acc_base, double* __restrict__ out) {
    extern __shared__ double zs[];  // kChunk x R
    const int k = blockIdx.x;
    const int c0 = k * kChunk;
    const int cn = min(kChunk, s - c0);
    for (int t = threadIdx.x; t < kChunk * R; t += blockDim.x) {
        const int cc = t / R;
        zs[t] = (cc < cn) ? Z[int64_t(c0) * R + t] : 0.0;
    }
    __syncthreads();
    const int RR = R * R;
    for (int p = threadIdx.x; p < RR; p += blockDim.x) {
        const int r1 = p % R, r2 = p / R;
        double acc = 0.0;
        for (int cc = 0; cc < cn; ++cc) acc = __fma_rn(zs[cc * R + r1], zs[cc * R + r2], acc);
        partial[int64_t(k) * RR + p] = acc;
    }
    const int nk = gridDim.x;
    const int msup = k / kSuper, m0 = msup * kSuper, m1 = min(nk, m0 + kSuper);
    if (!last_arrive_of(sc_counters + msup, unsigned(m1 - m0))) return;
    constexpr int kOB = 4;  // outputs per batch of loads
    for (int pb = threadIdx.x; pb < RR; pb += kOB * blockDim.x) {
        double pk[kOB][kSuper];
#pragma unroll
        for (int o = 0; o < kOB; ++o) {
            const int p = pb + o * int(blockDim.x);
#pragma unroll
            for (int u = 0; u < kSuper; ++u)
                pk[o][u] = (p < RR && m0 + u < m1) ? __ldcg(partial + int64_t(m0 + u) * RR + p) : 0.0;
        }
#pragma unroll
        for (int o = 0; o < kOB; ++o) {
            const int p = pb + o * int(blockDim.x);
            if (p < RR) {
                double q = pk[o][0];
#pragma unroll
                for (int u = 1; u < kSuper; ++u)
                    if (m0 + u < m1) q = q + pk[o][u];
                spart[int64_t(msup) * RR + p] = q;
            }
        }
    }
    const int nsup = (nk + kSuper - 1) / kSuper;
    if (!last_arrive_of(counter, unsigned(nsup))) return;
    for (int pb = threadIdx.x; pb < RR; pb += kOB * blockDim.x) {
        double sv[kOB][kSuper], bv[kOB];
#pragma unroll
        for (int o = 0; o < kOB; ++o) {
            const int p = pb + o * int(blockDim.x);
#pragma unroll
            for (int u = 0; u < kSuper; ++u) sv[o][u] = (p < RR && u < nsup) ? __ldcg(spart + int64_t(u) * RR + p) : 0.0;
            bv[o] = (p < RR && acc_base) ? acc_base[p] : 0.0;
        }
#pragma unroll
        for (int o = 0; o < kOB; ++o) {
            const int p = pb + o * int(blockDim.x);
            if (p < RR) {
                double tot = sv[o][0];
#pragma unroll
                for (int u = 1; u < kSuper; ++u)
                    if (u < nsup) tot = tot + sv[o][u];
                for (int u = kSuper; u < nsup; ++u) tot = tot + __ldcg(spart + int64_t(u) * RR + p);
                out[p] = acc_base ? bv[o] + tot : tot;  // column-major == row-major (symmetric)
            }
        }
    }
}

// ---------------------------------------------------------------------------
// K4b: skinny contraction out = X_s Z (I x S times S x R; solve.cpp:42,
// rocp.cpp:107), canonical two-level order, optionally out = base + X_s Z.
// Block = (32-row tile, one 256-sample superchunk): the X_s tile (32 x 256)
// and the Z tile (256 x R) are staged in shared memory with cp.async (all
// loads in flight at once: one memory round trip per block), then each thread
// (row lane, r-group of RB outputs) runs the 8 chunk fma chains from shared
// memory.  With more than one superchunk, partials go to `partial` and the
// last block of each row tile combines them in superchunk order.
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::); }

constexpr int kRowTile = 32;

__device__ __forceinline__ bool last_arrive_of(unsigned int* counter, unsigned int expected) {
    __shared__ bool is_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned int prev = atomicAdd(counter, 1u);
        is_last = (prev == expected - 1);
        if (is_last) *counter = 0u;
    }
    __syncthreads();
    if (is_last) __threadfence();
    return is_last;
}

template <int RB>
__global__ void __launch_bounds__(256) k_contract(const double* __restrict__ X, int32_t I, int32_t S,
                                                  const double* __restrict__ Z, int R,
                                                  const double* base, double* out,
                                                  double* __restrict__ partial,
                                                  unsigned int* __restrict__ counters, int tiled) {
    extern __shared__ double sm[];
    const int RP = int(blockDim.x >> 5) * RB;    // R padded to the r-groups (zero columns)
    double* xs = sm;                            // [256][32]
    double* zs = sm + kSuperSamples * kRowTile;  // [256][RP]
    const int tile = blockIdx.x, m = blockIdx.y, nsuper = gridDim.y;
    const int i0 = tile * kRowTile;
    const int c0 = m * kSuperSamples;
    const int cn = min(kSuperSamples, S - c0);
    const int rows = min(kRowTile, I - i0);
    const int tid = threadIdx.x;
    for (int e = tid; e < kRowTile * cn; e += blockDim.x) {
        const int c = e >> 5, r = e & 31;
        if (r < rows) cp_async8(xs + e, X + (tiled ? xs_offset(i0 + r, c0 + c, S) : int64_t(c0 + c) * I + i0 + r));
        else xs[e] = 0.0;
    }
    for (int e = tid; e < cn * RP; e += blockDim.x) {
        const int c = e / RP, r = e - c * RP;
        if (r < R) cp_async8(zs + e, Z + int64_t(c0 + c) * R + r);
        else zs[e] = 0.0;
    }
    cp_async_wait_all();
    __syncthreads();
    const int lane = tid & 31, rg = tid >> 5;
    const int r0 = rg * RB;
    double q[RB];
#pragma unroll
    for (int j = 0; j < RB; ++j) q[j] = 0.0;
    for (int k = 0; k < kSuper; ++k) {
        const int cc0 = k * kChunk;
        if (cc0 >= cn) break;
        const int ccn = min(kChunk, cn - cc0);
        double p[RB];
#pragma unroll
        for (int j = 0; j < RB; ++j) p[j] = 0.0;
        if (ccn == kChunk) {
#pragma unroll 8
            for (int cc = 0; cc < kChunk; ++cc) {
                const double x = xs[(cc0 + cc) * kRowTile + lane];
                const double* zr = zs + (cc0 + cc) * RP + r0;
#pragma unroll
                for (int j = 0; j < RB; ++j) p[j] = __fma_rn(x, zr[j], p[j]);
            }
        } else {
            for (int cc = 0; cc < ccn; ++cc) {
                const double x = xs[(cc0 + cc) * kRowTile + lane];
                const double* zr = zs + (cc0 + cc) * RP + r0;
#pragma unroll
                for (int j = 0; j < RB; ++j) p[j] = __fma_rn(x, zr[j], p[j]);
            }
        }
#pragma unroll
        for (int j = 0; j < RB; ++j) q[j] = (k == 0) ? p[j] : q[j] + p[j];
    }
    const int i = i0 + lane;
    const bool live = lane < rows;
    if (nsuper == 1) {
        if (live) {
#pragma unroll
            for (int j = 0; j < RB; ++j) {
                if (r0 + j >= R) break;
                const int64_t o = int64_t(i) * R + r0 + j;
                out[o] = base ? base[o] + q[j] : q[j];
            }
        }
        return;
    }
    if (live) {
#pragma unroll
        for (int j = 0; j < RB; ++j)
            if (r0 + j < R) partial[(int64_t(m) * I + i) * R + r0 + j] = q[j];
    }
    if (!last_arrive_of(counters + tile, unsigned(nsuper))) return;
    if (live) {
#pragma unroll
        for (int j = 0; j < RB; ++j) {
            if (r0 + j >= R) break;
            const int64_t o = int64_t(i) * R + r0 + j;
            double tot = __ldcg(partial + o);
            for (int mm = 1; mm < nsuper; ++mm) tot = tot + __ldcg(partial + int64_t(mm) * I * R + o);
            out[o] = base ? base[o] + tot : tot;
        }
    }
}

// Contraction for R <= 32 (primitives, cprand sweeps, the sharded stream's owned
// mode): same canonical order as k_contract, but warp w of a 256-thread block
// forms chunk w of the (32-row tile, superchunk) item with fp64 mma.sync (4 x
// RPAD/8 accumulator tiles) and the 8 chunk partials are summed left to right
// through shared memory.  k_contract used 32 * ceil(R/10) threads per item,
// each walking all 256 samples (configs[1]: 40 us per mode-1 contraction).
template <int RPAD>
__global__ void __launch_bounds__(256) k_contract_chunks(const double* __restrict__ X, int32_t I, int32_t S,
                                                         const double* __restrict__ Z, int R,
                                                         const double* base, double* out,
                                                         double* __restrict__ partial,
                                                         unsigned int* __restrict__ counters, int tiled) {
    extern __shared__ double sm[];
    double* xs = sm;                                 // [256][32]
    double* zs = sm + kSuperSamples * kRowTile;      // [256][RPAD]
    double* cps = zs + kSuperSamples * RPAD;         // [8][RPAD][32]
    const int tile = blockIdx.x, m = blockIdx.y, nsuper = gridDim.y;
    const int i0 = tile * kRowTile;
    const int c0 = m * kSuperSamples;
    const int cn = min(kSuperSamples, S - c0);
    const int rows = min(kRowTile, I - i0);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int e = tid; e < kRowTile * cn; e += blockDim.x) {
        const int c = e >> 5, r = e & 31;
        if (r < rows) cp_async8(xs + e, X + (tiled ? xs_offset(i0 + r, c0 + c, S) : int64_t(c0 + c) * I + i0 + r));
        else xs[e] = 0.0;
    }
    for (int e = tid; e < cn * RPAD; e += blockDim.x) {
        const int c = e / RPAD, r = e - c * RPAD;
        if (r < R) cp_async8(zs + e, Z + int64_t(c0 + c) * R + r);
        else zs[e] = 0.0;
    }
    cp_async_wait_all();
    __syncthreads();
    const int nk = (cn + kChunk - 1) / kChunk;
    if (warp < nk) {  // chunk `warp`: fma chain from +0.0 over its samples, increasing order, on the
                      // fp64 tensor cores (mma.sync m8n8k4 rounds like that chain; samples past the
                      // chunk enter as 0 x 0)
        const int cc0 = warp * kChunk, ccn = min(kChunk, cn - cc0);
        constexpr int NT = RPAD / 8;
        const int q4 = lane & 3, rr = lane >> 2;
        double acc[4][NT][2];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int n = 0; n < NT; ++n) acc[a][n][0] = acc[a][n][1] = 0.0;
        for (int k0 = 0; k0 < ccn; k0 += 4) {
            const bool valid = k0 + q4 < ccn;
            const int smp = cc0 + k0 + q4;
            double fa[4], fb[NT];
#pragma unroll
            for (int a = 0; a < 4; ++a) fa[a] = valid ? xs[smp * kRowTile + a * 8 + rr] : 0.0;
#pragma unroll
            for (int n = 0; n < NT; ++n) fb[n] = valid ? zs[smp * RPAD + n * 8 + rr] : 0.0;
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int n = 0; n < NT; ++n)
                    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                                 : "+d"(acc[a][n][0]), "+d"(acc[a][n][1])
                                 : "d"(fa[a]), "d"(fb[n]));
        }
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int n = 0; n < NT; ++n)
#pragma unroll
                for (int e = 0; e < 2; ++e)
                    cps[(warp * RPAD + n * 8 + 2 * q4 + e) * kRowTile + a * 8 + rr] = acc[a][n][e];
    }
    __syncthreads();
    const bool split = nsuper > 1;
    for (int e = tid; e < RPAD * kRowTile; e += blockDim.x) {
        const int r = e >> 5, l = e & 31;
        if (r >= R || l >= rows) continue;
        double q = cps[r * kRowTile + l];  // superchunk partial: chunk partials left to right
        for (int k = 1; k < nk; ++k) q = q + cps[(k * RPAD + r) * kRowTile + l];
        const int64_t o = int64_t(i0 + l) * R + r;
        if (split) partial[int64_t(m) * I * R + o] = q;
        else out[o] = base ? base[o] + q : q;
    }
    if (!split) return;
    if (!last_arrive_of(counters + tile, unsigned(nsuper))) return;
    for (int e = tid; e < RPAD * kRowTile; e += blockDim.x) {
        const int r = e >> 5, l = e & 31;
        if (r >= R || l >= rows) continue;
        const int64_t o = int64_t(i0 + l) * R + r;
        double tot = __ldcg(partial + o);
        for (int mm = 1; mm < nsuper; ++mm) tot = tot + __ldcg(partial + int64_t(mm) * I * R + o);
        out[o] = base ? base[o] + tot : tot;
    }
}

// ---------------------------------------------------------------------------
// Random-access ceiling probe (measurement only; no reference counterpart): every
// thread issues kProbeILP independent 8-byte loads at hashed offsets of x, the
// access pattern of the strided gather (each element its own DRAM page), so
// bench.py can state the gather against the device's isolated-read rate.
constexpr int kProbeILP = 8;
__global__ void __launch_bounds__(256) k_probe_random_reads(const double* __restrict__ x, uint64_t n,
                                                           int64_t reads, uint64_t seed, double* sink) {
    double acc = 0.0;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x * kProbeILP;
    for (int64_t base = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) * kProbeILP; base < reads; base += stride) {
        double v[kProbeILP];
#pragma unroll
        for (int u = 0; u < kProbeILP; ++u) {
            uint64_t h = seed + uint64_t(base + u) * 0x9E3779B97F4A7C15ull;  // splitmix64
            h = (h ^ (h >> 30)) * 0xBF58476D1CE4E5B9ull;
            h = (h ^ (h >> 27)) * 0x94D049BB133111EBull;
            h ^= h >> 31;
            v[u] = (base + u < reads) ? __ldcs(x + __umul64hi(h, n)) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kProbeILP; ++u) acc = acc + v[u];
    }
    if (acc == 1.2345678e300) *sink = acc;  // keeps the loads
}

// ---------------------------------------------------------------------------
// solve_gram's regularisation decision (solve.cpp:17-33), canonical form
// (oracle certificate / jacobi_eigen / decide_gram).  The
// reference decides from exact eigenvalues: zero solution if lambda_max <= 0,
// regularise if lambda_min <= 0 or lambda_max / lambda_min > 1e12.  Certificate
// first: dmax / dmin <= kappa (pivots of an SPD matrix lie in [lambda_min,
// lambda_max]) and maxdiag tau / R <= kappa <= |G|_inf tau with tau = tr(G^-1)
// from the explicit inverse the row solves use anyway.  Certainly above 4e12 ->
// regularise; certainly below 2.5e11 -> not; a non-positive max diagonal or
// pivot, or the band in between -> exact eigenvalues by the deterministic
// cyclic Jacobi method.
constexpr double kCertRegAbove = 4e12;
constexpr double kCertNoRegBelow = 2.5e11;
constexpr int kDecNoReg = 0, kDecReg = 1, kDecExact = 2;

__device__ __forceinline__ double butterfly32(double q) {
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) q = q + __shfl_xor_sync(0xffffffffu, q, off);
    return q;
}

// max(a, b) of the canonical row maxima: (b > a) ? b : a.
__device__ __forceinline__ double max_of(double a, double b) { return (b > a) ? b : a; }
__device__ __forceinline__ double butterfly_max32(double v) {
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) v = max_of(v, __shfl_xor_sync(0xffffffffu, v, off));
    return v;
}

// |G|_inf (max absolute row sum; row sums in column order), one warp; a(i,j) at G[i + j*ldg].
// The loads of 8 columns are issued before their adds (the sum is the only dependency).
__device__ __noinline__ double gram_inf_norm_warp(const double* G, int ldg, int R) {
    const int lane = threadIdx.x & 31;
    double r0 = 0.0, r1 = 0.0;
    for (int j0 = 0; j0 < R; j0 += 8) {
        double v0[8], v1[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int j = j0 + u;
            v0[u] = (j < R && lane < R) ? fabs(G[lane + j * ldg]) : 0.0;
            v1[u] = (j < R && lane + 32 < R) ? fabs(G[lane + 32 + j * ldg]) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (j0 + u < R) {
                r0 = r0 + v0[u];
                r1 = r1 + v1[u];
            }
    }
    double v = (lane < R) ? r0 : 0.0;
    if (lane + 32 < R) v = max_of(v, r1);
    return butterfly_max32(v);
}

// Device-wide decision statistics (rocp_decision_stats): [0] no-reg, [1] reg, [2] exact
// eigenvalues, [3] decisions that reached the tau bounds (the pivot ratio did not settle
// them).  One atomic per solve, off the chain's critical path.
__device__ unsigned long long g_dec_paths[4];
__device__ __forceinline__ void count_decision(int final_path, bool used_tau) {
    atomicAdd(&g_dec_paths[final_path], 1ull);
    if (used_tau) atomicAdd(&g_dec_paths[3], 1ull);
}

// The certificate (oracle certificate): pivot ratio, then the tau bounds, as products (no
// quotient on the finisher's chain).  *used_tau: whether the tau bounds were reached.
__device__ __forceinline__ int gram_certificate(double maxdiag, double gnorm, double dmin, double dmax, double tau,
                                                int R, bool* used_tau) {
    *used_tau = false;
    if (!(maxdiag > 0.0) || !(dmin > 0.0)) return kDecExact;
    if (dmax > kCertRegAbove * dmin) return kDecReg;
    *used_tau = true;
    if (maxdiag * tau > kCertRegAbove * double(R)) return kDecReg;
    if (gnorm * tau <= kCertNoRegBelow) return kDecNoReg;
    return kDecExact;
}


// ---------------------------------------------------------------------------
// G^-1 by the symmetric sweep (Gauss-Jordan without pivoting, oracle
// gram_sweep).  For k = 0..R-1, with c = column k of the working matrix A (A = G +
// lambda I at the start) and r = 1 / c_k (0 when |c_k| <= DBL_MIN):
//   A(i, k) = c_i r (i != k),  A(k, k) = -r,
//   A(k, j) = fma(c_j, r, +0) (j != k),
//   A(i, j) = fma(-(c_i r), c_j, A(i, j)) (i, j != k);
// then G^-1 = -A.  The pivots d_k = c_k are the LDL^T pivots of G (Schur complements)
// and feed the regularisation certificate.  One elimination, no separate triangular
// inverse: the critical path per step is one reciprocal, one multiply and one fma.

// The sweep by a whole block on the LOWER triangle (the canonical form, oracle gram_sweep:
// entries (i, j), i >= j, each step reading column k through symmetry, c_x = A(x, k) for
// x >= k and A(k, x) for x < k; G^-1 symmetric by construction).  R <= 64 with
// R (R + 1) / 2 <= EPT * (blockDim - 32): thread t owns the lower entries t, t + nt, ...
// (column by column; pairs[e] = (i << 8) | j when the caller has the table) in registers.
// Column k + 1 is published in cbuf (2 x 64, by step parity) by the owners of its entries as
// they update them, so a step is one block barrier, one reciprocal (formed redundantly by
// every thread) and one fma per entry.  Writes G^-1 to gi (both triangles; gi[i * R + j] =
// G^-1(i, j)); thread 0 gets min_k d_k, max_k d_k in *dmin, *dmax.  Block-uniform call.
template <int EPT>
__device__ __noinline__ void sweep_block(const double* G, double lambda, int R, const unsigned short* pairs,
                                         double* cbuf, double* gi, double* dmin, double* dmax) {
    // warps 0 .. nw-2 (blockDim - 32 threads, named barrier 1); the last warp is free for
    // the caller's independent work and joins at the final block barrier
    const int tid = threadIdx.x, nt = blockDim.x - 32;
    const int np = R * (R + 1) / 2;
    if (tid < nt) {
        double a[EPT];
        int ii[EPT], jj[EPT];
#pragma unroll
        for (int q = 0; q < EPT; ++q) {
            const int e = tid + q * nt;
            int i = 0, j = -1;  // j = -1: no entry
            if (e < np) {
                if (pairs) {
                    i = pairs[e] >> 8;
                    j = pairs[e] & 0xff;
                } else {  // lower entry e, column by column: column j holds R - j entries
                    int rem = e;
                    j = 0;
                    while (rem >= R - j) {
                        rem -= R - j;
                        ++j;
                    }
                    i = j + rem;
                }
            }
            ii[q] = i;
            jj[q] = j;
            const double g = (j >= 0) ? G[i + j * R] : 0.0;
            a[q] = (i == j) ? g + lambda : g;
            if (j == 0) cbuf[i] = a[q];
        }
        asm volatile("bar.sync 1, %0;" ::"r"(nt) : "memory");
        double lo = 0.0, hi = 0.0;
        for (int k = 0; k < R; ++k) {
            const double* c = cbuf + (k & 1) * 64;
            double* cn = cbuf + ((k + 1) & 1) * 64;
            const double d = c[k];
            if (k == 0) lo = hi = d;
            if (d < lo) lo = d;
            if (d > hi) hi = d;
            const double r = (fabs(d) > 2.2250738585072014e-308) ? 1.0 / d : 0.0;
#pragma unroll
            for (int q = 0; q < EPT; ++q) {
                const int i = ii[q], j = jj[q];
                const double ci = c[i], cj = c[j < 0 ? 0 : j];
                const double l = ci * r;
                const double ov = __fma_rn(-l, cj, a[q]);
                const double pv = __fma_rn(cj, r, 0.0);
                const bool jk = j == k, ik = i == k;
                const double v = jk ? (ik ? -r : l) : (ik ? pv : ov);
                a[q] = v;
                // column k + 1: below the diagonal (and the diagonal) from column k + 1, above it
                // through row k + 1 (one predicated store)
                const int tgt = (j == k + 1) ? i : ((i == k + 1 && j >= 0) ? j : -1);
                if (tgt >= 0) cn[tgt] = v;
            }
            asm volatile("bar.sync 1, %0;" ::"r"(nt) : "memory");
        }
#pragma unroll
        for (int q = 0; q < EPT; ++q)
            if (jj[q] >= 0) {
                gi[ii[q] * R + jj[q]] = -a[q];
                gi[jj[q] * R + ii[q]] = -a[q];
            }
        if (tid == 0) {
            *dmin = lo;
            *dmax = hi;
        }
    }
    __syncthreads();
}

// Deterministic parallel (round-robin) Jacobi eigenvalue extremes of a symmetric
// R x R matrix (a(i,j) at a[i + j*lda], destroyed) by a whole block: the oracle's
// jacobi_eigen round for round -- the pairs of a round (circle method) get their
// (t, c, s) from one thread each, then every 2 x 2 block (P, Q), P <= Q, is
// transformed by one thread (rows by pair P, then columns by pair Q, mirrored), in
// place: a block is the only reader of its own entries in a round.  prm: 4 * 32
// doubles of shared scratch, flag: a shared int.  Block-uniform call.  Rare path
// (the certificate settles every Gram of the BASELINE configs but a few of C5's).
__device__ __forceinline__ void jacobi_pair(int r, int k, int n, int* p, int* q) {
    int a, b;
    if (k == 0) {
        a = r;
        b = n - 1;
    } else {
        a = (r + k) % (n - 1);
        b = (r - k + (n - 1)) % (n - 1);
    }
    *p = min(a, b);
    *q = max(a, b);
}

__device__ __noinline__ void jacobi_eigen_block(double* a, int lda, int R, double* prm, int* flag, double* lo,
                                                double* hi) {
    const int tid = threadIdx.x, nt = blockDim.x;
    const int n = R + (R & 1), np = n / 2;
    for (int sweep = 0; sweep < 64 && R > 1; ++sweep) {
        if (tid == 0) *flag = 0;
        __syncthreads();
        for (int r = 0; r + 1 < n; ++r) {
            for (int k = tid; k < np; k += nt) {
                int p, q;
                jacobi_pair(r, k, n, &p, &q);
                double rotk = 0.0, c = 1.0, sn = 0.0, t = 0.0;
                if (q < R) {
                    const double apq = a[p + q * lda], app = a[p + p * lda], aqq = a[q + q * lda];
                    const double thr = 1e-9 * sqrt(fabs(app) * fabs(aqq));  // oracle kJacobiTol
                    if (fabs(apq) > thr) {
                        const double dl = aqq - app, h = sqrt(dl * dl + 4.0 * (apq * apq));
                        const double sg = ((dl >= 0.0) == (apq >= 0.0)) ? 1.0 : -1.0;
                        t = sg * (2.0 * fabs(apq)) / (fabs(dl) + h);
                        c = 1.0 / sqrt(t * t + 1.0);
                        sn = t * c;
                        rotk = 1.0;
                        *flag = 1;
                    }
                }
                prm[4 * k + 0] = c;
                prm[4 * k + 1] = sn;
                prm[4 * k + 2] = t;
                prm[4 * k + 3] = rotk;
            }
            __syncthreads();
            for (int idx = tid; idx < np * np; idx += nt) {
                const int P = idx / np, Q = idx - (idx / np) * np;
                if (Q < P) continue;
                const bool rP = prm[4 * P + 3] != 0.0, rQ = prm[4 * Q + 3] != 0.0;
                int p, q, u, v;
                jacobi_pair(r, P, n, &p, &q);
                jacobi_pair(r, Q, n, &u, &v);
                if (P == Q) {
                    if (!rP) continue;
                    const double apq = a[p + q * lda], app = a[p + p * lda], aqq = a[q + q * lda];
                    const double t = prm[4 * P + 2];
                    a[p + p * lda] = app - t * apq;
                    a[q + q * lda] = aqq + t * apq;
                    a[p + q * lda] = 0.0;
                    a[q + p * lda] = 0.0;
                    continue;
                }
                if (!rP && !rQ) continue;
                const bool qv = q < R, vv = v < R;
                double x_pu = a[p + u * lda], x_pv = vv ? a[p + v * lda] : 0.0;
                double x_qu = qv ? a[q + u * lda] : 0.0, x_qv = (qv && vv) ? a[q + v * lda] : 0.0;
                if (rP) {  // rows by pair P
                    const double c = prm[4 * P], sn = prm[4 * P + 1];
                    const double y_pu = c * x_pu - sn * x_qu, y_qu = sn * x_pu + c * x_qu;
                    const double y_pv = c * x_pv - sn * x_qv, y_qv = sn * x_pv + c * x_qv;
                    x_pu = y_pu;
                    x_qu = y_qu;
                    x_pv = y_pv;
                    x_qv = y_qv;
                }
                if (rQ) {  // then columns by pair Q
                    const double c = prm[4 * Q], sn = prm[4 * Q + 1];
                    const double z_pu = c * x_pu - sn * x_pv, z_pv = sn * x_pu + c * x_pv;
                    const double z_qu = c * x_qu - sn * x_qv, z_qv = sn * x_qu + c * x_qv;
                    x_pu = z_pu;
                    x_pv = z_pv;
                    x_qu = z_qu;
                    x_qv = z_qv;
                }
                a[p + u * lda] = x_pu;
                a[u + p * lda] = x_pu;
                if (vv) {
                    a[p + v * lda] = x_pv;
                    a[v + p * lda] = x_pv;
                }
                if (qv) {
                    a[q + u * lda] = x_qu;
                    a[u + q * lda] = x_qu;
                }
                if (qv && vv) {
                    a[q + v * lda] = x_qv;
                    a[v + q * lda] = x_qv;
                }
            }
            __syncthreads();
        }
        const int any = *flag;
        __syncthreads();
        if (!any) break;
    }
    double l = a[0], h = a[0];
    for (int k = 1; k < R; ++k) {
        const double v = a[k + k * lda];
        if (v < l) l = v;
        if (v > h) h = v;
    }
    *lo = l;
    *hi = h;
}

// The exact branch: (mode, reg) from the Jacobi extremes (solve.cpp:21-33).
__device__ __forceinline__ void exact_decision(double lo, double hi, int* mode, int* reg) {
    if (hi <= 0.0) {
        *mode = 0;
        *reg = 1;
    } else {
        *mode = 1;
        *reg = (lo <= 0.0 || hi / lo > kGramConditionLimit) ? 1 : 0;
    }
}

// solve_gram (solve.cpp:9-35) for a block in canonical form: the sweep of G
// (sweep_block), the regularisation decision (pivot ratio and tau bounds; exact Jacobi
// eigenvalues in the band), the sweep of G + 1e-12 tr(G) I when it regularises.  G: R x R
// (column-major, symmetric; not modified), pairs: the lower-pair table or nullptr, gi: G^-1
// (row-major, symmetric) when the mode is 1, cbuf: 128 doubles, jscr: R * R + 128 doubles
// (exact path).  Returns (mode, reg), mode 0 = zero solution.  count: add the path to the
// decision statistics.  Block-uniform call.
template <int EPT>
__device__ __noinline__ int2 gram_solve_block(const double* G, int R, const unsigned short* pairs, double* gi,
                                              double* cbuf, double* jscr, bool count) {
    __shared__ double s_tr, s_maxdiag, s_gnorm, s_dmin, s_dmax;
    __shared__ int s_path, s_mode, s_reg, s_jflag;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, nw = blockDim.x >> 5;
    // the last warp forms |G|_inf, the max diagonal and the trace (k order, solve.cpp:9-16)
    // while the others run the sweep
    if (warp == nw - 1) {
        const double gn = gram_inf_norm_warp(G, R, R);
        if (lane == 0) {
            s_gnorm = gn;
            double maxdiag = G[0], trc = G[0];
            for (int k = 1; k < R; ++k) {
                const double dg = G[k * R + k];
                if (dg > maxdiag) maxdiag = dg;
                trc = trc + dg;
            }
            s_tr = trc;
            s_maxdiag = maxdiag;
        }
    }
    sweep_block<EPT>(G, 0.0, R, pairs, cbuf, gi, &s_dmin, &s_dmax);
    if (warp == 0) {  // tau = tr(G^-1), lane pairs then butterfly (oracle ginv_trace_lanes)
        double v = (lane < R) ? gi[lane * R + lane] : 0.0;
        v = v + ((lane + 32 < R) ? gi[(lane + 32) * R + lane + 32] : 0.0);
        v = butterfly32(v);
        if (lane == 0) {
            bool ut;
            const int path = gram_certificate(s_maxdiag, s_gnorm, s_dmin, s_dmax, v, R, &ut);
            if (count) count_decision(path, ut);
            s_path = path;
            s_mode = 1;
            s_reg = (path == kDecReg) ? 1 : 0;
        }
    }
    __syncthreads();
    if (s_path == kDecExact) {  // rare: Jacobi eigenvalues of a copy of G
        for (int t = tid; t < R * R; t += blockDim.x) jscr[t] = G[t];
        __syncthreads();
        double lo, hi;
        jacobi_eigen_block(jscr, R, R, jscr + R * R, &s_jflag, &lo, &hi);
        if (tid == 0) {
            int md, rg;
            exact_decision(lo, hi, &md, &rg);
            s_mode = md;
            s_reg = rg;
        }
        __syncthreads();
    }
    if (s_mode == 1 && s_reg) {
        double dlo, dhi;
        sweep_block<EPT>(G, 1e-12 * s_tr, R, pairs, cbuf, gi, &dlo, &dhi);
    }
    const int2 res = make_int2(s_mode, s_reg);
    __syncthreads();  // the shared scalars are reused by the next call
    return res;
}

// ---------------------------------------------------------------------------
// K5: solve_gram (solve.cpp:9-35), canonical form: gram_solve_block (sweep,
// decision, regularised sweep), then rows u_j = fma chain over k of b_k G^-1(k, j).  Every
// block solves G redundantly in shared memory; each warp then solves one row.
// flags[0] |= 1 if regularized; flags[1] = nonfinite_code if any output is not finite
// (cprand's NumericalError check, cprand.cpp:42-43).
// Dynamic shared memory: ksolve_smem_bytes(MAXR).
__host__ __device__ constexpr int ksolve_smem_bytes(int maxr) { return (2 * maxr * maxr + maxr + 2 * 128) * 8; }

template <int MAXR>
__global__ void __launch_bounds__(256) k_solve(const double* __restrict__ G, int R,
                                               const double* __restrict__ RHS, int32_t rows,
                                               double* __restrict__ OUT, int* flags,
                                               int nonfinite_code) {
    extern __shared__ double ks_dyn[];  // G^-1 (R x R), jscr (R x R + 128), cbuf (128)
    double* gi = ks_dyn;
    double* jscr = gi + R * R;
    double* cbuf = jscr + R * R + 128;
    constexpr int kEpt = (MAXR * (MAXR + 1) / 2 + 223) / 224;  // lower entries per thread (224 sweep threads)
    const int2 mr = gram_solve_block<kEpt>(G, R, nullptr, gi, cbuf, jscr, blockIdx.x == 0);
    if (blockIdx.x == 0 && threadIdx.x == 0 && mr.y && flags) atomicOr(flags, 1);
    // rows: one warp per row, lane j holds entries j and j + 32 (R <= 64)
    // (the grid is capped at one block per SM: a block pays for the sweep once and walks its rows)
    const int tid = threadIdx.x, lane = tid & 31, nw = blockDim.x >> 5;
    const int j0 = lane, j1 = lane + 32;
    const bool v0 = j0 < R, v1 = MAXR > 32 && j1 < R;
    for (int32_t row = int32_t(blockIdx.x) * nw + (tid >> 5); row < rows; row += int32_t(gridDim.x) * nw) {
        double w0 = v0 ? RHS[int64_t(row) * R + j0] : 0.0;
        double w1 = v1 ? RHS[int64_t(row) * R + j1] : 0.0;
        if (mr.x == 0) {
            w0 = w1 = 0.0;
        } else {
            double a0 = 0.0, a1 = 0.0;
            for (int k = 0; k < R; ++k) {
                const double bk = __shfl_sync(0xffffffffu, k < 32 ? w0 : w1, k & 31);
                if (v0) a0 = __fma_rn(bk, gi[k * R + j0], a0);
                if (v1) a1 = __fma_rn(bk, gi[k * R + j1], a1);
            }
            w0 = a0;
            w1 = a1;
        }
        if (v0) OUT[int64_t(row) * R + j0] = w0;
        if (v1) OUT[int64_t(row) * R + j1] = w1;
        const bool finite = (!v0 || isfinite(w0)) && (!v1 || isfinite(w1));
        if (!finite && flags) flags[1] = nonfinite_code;
    }
}

// ---------------------------------------------------------------------------
// Warp / group reductions of the canonical fitness order:
// butterfly32 above.

// Sum of v[0..n) (n <= 256, missing = +0.0) by one warp: lane-strided then butterfly.
// GLOBAL = true reads through L2 (__ldcg): the values may have been written by
// other blocks.  GLOBAL = false for shared-memory input.
template <bool GLOBAL>
__device__ __forceinline__ double ld_sum(const double* p) {
    if constexpr (GLOBAL) return __ldcg(p);
    else return *p;
}
template <bool GLOBAL>
__device__ __forceinline__ double group_sum256_warp(const double* v, int n, int lane) {
    double q = (lane < n) ? ld_sum<GLOBAL>(v + lane) : 0.0;
#pragma unroll
    for (int m = 1; m < 8; ++m) {
        const int t = lane + 32 * m;
        q = q + ((t < n) ? ld_sum<GLOBAL>(v + t) : 0.0);
    }
    return butterfly32(q);
}

// hsum of v[0..n) in place by one block (8 warps); result in v[0].  v is
// global scratch (n entries) visible to this block.
__device__ void block_hsum_inplace(double* v, int64_t n, double* tmp) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    while (n > 1) {
        const int64_t ng = (n + kGroup - 1) / kGroup;
        for (int64_t g = warp; g < ng; g += nw) {
            const double r = group_sum256_warp<true>(v + g * kGroup, int(min64(kGroup, n - g * kGroup)), lane);
            if (lane == 0) tmp[g] = r;
        }
        __syncthreads();
        __threadfence_block();
        for (int64_t g = threadIdx.x; g < ng; g += blockDim.x) v[g] = tmp[g];
        __syncthreads();
        __threadfence_block();
        n = ng;
    }
}

// ---------------------------------------------------------------------------
// K7: fused fitness, sum over the tensor of (x_hat - x)^2 (with_model) or x^2,
// never materialising x_hat or the full Khatri-Rao product (replaces
// reconstruct + fitness, kruskal.cpp:55-89).  Block = 256 threads handles a
// group of 256 mode-1 fibres: w_j (the KR row of fibre j) in shared memory,
// each warp runs 8 fibres at a time with lanes over i1 (U1 row reused across
// the 8 fibres), butterfly per fibre, group_sum256 per group; the last block
// reduces the group partials with hsum.
struct FitJob {
    const double* t;
    int64_t I1;
    int64_t nfib;
    int N;
    int R;
    int with_model;
    const double* U[kMaxOrder];  // row-major factors (U[0] = mode 1)
    int64_t dims[kMaxOrder];
    double* group_partial;  // ngroups
    double* group_tmp;      // ngroups
    unsigned int* counter;
    double* out;            // 1 value
};

// K7: fused fitness (kruskal.cpp:55-89 semantics) on the fp64 tensor cores.
// A block takes a group of 256 mode-1 fibres: thread per fibre forms w_r (U_N ... U_2 left to
// right) into shared memory; warp w of 8 takes the fibre tiles w, w + 8, w + 16, w + 24 (8
// fibres each; for R > 20 two tiles at a time, registers) and streams the fibres' rows in
// blocks of 32: x_hat = U1 . W^T with mma.sync m8n8k4
// (A = 8 rows of U1, loaded once per row block for the warp's four tiles; B = the tile's w,
// held in registers), so x_hat(i1, j) is the fma chain over r from +0.0 (the mma rounds
// like that chain); the C fragment puts row i1 = 32 rb + 8 a + (lane >> 2) on the lane,
// so the lane's partial of d^2 runs over i1 = m, m + 8, ... (m = lane >> 2) in increasing
// i1, and the 8 partials of a fibre meet in an xor butterfly over lane bits 2..4.  The
// tensor is read once, streaming.  KS = padded R / 4 (w and U1 are zero past R).
template <int KS>
__global__ void __launch_bounds__(256) k_fitness(const FitJob J) {
    extern __shared__ double smem[];
    constexpr int RP4 = 4 * KS;
    double* W = smem;                 // [256][RP4]
    double* F = smem + kGroup * RP4;  // 256
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int q = lane & 3, rr = lane >> 2;
    constexpr int kFW = 8;                   // warps: warp w takes fibre tiles w, w + 8, ...
    constexpr int kTW = KS <= 5 ? 4 : 2;     // fibre tiles (of 8) per warp and pass (registers)
    constexpr int kPass = kGroup / 8 / (kFW * kTW);
    const int R = J.R;
    const int64_t I1 = J.I1;
    const int64_t nrb = (I1 + 31) / 32;
    const int64_t ngroups = (J.nfib + kGroup - 1) / kGroup;
    const double* U1 = J.U[0];
    for (int64_t g = blockIdx.x; g < ngroups; g += gridDim.x) {
        const int64_t j0 = g * kGroup;
        const int n = int(min64(kGroup, J.nfib - j0));
        __syncthreads();
        {
            double w[RP4];
#pragma unroll
            for (int r = 0; r < RP4; ++r) w[r] = 0.0;
            if (J.with_model && tid < n && tid < kGroup) {
                int64_t idx[kMaxOrder];
                int64_t rem = j0 + tid;
                for (int m = 1; m < J.N; ++m) {
                    const int64_t qq = rem / J.dims[m];
                    idx[m] = rem - qq * J.dims[m];
                    rem = qq;
                }
#pragma unroll
                for (int r = 0; r < RP4; ++r) {
                    if (r < R) {
                        double acc = J.U[J.N - 1][idx[J.N - 1] * R + r];
                        for (int m = J.N - 2; m >= 1; --m) acc = acc * J.U[m][idx[m] * R + r];
                        w[r] = acc;
                    }
                }
            }
            if (tid < kGroup)
#pragma unroll
                for (int r = 0; r < RP4; ++r) W[tid * RP4 + r] = w[r];
        }
        __syncthreads();
      for (int pass = 0; pass < kPass; ++pass) {
        double bf[kTW][KS], acc[kTW][2];
#pragma unroll
        for (int t = 0; t < kTW; ++t) {
            const int fb = 8 * (warp + kFW * (t + kTW * pass));
#pragma unroll
            for (int ks = 0; ks < KS; ++ks) bf[t][ks] = W[(fb + rr) * RP4 + 4 * ks + q];
            acc[t][0] = acc[t][1] = 0.0;
        }
        const double* tg = J.t + j0 * I1;
        // the row block's 32 tensor values per lane are loaded a block ahead (two register
        // buffers, the loop unrolled by two), so every warp keeps 32 streaming loads in flight
        double xa[4][kTW][2], xb[4][kTW][2];
        auto load_x = [&](int64_t rb, double (&xv)[4][kTW][2]) {
#pragma unroll
            for (int a = 0; a < 4; ++a) {
                const int64_t i1 = rb * 32 + 8 * a + rr;
                const bool rowok = rb < nrb && i1 < I1;
#pragma unroll
                for (int t = 0; t < kTW; ++t) {
                    const int f = 8 * (warp + kFW * (t + kTW * pass)) + 2 * q;
                    xv[a][t][0] = (rowok && f < n) ? __ldcs(tg + int64_t(f) * I1 + i1) : 0.0;
                    xv[a][t][1] = (rowok && f + 1 < n) ? __ldcs(tg + int64_t(f + 1) * I1 + i1) : 0.0;
                }
            }
        };
        auto block = [&](int64_t rb, const double (&xv)[4][kTW][2]) {
#pragma unroll
            for (int a = 0; a < 4; ++a) {
                const int64_t i1 = rb * 32 + 8 * a + rr;
                const bool rowok = i1 < I1;
                double af[KS];
#pragma unroll
                for (int ks = 0; ks < KS; ++ks)
                    af[ks] = (J.with_model && rowok && 4 * ks + q < R) ? __ldg(U1 + i1 * R + 4 * ks + q) : 0.0;
#pragma unroll
                for (int t = 0; t < kTW; ++t) {
                    double c0 = 0.0, c1 = 0.0;
                    if (J.with_model) {
#pragma unroll
                        for (int ks = 0; ks < KS; ++ks)
                            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                                         : "+d"(c0), "+d"(c1)
                                         : "d"(af[ks]), "d"(bf[t][ks]));
                    }
                    const double d0 = c0 - xv[a][t][0], d1 = c1 - xv[a][t][1];
                    acc[t][0] = __fma_rn(d0, d0, acc[t][0]);
                    acc[t][1] = __fma_rn(d1, d1, acc[t][1]);
                }
            }
        };
        load_x(0, xa);
        for (int64_t rb = 0; rb < nrb; rb += 2) {
            load_x(rb + 1, xb);
            block(rb, xa);
            if (rb + 1 >= nrb) break;
            load_x(rb + 2, xa);
            block(rb + 1, xb);
        }
#pragma unroll
        for (int t = 0; t < kTW; ++t)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                double v = acc[t][e];
                v = v + __shfl_xor_sync(0xffffffffu, v, 4);
                v = v + __shfl_xor_sync(0xffffffffu, v, 8);
                v = v + __shfl_xor_sync(0xffffffffu, v, 16);
                const int f = 8 * (warp + kFW * (t + kTW * pass)) + 2 * q + e;
                if (rr == 0) F[f] = (f < n) ? v : 0.0;
            }
      }
        __syncthreads();
        if (warp == 0) {
            const double r = group_sum256_warp<false>(F, n, lane);
            if (lane == 0) J.group_partial[g] = r;
        }
    }
    if (!last_block_arrive(J.counter)) return;
    block_hsum_inplace(J.group_partial, ngroups, J.group_tmp);
    if (threadIdx.x == 0) *J.out = J.group_partial[0];
}

// ---------------------------------------------------------------------------
// Sampled residual |X_s - U Z^T|^2 and |X_s|^2, one warp per
// sample column; partials per column, last block hsums both.
struct ResidJob {
    int tiled;
    const double* X;  // I x S col-major (or row-tiled)
    const double* U;  // I x R row-major
    const double* Z;  // S x R row-major
    int32_t I, S;
    int R;
    double* col_num;  // S
    double* col_den;  // S
    double* tmp;      // S
    unsigned int* counter;
    double* out;      // 2 values: num, den
};

__global__ void __launch_bounds__(256) k_residual(const ResidJob J) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nw = blockDim.x >> 5;
    for (int32_t c = blockIdx.x * nw + warp; c < J.S; c += gridDim.x * nw) {
        double qn = 0.0, qd = 0.0;
        const double* z = J.Z + int64_t(c) * J.R;
        for (int32_t i = lane; i < J.I; i += 32) {
            double uz = 0.0;
            const double* u = J.U + int64_t(i) * J.R;
            for (int r = 0; r < J.R; ++r) uz = __fma_rn(u[r], z[r], uz);
            const double xv = J.X[J.tiled ? xs_offset(i, c, J.S) : int64_t(c) * J.I + i];
            const double e = xv - uz;
            qn = __fma_rn(e, e, qn);
            qd = __fma_rn(xv, xv, qd);
        }
        qn = butterfly32(qn);
        qd = butterfly32(qd);
        if (lane == 0) {
            J.col_num[c] = qn;
            J.col_den[c] = qd;
        }
    }
    if (!last_block_arrive(J.counter)) return;
    block_hsum_inplace(J.col_num, J.S, J.tmp);
    block_hsum_inplace(J.col_den, J.S, J.tmp);
    if (threadIdx.x == 0) {
        J.out[0] = J.col_num[0];
        J.out[1] = J.col_den[0];
    }
}

// ---------------------------------------------------------------------------
// init_state (rocp.cpp:57-64): P = U Q, P[i][r] = fma chain over k from +0.0.
__global__ void k_mul_uq(const double* __restrict__ U, int32_t I, int R, const double* __restrict__ Q,
                         double* __restrict__ P) {
    const int64_t total = int64_t(I) * R;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t i = e / R;
        const int r = int(e - i * R);
        double acc = 0.0;
        for (int k = 0; k < R; ++k) acc = __fma_rn(U[i * R + k], Q[k * R + r], acc);
        P[e] = acc;
    }
}

// ---------------------------------------------------------------------------
// Synthetic data (gen_synthetic semantics, synthetic.cpp:8-31): signal in the
// canonical x_hat order, Philox/Box-Muller noise keyed by the flat index,
// deterministic fixed-grid norm partials.
struct SynJob {
    double* t;
    int64_t numel;
    int64_t I1;
    int N, R;
    const double* U[kMaxOrder];
    int64_t dims[kMaxOrder];
    uint64_t seed;
    double* part_sig;    // gridDim.x
    double* part_noise;  // gridDim.x
};

__device__ __forceinline__ double noise_at(uint64_t seed, int64_t e) {
    uint32_t c[4] = {uint32_t(uint64_t(e)), uint32_t(uint64_t(e) >> 32), 0x6e6f6973u, 0u};
    philox4x32_10(c, uint32_t(seed), uint32_t(seed >> 32));
    const uint64_t a = (uint64_t(c[0]) | (uint64_t(c[1]) << 32)) >> 11;
    const uint64_t b = (uint64_t(c[2]) | (uint64_t(c[3]) << 32)) >> 11;
    const double u1 = 1.0 - double(a) * 0x1.0p-53;  // (0, 1]
    const double u2 = double(b) * 0x1.0p-53;
    return sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
}

__global__ void __launch_bounds__(256) k_synth_signal(const SynJob J) {
    __shared__ double red_s[256], red_n[256];
    double ps = 0.0, pn = 0.0;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < J.numel; e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t i1 = e % J.I1;
        int64_t rem = e / J.I1;
        int64_t idx[kMaxOrder];
        for (int m = 1; m < J.N; ++m) {
            const int64_t q = rem / J.dims[m];
            idx[m] = rem - q * J.dims[m];
            rem = q;
        }
        double xh = 0.0;
        for (int r = 0; r < J.R; ++r) {
            double w = J.U[J.N - 1][idx[J.N - 1] * J.R + r];
            for (int m = J.N - 2; m >= 1; --m) w = w * J.U[m][idx[m] * J.R + r];
            xh = __fma_rn(J.U[0][i1 * J.R + r], w, xh);
        }
        J.t[e] = xh;
        ps = __fma_rn(xh, xh, ps);
        if (J.part_noise) {
            const double n = noise_at(J.seed, e);
            pn = __fma_rn(n, n, pn);
        }
    }
    red_s[threadIdx.x] = ps;
    red_n[threadIdx.x] = pn;
    __syncthreads();
    for (int off = 128; off >= 1; off >>= 1) {
        if (threadIdx.x < off) {
            red_s[threadIdx.x] = red_s[threadIdx.x] + red_s[threadIdx.x + off];
            red_n[threadIdx.x] = red_n[threadIdx.x] + red_n[threadIdx.x + off];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        J.part_sig[blockIdx.x] = red_s[0];
        if (J.part_noise) J.part_noise[blockIdx.x] = red_n[0];
    }
}

__global__ void __launch_bounds__(256) k_synth_noise(double* t, int64_t numel, uint64_t seed,
                                                     const double* scale_ptr) {
    const double scale = *scale_ptr;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < numel; e += int64_t(gridDim.x) * blockDim.x)
        t[e] = t[e] + scale * noise_at(seed, e);
}


}  // namespace rocpk
