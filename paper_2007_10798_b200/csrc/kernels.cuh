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
// last block sums them in increasing chunk order and optionally accumulates
// (Q + G, rocp.cpp:108).
__global__ void __launch_bounds__(256) k_gram(const double* __restrict__ Z, int32_t s, int R,
                                              double* __restrict__ partial, unsigned int* counter,
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
    if (!last_block_arrive(counter)) return;
    const int nk = gridDim.x;
    for (int p = threadIdx.x; p < RR; p += blockDim.x) {
        // two-level canonical combine: superchunks of kSuper chunks
        double tot = 0.0;
        for (int m0 = 0; m0 < nk; m0 += kSuper) {
            const int m1 = min(nk, m0 + kSuper);
            double pk[kSuper];
#pragma unroll
            for (int u = 0; u < kSuper; ++u)
                pk[u] = (m0 + u < m1) ? __ldcg(partial + int64_t(m0 + u) * RR + p) : 0.0;
            double q = pk[0];
#pragma unroll
            for (int u = 1; u < kSuper; ++u)
                if (m0 + u < m1) q = q + pk[u];
            tot = (m0 == 0) ? q : tot + q;
        }
        out[p] = acc_base ? acc_base[p] + tot : tot;  // column-major == row-major (symmetric)
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

// ---------------------------------------------------------------------------
// K5: solve_gram (solve.cpp:9-35), canonical form:
// zero solution if max diag <= 0; unpivoted LDL^T; regularize with
// 1e-12 tr(G) when a pivot is <= 0 or max/min pivot > 1e12; then per row
// forward (increasing k), diagonal, backward (decreasing k) substitution.
// Every block factors G redundantly in shared memory and solves its rows.
// flags[0] |= 1 if regularized; flags[1] = nonfinite_code if any output is
// not finite (cprand's NumericalError check, cprand.cpp:42-43).
template <int MAXR>
__global__ void __launch_bounds__(256) k_solve(const double* __restrict__ G, int R,
                                               const double* __restrict__ RHS, int32_t rows,
                                               double* __restrict__ OUT, int* flags,
                                               int nonfinite_code) {
    // A holds the working lower triangle (A[i][j], i >= j); the strict upper
    // triangle stores the multipliers, L(i, k) at A[k][i] (never touched by
    // the trailing updates, which only write i >= j > k).
    __shared__ double A[MAXR][MAXR + 1];
    __shared__ double D[MAXR];
    __shared__ int s_mode;  // 0 = zero solution, 1 = solve
    __shared__ int s_reg;
    __shared__ double s_tr;
    const int tid = threadIdx.x;

    auto load = [&](double lambda) {
        for (int t = tid; t < R * R; t += blockDim.x) {
            const int i = t % R, j = t / R;
            if (i >= j) A[i][j] = (i == j) ? G[t] + lambda : G[t];
        }
    };
    auto factor = [&]() {
        for (int k = 0; k < R; ++k) {
            __syncthreads();
            const double dk = A[k][k];
            for (int i = k + 1 + tid; i < R; i += blockDim.x)
                A[k][i] = (dk != 0.0) ? A[i][k] / dk : 0.0;
            if (tid == 0) D[k] = dk;
            __syncthreads();
            const int m = R - k - 1;  // trailing size
            for (int t = tid; t < m * m; t += blockDim.x) {
                const int i = k + 1 + t % m, j = k + 1 + t / m;
                if (j <= i) A[i][j] = __fma_rn(-A[k][i], A[j][k], A[i][j]);
            }
        }
        __syncthreads();
    };

    for (int k = tid; k < R; k += blockDim.x) D[k] = G[k * R + k];  // diagonal, staged
    __syncthreads();
    if (tid == 0) {
        double maxdiag = D[0];
        for (int k = 1; k < R; ++k)
            if (D[k] > maxdiag) maxdiag = D[k];
        double tr = D[0];
        for (int k = 1; k < R; ++k) tr = tr + D[k];
        s_tr = tr;
        s_mode = (maxdiag <= 0.0) ? 0 : 1;
        s_reg = (s_mode == 0) ? 1 : 0;
    }
    __syncthreads();
    if (s_mode == 1) {
        load(0.0);
        factor();
        if (tid == 0) {
            double dmin = D[0], dmax = D[0];
            for (int k = 0; k < R; ++k) {
                if (D[k] < dmin) dmin = D[k];
                if (D[k] > dmax) dmax = D[k];
            }
            s_reg = (!(dmin > 0.0) || dmax > kGramConditionLimit * dmin) ? 1 : 0;
        }
        __syncthreads();
        if (s_reg) {
            load(1e-12 * s_tr);
            factor();
        }
    }
    if (blockIdx.x == 0 && tid == 0 && s_reg && flags) atomicOr(flags, 1);

    const int32_t row = blockIdx.x * blockDim.x + tid;
    if (row >= rows) return;
    double w[MAXR];
#pragma unroll
    for (int j = 0; j < MAXR; ++j) w[j] = (j < R) ? RHS[int64_t(row) * R + j] : 0.0;
    bool finite = true;
    if (s_mode == 0) {
#pragma unroll
        for (int j = 0; j < MAXR; ++j) w[j] = 0.0;
    } else {
        // forward: w[j] -= L(j,k) w[k], k increasing (same bits as the row-wise
        // oracle loop); L(j,k) = A[k][j]
#pragma unroll
        for (int k = 0; k < MAXR; ++k) {
            if (k < R) {
#pragma unroll
                for (int j = k + 1; j < MAXR; ++j)
                    if (j < R) w[j] = __fma_rn(-A[k][j], w[k], w[j]);
            }
        }
#pragma unroll
        for (int j = 0; j < MAXR; ++j) {
            if (j < R) {
                const double dj = D[j];
                w[j] = (fabs(dj) > 2.2250738585072014e-308) ? w[j] / dj : 0.0;
            }
        }
        // backward: w[j] -= L(k,j) w[k], k decreasing; L(k,j) = A[j][k]
#pragma unroll
        for (int k = MAXR - 1; k >= 0; --k) {
            if (k < R) {
#pragma unroll
                for (int j = 0; j < k; ++j) w[j] = __fma_rn(-A[j][k], w[k], w[j]);
            }
        }
    }
#pragma unroll
    for (int j = 0; j < MAXR; ++j) {
        if (j < R) {
            OUT[int64_t(row) * R + j] = w[j];
            finite = finite && isfinite(w[j]);
        }
    }
    if (!finite && flags) flags[1] = nonfinite_code;
}

// ---------------------------------------------------------------------------
// Warp / group reductions of the canonical fitness order.
__device__ __forceinline__ double butterfly32(double q) {
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) q = q + __shfl_xor_sync(0xffffffffu, q, off);
    return q;
}

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

constexpr int kFitFibres = 8;

__global__ void __launch_bounds__(256) k_fitness(const FitJob J) {
    extern __shared__ double smem[];
    double* W = smem;                       // 256 x R
    double* F = smem + kGroup * J.R;        // 256
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t ngroups = (J.nfib + kGroup - 1) / kGroup;
    for (int64_t g = blockIdx.x; g < ngroups; g += gridDim.x) {
        const int64_t j0 = g * kGroup;
        __syncthreads();
        if (J.with_model) {
            const int64_t j = j0 + threadIdx.x;
            if (j < J.nfib) {
                int64_t idx[kMaxOrder];
                int64_t rem = j;
                for (int m = 1; m < J.N; ++m) {
                    const int64_t q = rem / J.dims[m];
                    idx[m] = rem - q * J.dims[m];
                    rem = q;
                }
                for (int r = 0; r < J.R; ++r) {
                    double acc = J.U[J.N - 1][idx[J.N - 1] * J.R + r];
                    for (int m = J.N - 2; m >= 1; --m) acc = acc * J.U[m][idx[m] * J.R + r];
                    W[threadIdx.x * J.R + r] = acc;
                }
            }
        }
        __syncthreads();
        for (int pass = 0; pass < 32 / kFitFibres; ++pass) {
            const int jj = warp * 32 + pass * kFitFibres;
            double acc[kFitFibres];
#pragma unroll
            for (int q = 0; q < kFitFibres; ++q) acc[q] = 0.0;
            int nv = int(min64(kFitFibres, J.nfib - (j0 + jj)));
            if (nv > 0) {
                for (int64_t i1 = lane; i1 < J.I1; i1 += 32) {
                    double x[kFitFibres], xh[kFitFibres];
#pragma unroll
                    for (int q = 0; q < kFitFibres; ++q) {
                        x[q] = (q < nv) ? __ldcs(J.t + (j0 + jj + q) * J.I1 + i1) : 0.0;
                        xh[q] = 0.0;
                    }
                    if (J.with_model) {
                        const double* u = J.U[0] + i1 * J.R;
                        for (int r = 0; r < J.R; ++r) {
                            const double ur = __ldg(u + r);
#pragma unroll
                            for (int q = 0; q < kFitFibres; ++q)
                                xh[q] = __fma_rn(ur, W[(jj + q) * J.R + r], xh[q]);
                        }
#pragma unroll
                        for (int q = 0; q < kFitFibres; ++q) {
                            const double d = xh[q] - x[q];
                            acc[q] = __fma_rn(d, d, acc[q]);
                        }
                    } else {
#pragma unroll
                        for (int q = 0; q < kFitFibres; ++q) acc[q] = __fma_rn(x[q], x[q], acc[q]);
                    }
                }
            }
#pragma unroll
            for (int q = 0; q < kFitFibres; ++q) {
                const double f = butterfly32(acc[q]);
                if (lane == 0) F[jj + q] = (q < nv) ? f : 0.0;
            }
        }
        __syncthreads();
        if (warp == 0) {
            const int n = int(min64(kGroup, J.nfib - j0));
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


// ===========================================================================
// K6: persistent stream chain.  One cooperative launch runs the whole
// factor-dependent chain of a window of nb batches (RocpStream::consume,
// rocp.cpp:144-160, after the hoisted draw + gather): for every batch the
// temporal stage (update_last_mode_with, rocp.cpp:71-84), then modes
// 1..N-1 (update_mode_with, rocp.cpp:96-113, Gauss-Seidel).  Per stage:
//   stage start  contraction blocks start a TMA bulk copy of their X_s tile
//                (row-tiled layout: one contiguous 64 KB block; X_s never
//                depends on factors)
//   phase 0      sampled Khatri-Rao Z (S x RP, zero-padded), all blocks | barrier
//   phase 1      concurrently:
//                - contraction blocks: Z tile by TMA, warp w = chunk w of the
//                  superchunk (32 rows x all r per lane), chunk partials
//                  combined in order -> superchunk partials of X_s Z
//                - Gram blocks: (superchunk, output range) partials; the last
//                  to arrive combines (Q += G), factors (canonical LDL^T, one
//                  barrier per pivot) and publishes L, D
//                - idle blocks of the temporal stage: sampled residual of the
//                  previous batch's temporal solve                   | barrier
//   phase 2      warp per row: combine partials, P += X_s Z, forward /
//                diagonal / backward solve -> U(n) or u_new row      | barrier
// Arithmetic is exactly that of the per-stage kernels above (bitwise equal).

struct ChainParams {
    int N, R, S, nb, B, nsuper, resid_level;
    int32_t head[kMaxOrder];
    double* U[kMaxOrder];  // U[n-1], n = 1..N-1, row-major I_n x R
    double* P[kMaxOrder];
    double* Q[kMaxOrder];
    double* temporal;      // row-major; batch b's rows start at t_len0 + b*B
    int64_t t_len0;
    const int32_t* idx_base;  // window: [b][stage] S x (N-1)
    const double* X_base;     // window: [b][stage] row-tiled I_stage x S
    const int64_t* xoff;      // [b*N + stage]
    double* zbuf;             // nb x S x RP: the temporal Z of each batch (window residual pass)
    double* gch;              // N x S x RP: Z of the mode stages
    double* gpart;            // nsuper x R x R Gram superchunk partials
    double* chpart;           // nchunks x R x R Gram chunk partials (phase 0)
    double* cpart;            // nsuper x rows x R
    double* LD;               // R x R (L(i,k) at [k*R + i], i > k) + R (D)
    int* mode_flag;           // [0]: 0 = zero solution, 1 = solve
    int* flags;               // stream flags ([0] temporal regularized, [2] mode solve)
    double* resid;            // N x 2 (num, den) of the last batch
    double* rpart;            // 3 x S
    unsigned int* counter;    // [0] Gram arrivals, [1] residual arrivals
    unsigned long long* trace;  // optional phase timestamps (globaltimer ns), 16 per stage
};

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// ---- TMA bulk copy (cp.async.bulk) + mbarrier helpers ----------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
            smem_u32(bar)),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

constexpr int kChainThreads = 256;
constexpr int kCRB = 8;        // padding unit of R (RP = multiple of 8)
constexpr int kLdStride = 65;  // smem row stride of the factorization triangle (R <= 64)
constexpr int kMaxPairsPerThread = (64 * 65 / 2 + kChainThreads - 1) / kChainThreads;


// Canonical LDL^T of G (R x R column-major in smem) by one block, one barrier
// per pivot step; same per-element operation sequence as k_solve / the oracle.
// Thread t owns the lower-triangle pairs t, t + 256, ... (column order).
// d_{k+1} is formed redundantly in registers by every thread that needs it
// (its last update), so the diagonal entry is never written in the step that
// finishes it.  L(i,k) at A[k*kLdStride + i].
__device__ __noinline__ void ldlt_one_sync(double* A, double* D, int R, double lambda, const double* G,
                                           const unsigned short* pairs, int npairs) {
    const int tid = threadIdx.x, nt = blockDim.x;
    int pi[kMaxPairsPerThread], pj[kMaxPairsPerThread];
#pragma unroll
    for (int u = 0; u < kMaxPairsPerThread; ++u) {
        const int pp = tid + u * nt;
        pi[u] = (pp < npairs) ? (pairs[pp] >> 8) : -1;
        pj[u] = (pp < npairs) ? (pairs[pp] & 0xff) : -1;
    }
    for (int t = tid; t < R * R; t += nt) {
        const int i = t % R, j = t / R;
        if (i >= j) A[i * kLdStride + j] = (i == j) ? G[t] + lambda : G[t];
    }
    __syncthreads();
    const double d0 = A[0];
    if (tid == 0) D[0] = d0;
    for (int i = 1 + tid; i < R; i += nt) A[i] = (d0 != 0.0) ? A[i * kLdStride] / d0 : 0.0;
    __syncthreads();
    for (int k = 0; k + 1 < R; ++k) {
        const double* rowk = A + k * kLdStride;  // L(., k) in the strict upper part
        const double dn = __fma_rn(-rowk[k + 1], A[(k + 1) * kLdStride + k], A[(k + 1) * kLdStride + k + 1]);
        if (tid == 0) D[k + 1] = dn;
#pragma unroll
        for (int u = 0; u < kMaxPairsPerThread; ++u) {
            const int i = pi[u], j = pj[u];
            if (j > k && !(i == j && j == k + 1)) {
                const double v = __fma_rn(-rowk[i], A[j * kLdStride + k], A[i * kLdStride + j]);
                if (j == k + 1) A[(k + 1) * kLdStride + i] = (dn != 0.0) ? v / dn : 0.0;
                A[i * kLdStride + j] = v;
            }
        }
        __syncthreads();
    }
}

// Canonical LDL^T for R <= MAXR <= 32 by ONE warp, no block barriers: lane i
// holds row i of the lower triangle in registers.  Step k: d_k = lane k's
// r[k] (final), l(i,k) = r[k] / d_k on lanes i > k, then r[j] = fma(-l(i,k),
// a(j,k), r[j]) for k < j <= i with a(j,k) = lane j's r[k].  Identical
// per-element operation sequence to ldlt_one_sync / k_solve / the oracle.
// L(i,k) at A[k*kLdStride + i], D in D[].
//
// Software-pipelined so a step's critical path is divide -> the single fma
// that finishes the next pivot column entry -> shuffle of d_{k+1}: the other
// updates of step k (j >= k+2) are deferred to step k+1, where they fill the
// shuffle latency before the next divide, and column k+1 is read from shared
// memory (published one step ahead) while the divide runs.  Upper-triangle
// registers and lanes >= R receive harmless updates but are never read as
// lower entries; dividends of inactive lanes are 1.0 (a zero dividend takes
// the divide's slow path).
template <int MAXR>
__device__ __noinline__ void ldlt_warp(const double* G, double lambda, int R, double* A, double* D, double* col) {
    // col: three 32-entry column buffers; column k lives in col[(k % 3) * 32]
    // from step k-1 (published) to step k+1 (read by the deferred updates).
    // The fmas read the broadcast column straight from shared memory (no
    // register copy, which the compiler would place in local memory).
    const int lane = threadIdx.x & 31;
    double r[MAXR];
#pragma unroll
    for (int j = 0; j < MAXR; ++j)
        r[j] = (lane < R && j <= lane) ? ((j == lane) ? G[lane + j * R] + lambda : G[lane + j * R]) : 0.0;
    col[lane] = r[0];
    __syncwarp();
    double dk = __shfl_sync(0xffffffffu, r[0], 0);
    double lp = 0.0;  // l(lane, k-1)
#pragma unroll
    for (int k = 0; k < MAXR; ++k) {
        if (k < R) {
            const double* cb = col + (k % 3) * 32;  // column k
            if (k > 0) {  // deferred updates of step k-1 (j >= k+1): fill the shuffle latency
                const double* cp = col + ((k + 2) % 3) * 32;  // column k-1
#pragma unroll
                for (int j = k + 1; j < MAXR; ++j) r[j] = __fma_rn(-lp, cp[j], r[j]);
            }
            const bool act = lane > k && lane < R;
            const double num = act ? r[k] : 1.0;
            const double q = num / dk;
            const double l = (act && dk != 0.0) ? q : 0.0;
            double dn = 0.0;
            if (k + 1 < MAXR) {  // critical: finish a(., k+1), broadcast d_{k+1}, publish column k+1
                r[k + 1] = __fma_rn(-l, cb[k + 1], r[k + 1]);
                dn = __shfl_sync(0xffffffffu, r[k + 1], (k + 1) & 31);
                col[((k + 1) % 3) * 32 + lane] = r[k + 1];
            }
            if (lane == 0) D[k] = dk;
            if (act) A[k * kLdStride + lane] = l;
            __syncwarp();
            lp = l;
            dk = dn;
        }
    }
}

constexpr int kMaxSuperRows = 8;  // superchunk partials prefetched per row entry
constexpr int kQPre = 3;          // Q pairs per thread prefetched by the Gram finisher

// Row solves of phase 2: warp per row, lanes own entries j and j + 32.
__device__ __noinline__ void chain_rows_warp(const double* __restrict__ cpart, double* Prow_base, int st,
                                             int rows, int R, int nsuper, double* out, const double* Ls,
                                             const double* Ds, int mode) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int j0 = lane, j1 = lane + 32;
    const bool v0 = j0 < R, v1 = j1 < R;
    for (int row = blockIdx.x + warp * gridDim.x; row < rows; row += gridDim.x * nw) {
        double w0 = 0.0, w1 = 0.0;
        // every load of the row (superchunk partials, P) in flight at once
        double c0[kMaxSuperRows], c1[kMaxSuperRows], p0 = 0.0, p1 = 0.0;
#pragma unroll
        for (int m = 0; m < kMaxSuperRows; ++m) {
            c0[m] = (v0 && m < nsuper) ? __ldcg(cpart + (int64_t(m) * rows + row) * R + j0) : 0.0;
            c1[m] = (v1 && m < nsuper) ? __ldcg(cpart + (int64_t(m) * rows + row) * R + j1) : 0.0;
        }
        if (st > 0) {
            if (v0) p0 = __ldcg(Prow_base + int64_t(row) * R + j0);
            if (v1) p1 = __ldcg(Prow_base + int64_t(row) * R + j1);
        }
        if (v0) {
            double tot = c0[0];
#pragma unroll
            for (int m = 1; m < kMaxSuperRows; ++m)
                if (m < nsuper) tot = tot + c0[m];
            for (int m = kMaxSuperRows; m < nsuper; ++m) tot = tot + __ldcg(cpart + (int64_t(m) * rows + row) * R + j0);
            if (st > 0) {
                tot = p0 + tot;
                Prow_base[int64_t(row) * R + j0] = tot;
            }
            w0 = tot;
        }
        if (v1) {
            double tot = c1[0];
#pragma unroll
            for (int m = 1; m < kMaxSuperRows; ++m)
                if (m < nsuper) tot = tot + c1[m];
            for (int m = kMaxSuperRows; m < nsuper; ++m) tot = tot + __ldcg(cpart + (int64_t(m) * rows + row) * R + j1);
            if (st > 0) {
                tot = p1 + tot;
                Prow_base[int64_t(row) * R + j1] = tot;
            }
            w1 = tot;
        }
        if (mode == 0) {
            w0 = 0.0;
            w1 = 0.0;
        } else {
            for (int k = 0; k < R; ++k) {  // forward, k increasing
                const double wk = __shfl_sync(0xffffffffu, k < 32 ? w0 : w1, k & 31);
                if (v0 && j0 > k) w0 = __fma_rn(-Ls[k * R + j0], wk, w0);
                if (v1 && j1 > k) w1 = __fma_rn(-Ls[k * R + j1], wk, w1);
            }
            if (v0) w0 = (fabs(Ds[j0]) > 2.2250738585072014e-308) ? w0 / Ds[j0] : 0.0;
            if (v1) w1 = (fabs(Ds[j1]) > 2.2250738585072014e-308) ? w1 / Ds[j1] : 0.0;
            for (int k = R - 1; k >= 0; --k) {  // backward, k decreasing
                const double wk = __shfl_sync(0xffffffffu, k < 32 ? w0 : w1, k & 31);
                if (j0 < k) w0 = __fma_rn(-Ls[j0 * R + k], wk, w0);
                if (v1 && j1 < k) w1 = __fma_rn(-Ls[j1 * R + k], wk, w1);
            }
        }
        if (v0) out[int64_t(row) * R + j0] = w0;
        if (v1) out[int64_t(row) * R + j1] = w1;
    }
}

// One warp's chunk of the contraction: lane = row, NG groups of 8 r's at a
// time (x loaded once per sample), z rows read as broadcast 16-byte loads.
// Partials go to cps[(warp * CW + j) * 32 + lane], j < NG * 8.
template <int NG>
__device__ __forceinline__ void chain_chunk(const double* __restrict__ xs, const double* __restrict__ zs, int RP,
                                           int g0, int cc0, int ccn, int lane, double* cps, int warp, int CW) {
    double acc[NG * kCRB];
#pragma unroll
    for (int a = 0; a < NG * kCRB; ++a) acc[a] = 0.0;
    if (ccn == kChunk) {
#pragma unroll 4
        for (int cc = 0; cc < kChunk; ++cc) {
            const double x = xs[(cc0 + cc) * kRowTile + lane];
            const double2* zr = reinterpret_cast<const double2*>(zs + (cc0 + cc) * RP + g0 * kCRB);
#pragma unroll
            for (int q = 0; q < NG * kCRB / 2; ++q) {
                const double2 zz = zr[q];
                acc[2 * q] = __fma_rn(x, zz.x, acc[2 * q]);
                acc[2 * q + 1] = __fma_rn(x, zz.y, acc[2 * q + 1]);
            }
        }
    } else {
        for (int cc = 0; cc < ccn; ++cc) {
            const double x = xs[(cc0 + cc) * kRowTile + lane];
            const double2* zr = reinterpret_cast<const double2*>(zs + (cc0 + cc) * RP + g0 * kCRB);
#pragma unroll
            for (int q = 0; q < NG * kCRB / 2; ++q) {
                const double2 zz = zr[q];
                acc[2 * q] = __fma_rn(x, zz.x, acc[2 * q]);
                acc[2 * q + 1] = __fma_rn(x, zz.y, acc[2 * q + 1]);
            }
        }
    }
#pragma unroll
    for (int a = 0; a < NG * kCRB; ++a) cps[(warp * CW + a) * kRowTile + lane] = acc[a];
}

constexpr int kRedStride = 33;  // padded row stride of the blocked partials (bank-conflict free)

// Register-blocked contraction item for RP = 4 * CPL > 32 (R in 33..64): warp w
// = chunk w of the superchunk; lane = (row group rg = lane / 4: rows 4rg..4rg+3)
// x (column group cg = lane % 4: columns cg*CPL .. cg*CPL + CPL - 1), so one
// sample costs 2 + CPL/2 shared loads for 4*CPL fmas.  Each output's chunk
// partial is its fma chain over the chunk's samples from +0.0 (canonical);
// after the compute the X tile region holds the partials of one column half at
// a time (8 x RP/2 x 33 doubles; the Z tile stays resident for the block's
// next item of the same superchunk) and the superchunk partial sums them in
// chunk order.
template <int CPL>
__device__ __noinline__ void chain_contract_blocked(const double* xs, const double* zs, double* red, int cc0, int ccn,
                                                    int nk, int nrows, int R, double* out_rows) {
    constexpr int RP = 4 * CPL;  // padded width
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int rg = lane >> 2, cg = lane & 3;
    double acc[4][CPL];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int j = 0; j < CPL; ++j) acc[a][j] = 0.0;
    for (int cc = 0; cc < ccn; ++cc) {
        const double2* xp = reinterpret_cast<const double2*>(xs + (cc0 + cc) * kRowTile + 4 * rg);
        const double2 xa = xp[0], xb = xp[1];
        const double x[4] = {xa.x, xa.y, xb.x, xb.y};
        const double2* zp = reinterpret_cast<const double2*>(zs + (cc0 + cc) * RP + cg * CPL);
#pragma unroll
        for (int q = 0; q < CPL / 2; ++q) {
            const double2 zz = zp[q];
#pragma unroll
            for (int a = 0; a < 4; ++a) {
                acc[a][2 * q] = __fma_rn(x[a], zz.x, acc[a][2 * q]);
                acc[a][2 * q + 1] = __fma_rn(x[a], zz.y, acc[a][2 * q + 1]);
            }
        }
    }
    __syncthreads();  // every warp is done with the X tile (the Z tile stays resident)
    constexpr int HC = 2 * CPL;  // columns per half
    constexpr int RS = (8 * HC * kRedStride <= kSuperSamples * kRowTile) ? kRedStride : kRowTile;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        if ((cg >> 1) == h && warp < nk) {
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int j = 0; j < CPL; ++j) red[(warp * HC + (cg & 1) * CPL + j) * RS + 4 * rg + a] = acc[a][j];
        }
        __syncthreads();
        for (int e = tid; e < HC * kRowTile; e += blockDim.x) {
            const int c = e >> 5, i = e & 31, r = h * HC + c;
            if (i < nrows && r < R) {
                double qq = red[c * RS + i];
                for (int k = 1; k < nk; ++k) qq = qq + red[(k * HC + c) * RS + i];
                out_rows[int64_t(i) * R + r] = qq;
            }
        }
        __syncthreads();
    }
}

// Shared-memory map of k_chain (doubles):
//   [0, 8192)                X_s tile (TMA); phase B: L/D (TMA); Gram items: Z tile + chunk partials
//   [8192, 8192 + 256*RP)    contraction Z tile (TMA)
//   then                     contraction chunk partials [8][CW][32]
//   [16384, ...)             factor block: A [64][65], D[64], G [64*64], column buffer [64]
constexpr int kSmXs = 0;
constexpr int kSmZs = kSuperSamples * kRowTile;  // 8192
constexpr int kSmFact = 16384;
constexpr int kSmTotal = 27136;                  // doubles
constexpr int kZU = 4;                           // phase-0 Z elements per thread per round (registers)
constexpr int kGramSplitC = 8;                   // Gram output ranges per superchunk
constexpr int kGramOneBlock = 16384;
constexpr int kGramBlocksMax = 4;  // Gram pre-combine blocks when one block does not hold every partial
constexpr int kTraceSlots = 24;                  // globaltimer stamps per stage (profiling aid)             // R^2 x chunks combined by one block up to this

// kWide: R in 33..64 (register-blocked contraction); the R <= 32 instance
// carries none of that code, so its register allocation is unaffected.
template <bool kWide>
__global__ void __launch_bounds__(kChainThreads, 1) k_chain(const ChainParams p) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    extern __shared__ __align__(128) double sm[];
    __shared__ unsigned short pairs[64 * 65 / 2];
    __shared__ __align__(8) uint64_t bar;
    __shared__ int s_mode, s_reg;
    __shared__ double s_tr;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int N = p.N, R = p.R, S = p.S, nsuper = p.nsuper, n_other = N - 1;
    const int ng = (R + kCRB - 1) / kCRB, RP = ng * kCRB;
    const int NGP = (RP <= 32) ? 4 : 1;  // r-groups per contraction pass
    const int CW = NGP * kCRB;           // chunk-partial width
    const int RR = R * R;
    const int G = gridDim.x;
    const int npairs = R * (R + 1) / 2;
    unsigned phase = 0;
    if (tid == 0) {
        int off = 0;
        for (int j = 0; j < R; ++j)
            for (int i = j; i < R; ++i) pairs[off++] = (unsigned short)((i << 8) | j);
        mbar_init(&bar, 1);
    }
    __syncthreads();
    // Gram: chunk partials are formed in phase 0 by the blocks that build each
    // 32-sample chunk of Z; phase 1 only combines them (canonical superchunk
    // then total order).  Small R^2 x chunks: one block combines everything;
    // otherwise superchunk items pre-combine and the last arrival finishes.
    const int nch = (S + kChunk - 1) / kChunk;
    const int NPp = (npairs + 1) & ~1;  // chunk-partial stride (lower pairs): 16-byte multiple for the bulk copy
    const bool gram_one = int64_t(NPp) * nch <= kGramOneBlock;
    const int n_gram = nsuper * kGramSplitC;
    // the superchunk pre-combine is a few microseconds of work: keep nearly every block
    // on the contraction, which bounds phase 1 for large R (C4)
    const int gram_blocks = gram_one ? 1 : min(n_gram, kGramBlocksMax);
    const int cblocks = G - gram_blocks;  // contraction blocks [0, cblocks), Gram blocks after them
    const int gb0 = cblocks;
    const bool is_gram_block = int(blockIdx.x) >= gb0;
    const int cix = int(blockIdx.x);  // contraction index
    double* xs = sm + kSmXs;
    double* zs = sm + kSmZs;
    double* cps = zs + kSuperSamples * RP;
    const int czt = kChunk * RP;  // Z elements of one chunk

    // idx of this thread's phase-0 Z elements (chunk blockIdx.x) of stage (b, st), in
    // registers; loaded one phase ahead so the phase-0 critical path is a single L2 gather.
    int32_t nidx[kZU][kMaxOrder - 1];
    auto load_idx = [&](int b, int st) {
        if (b >= p.nb) return;
        const int32_t* idx = p.idx_base + int64_t(b * N + st) * S * n_other;
#pragma unroll
        for (int u = 0; u < kZU; ++u) {
            const int e = tid + u * blockDim.x;
            const int c = int(blockIdx.x) * kChunk + e / RP;
            const bool ok = int(blockIdx.x) < nch && e < czt && c < S;
#pragma unroll
            for (int l = 0; l < kMaxOrder - 1; ++l)
                nidx[u][l] = (ok && l < n_other) ? __ldg(idx + int64_t(c) * n_other + (n_other - 1 - l)) : 0;
        }
    };
    load_idx(0, 0);

    for (int b = 0; b < p.nb; ++b) {
        double* u_new = p.temporal + (p.t_len0 + int64_t(b) * p.B) * R;
        for (int st = 0; st < N; ++st) {
            // [u_new (modes)] + U(N-1), ..., U(1) without U(st), built with compile-time
            // positions so the list stays in registers
            const double* F[kMaxOrder - 1];
#pragma unroll
            for (int l = 0; l < kMaxOrder - 1; ++l) {
                const int m = (st > 0) ? l - 1 : l;
                int k = N - 1 - m;
                if (st > 0 && k <= st) k -= 1;
                F[l] = (st > 0 && l == 0) ? u_new : ((m >= 0 && k >= 1) ? p.U[k - 1] : nullptr);
            }
            const int rows = (st == 0) ? p.B : p.head[st - 1];
            const double* X = p.X_base + p.xoff[b * N + st];
            // Z of this stage: the temporal Z is kept per batch for the residual pass
            double* Z = (st == 0) ? p.zbuf + int64_t(b) * S * RP : p.gch + int64_t(st) * S * RP;
            const int tiles = (rows + kRowTile - 1) / kRowTile;
            const int n_contract = tiles * nsuper;
            unsigned long long* tr = p.trace ? p.trace + (int64_t(b) * N + st) * kTraceSlots : nullptr;
            if (tr && blockIdx.x == 0 && tid == 0) tr[0] = gtimer();

            // stage start: TMA the first X_s tile of this block (independent of factors);
            // its arrive.expect_tx is issued with the Z tile in phase 1.
            // item schedule: (tile, superchunk) pairs; the wide kernel gives each block one
            // superchunk (its Z tile, up to 128 KB, is loaded once per stage), the narrow one
            // strides over all items
            const bool zreuse = kWide && cblocks >= nsuper;
            const int zm = cix % nsuper, zrank = cix / nsuper, zcnt = (cblocks - zm + nsuper - 1) / nsuper;
            const int first_item = zreuse ? ((zrank < tiles) ? zm * tiles + zrank : n_contract) : cix;
            const bool contract_block = !is_gram_block && first_item < n_contract;
            if (contract_block && tid == 0) {
                const int tile = first_item % tiles, m = first_item / tiles;
                const int c0 = m * kSuperSamples, cn = min(kSuperSamples, S - c0);
                fence_proxy_async();
                tma_load_1d(xs, X + (int64_t(tile) * S + c0) * kRowTile, unsigned(cn * kRowTile * 8), &bar);
            }

            // the single Gram finisher fetches its Q entries during phase 0 (Q(st) only
            // changes in this stage's finisher): off the phase-1 critical path, where the
            // contraction blocks' tile copies congest L2
            double qa[kQPre], qb[kQPre];
#pragma unroll
            for (int u = 0; u < kQPre; ++u) {
                const int q = tid + u * int(blockDim.x);
                qa[u] = qb[u] = 0.0;
                if (is_gram_block && gram_one && st > 0 && q < npairs) {
                    const int i = pairs[q] >> 8, j = pairs[q] & 0xff;
                    qa[u] = __ldcg(p.Q[st - 1] + i + j * R);
                    qb[u] = __ldcg(p.Q[st - 1] + j + i * R);
                }
            }

            // ---------------- phase 0: Z (S x RP, zero padded), one 32-sample chunk per block
            // (sampling.cpp:90-103: 1.0 * F_0 * F_1 * ... left to right), then the chunk's
            // Gram partial from shared memory: fma chain over its samples from +0.0
            // (k_gram's per-chunk sequence), lower pairs mirrored.
            for (int ch = blockIdx.x; ch < nch; ch += G) {
                const int c0 = ch * kChunk, cn = min(kChunk, S - c0);
                double* zc = zs;  // [32][RP]; the contraction Z tile is not loaded before phase 1
                const int32_t* idx = p.idx_base + int64_t(b * N + st) * S * n_other;
                if (ch == int(blockIdx.x)) {
                    double f[kZU][kMaxOrder - 1];
#pragma unroll
                    for (int u = 0; u < kZU; ++u) {
                        const int e = tid + u * blockDim.x;
                        const int cc = e / RP, r = e - cc * RP;
                        const bool live = e < czt && cc < cn && r < R;
#pragma unroll
                        for (int l = 0; l < kMaxOrder - 1; ++l)
                            f[u][l] = (live && l < n_other) ? __ldcg(F[l] + int64_t(nidx[u][l]) * R + r) : 1.0;
                    }
#pragma unroll
                    for (int u = 0; u < kZU; ++u) {
                        const int e = tid + u * blockDim.x;
                        if (e < czt) {
                            const int cc = e / RP, r = e - cc * RP;
                            double z = 0.0;
                            if (cc < cn && r < R) {
                                z = 1.0;
#pragma unroll
                                for (int l = 0; l < kMaxOrder - 1; ++l)
                                    if (l < n_other) z = z * f[u][l];
                            }
                            zc[e] = z;
                            if (cc < cn) Z[int64_t(c0) * RP + e] = z;
                        }
                    }
                }
                const int e0 = (ch == int(blockIdx.x)) ? kZU * int(blockDim.x) : 0;
                for (int e = e0 + tid; e < czt; e += blockDim.x) {  // rare: RP > 32 or extra chunks
                    const int cc = e / RP, r = e - cc * RP;
                    double z = 0.0;
                    if (cc < cn && r < R) {
                        z = 1.0;
#pragma unroll
                        for (int l = 0; l < kMaxOrder - 1; ++l)
                            if (l < n_other)
                                z = z * __ldcg(F[l] + int64_t(__ldg(idx + int64_t(c0 + cc) * n_other + (n_other - 1 - l))) * R + r);
                    }
                    zc[e] = z;
                    if (cc < cn) Z[int64_t(c0) * RP + e] = z;
                }
                __syncthreads();
                if (tr && blockIdx.x == 0 && tid == 0 && ch == 0) tr[14] = gtimer();
                for (int q = tid; q < npairs; q += blockDim.x) {
                    const int i = pairs[q] >> 8, j = pairs[q] & 0xff;
                    double acc = 0.0;
                    if (cn == kChunk) {
#pragma unroll 8
                        for (int cc = 0; cc < kChunk; ++cc) acc = __fma_rn(zc[cc * RP + i], zc[cc * RP + j], acc);
                    } else {
                        for (int cc = 0; cc < cn; ++cc) acc = __fma_rn(zc[cc * RP + i], zc[cc * RP + j], acc);
                    }
                    p.chpart[int64_t(ch) * NPp + q] = acc;  // lower pair q; (j, i) is the same value
                }
                __syncthreads();
                if (tr && blockIdx.x == 0 && tid == 0 && ch == 0) tr[15] = gtimer();
            }
            asm volatile("fence.proxy.async.global;" ::: "memory");  // Z is read by TMA in phase 1
            grid.sync();
            if (tr && blockIdx.x == 0 && tid == 0) tr[1] = gtimer();

            // ---------------- phase 1
            if (is_gram_block) {
                // superchunk sums of the chunk partials, superchunk m = chunks 8m..8m+7 in order
                auto super_sum = [&](int m, int pp) {
                    const int k0 = m * kSuper, k1 = min(nch, k0 + kSuper);
                    double v[kSuper];
#pragma unroll
                    for (int u = 0; u < kSuper; ++u) v[u] = (k0 + u < k1) ? __ldcg(p.chpart + int64_t(k0 + u) * NPp + pp) : 0.0;
                    double q = v[0];
#pragma unroll
                    for (int u = 1; u < kSuper; ++u)
                        if (k0 + u < k1) q = q + v[u];
                    return q;
                };
                bool finisher = gram_one;
                if (!gram_one) {
                    for (int gi = int(blockIdx.x) - gb0; gi < n_gram; gi += gram_blocks) {
                        const int m = gi / kGramSplitC, part = gi % kGramSplitC;
                        const int pp0 = (npairs * part) / kGramSplitC, pp1 = (npairs * (part + 1)) / kGramSplitC;
                        for (int pp = pp0 + tid; pp < pp1; pp += blockDim.x) p.gpart[int64_t(m) * NPp + pp] = super_sum(m, pp);
                    }
                    finisher = last_arrive_of(p.counter, unsigned(gram_blocks));
                }
                if (finisher) {
                    if (tr && tid == 0) tr[3] = gtimer();
                    double* A = sm + kSmFact;        // [64][65]
                    double* D = A + 64 * kLdStride;  // 64
                    double* Gs = D + 64;             // R x R column-major
                    double* colb = Gs + 64 * 64;     // 3 x 32 (ldlt_warp column buffers)
                    // total = superchunk sums in order; Q += G for the modes (rocp.cpp:108)
                    double* chs = sm;  // gram_one: every chunk partial, one TMA bulk copy (nch x NPp <= 16384)
                    if (gram_one && tid == 0) {
                        const unsigned bytes = unsigned(nch * NPp * 8);
                        fence_proxy_async();
                        tma_load_1d(chs, p.chpart, bytes, &bar);
                        mbar_expect_tx(&bar, bytes);
                    }
                    // Q entries of this thread's first kQPre pairs (prefetched in phase 0 when gram_one)
                    if (!gram_one) {
#pragma unroll
                        for (int u = 0; u < kQPre; ++u) {
                            const int q = tid + u * int(blockDim.x);
                            if (st > 0 && q < npairs) {
                                const int i = pairs[q] >> 8, j = pairs[q] & 0xff;
                                qa[u] = __ldcg(p.Q[st - 1] + i + j * R);
                                qb[u] = __ldcg(p.Q[st - 1] + j + i * R);
                            }
                        }
                    }
                    if (gram_one) {
                        mbar_wait(&bar, phase);
                        phase ^= 1u;
                    }
                    if (tr && tid == 0) tr[18] = gtimer();
#pragma unroll
                    for (int u = 0; u < kMaxPairsPerThread; ++u) {
                        const int q = tid + u * int(blockDim.x);
                        if (q >= npairs) break;
                        double tot;
                        if (gram_one) {
                            for (int m = 0; m < nsuper; ++m) {
                                const int k0 = m * kSuper, k1 = min(nch, k0 + kSuper);
                                double sq = chs[k0 * NPp + q];
                                for (int k = k0 + 1; k < k1; ++k) sq = sq + chs[k * NPp + q];
                                tot = (m == 0) ? sq : tot + sq;
                            }
                        } else {
                            double v[8];
#pragma unroll
                            for (int m = 0; m < 8; ++m) v[m] = (m < nsuper) ? __ldcg(p.gpart + int64_t(m) * NPp + q) : 0.0;
                            tot = v[0];
#pragma unroll
                            for (int m = 1; m < 8; ++m)
                                if (m < nsuper) tot = tot + v[m];
                            for (int m = 8; m < nsuper; ++m) tot = tot + __ldcg(p.gpart + int64_t(m) * NPp + q);
                        }
                        // Q + G entry by entry (rocp.cpp:108); G is symmetric bit for bit
                        const int i = pairs[q] >> 8, j = pairs[q] & 0xff;
                        double ga = tot, gb = tot;
                        if (st > 0) {
                            const double qva = (u < kQPre) ? qa[u < kQPre ? u : 0] : __ldcg(p.Q[st - 1] + i + j * R);
                            const double qvb = (u < kQPre) ? qb[u < kQPre ? u : 0] : __ldcg(p.Q[st - 1] + j + i * R);
                            ga = qva + tot;
                            gb = qvb + tot;
                            p.Q[st - 1][i + j * R] = ga;
                            p.Q[st - 1][j + i * R] = gb;
                        }
                        Gs[i + j * R] = ga;
                        Gs[j + i * R] = gb;
                    }
                    __syncthreads();
                    if (tr && tid == 0) tr[10] = gtimer();
                    // canonical solve_gram prologue (solve.cpp:9-35; same sequence as k_solve)
                    if (tid == 0) {
                        double maxdiag = Gs[0], trc = Gs[0];
#pragma unroll 8
                        for (int k = 1; k < R; ++k) {
                            const double dg = Gs[k * R + k];
                            if (dg > maxdiag) maxdiag = dg;
                            trc = trc + dg;
                        }
                        s_tr = trc;
                        s_mode = (maxdiag <= 0.0) ? 0 : 1;
                        s_reg = (s_mode == 0) ? 1 : 0;
                    }
                    __syncthreads();
                    if (tr && tid == 0) tr[12] = gtimer();
                    auto factor = [&](double lambda) {
                        if (R <= 32) {
                            if (warp == 0) {
                                if (R <= 8) ldlt_warp<8>(Gs, lambda, R, A, D, colb);
                                else if (R <= 16) ldlt_warp<16>(Gs, lambda, R, A, D, colb);
                                else if (R <= 24) ldlt_warp<24>(Gs, lambda, R, A, D, colb);
                                else ldlt_warp<32>(Gs, lambda, R, A, D, colb);
                            }
                            __syncthreads();
                        } else {
                            ldlt_one_sync(A, D, R, lambda, Gs, pairs, npairs);
                        }
                    };
                    if (s_mode == 1) {
                        factor(0.0);
                        if (tr && tid == 0) tr[13] = gtimer();
                        if (tid == 0) {
                            double dmin = D[0], dmax = D[0];
#pragma unroll 8
                            for (int k = 0; k < R; ++k) {
                                const double dk = D[k];
                                if (dk < dmin) dmin = dk;
                                if (dk > dmax) dmax = dk;
                            }
                            s_reg = (!(dmin > 0.0) || dmax > kGramConditionLimit * dmin) ? 1 : 0;
                        }
                        __syncthreads();
                        if (s_reg) factor(1e-12 * s_tr);
                    }
                    __syncthreads();
                    if (tr && tid == 0) tr[11] = gtimer();
                    for (int t = tid; t < RR; t += blockDim.x) {
                        const int k = t / R, i = t % R;
                        p.LD[t] = (i > k) ? A[k * kLdStride + i] : 0.0;
                    }
                    for (int k = tid; k < R; k += blockDim.x) p.LD[RR + k] = D[k];
                    if (tid == 0) {
                        p.mode_flag[0] = s_mode;
                        if (s_reg) atomicOr(p.flags + (st == 0 ? 0 : 2), 1);
                        if (tr) tr[4] = gtimer();
                    }
                    asm volatile("fence.proxy.async.global;" ::: "memory");  // LD is read by TMA
                }
            } else {
                for (int item = first_item; item < n_contract;
                     item = zreuse ? ((item % tiles) + zcnt < tiles ? item + zcnt : n_contract) : item + cblocks) {
                    const int tile = item % tiles, m = item / tiles;
                    const int c0 = m * kSuperSamples, cn = min(kSuperSamples, S - c0);
                    const int i0 = tile * kRowTile, nrows = min(kRowTile, rows - i0);
                    if (tid == 0) {
                        fence_proxy_async();
                        if (item != first_item)  // later items: X tile now
                            tma_load_1d(xs, X + (int64_t(tile) * S + c0) * kRowTile, unsigned(cn * kRowTile * 8), &bar);
                        const bool zload = !zreuse || item == first_item;
                        if (zload) tma_load_1d(zs, Z + int64_t(c0) * RP, unsigned(cn * RP * 8), &bar);
                        mbar_expect_tx(&bar, unsigned(cn * kRowTile * 8 + (zload ? cn * RP * 8 : 0)));
                    }
                    mbar_wait(&bar, phase);
                    phase ^= 1u;
                    if (tr && blockIdx.x == 0 && tid == 0 && item == 0) tr[8] = gtimer();
                    const int nk = (cn + kChunk - 1) / kChunk;
                    const int cc0 = warp * kChunk;
                    const int ccn = min(kChunk, cn - cc0);
                    if constexpr (kWide) {  // register-blocked item (R in 33..64)
                        double* orow = p.cpart + (int64_t(m) * rows + i0) * R;
                        const int cn0 = max(ccn, 0);
                        if (RP == 40) chain_contract_blocked<10>(xs, zs, xs, cc0, cn0, nk, nrows, R, orow);
                        else if (RP == 48) chain_contract_blocked<12>(xs, zs, xs, cc0, cn0, nk, nrows, R, orow);
                        else if (RP == 56) chain_contract_blocked<14>(xs, zs, xs, cc0, cn0, nk, nrows, R, orow);
                        else chain_contract_blocked<16>(xs, zs, xs, cc0, cn0, nk, nrows, R, orow);
                    }
                    for (int g0 = 0; g0 < ng && !kWide; g0 += NGP) {
                        if (ccn > 0) {  // warp w = chunk w of the superchunk; lane = row
                            const int ngp = min(NGP, ng - g0);
                            if (ngp == 4) chain_chunk<4>(xs, zs, RP, g0, cc0, ccn, lane, cps, warp, CW);
                            else if (ngp == 3) chain_chunk<3>(xs, zs, RP, g0, cc0, ccn, lane, cps, warp, CW);
                            else if (ngp == 2) chain_chunk<2>(xs, zs, RP, g0, cc0, ccn, lane, cps, warp, CW);
                            else chain_chunk<1>(xs, zs, RP, g0, cc0, ccn, lane, cps, warp, CW);
                        }
                        __syncthreads();
                        // superchunk partial = chunk partials in increasing chunk order
                        for (int e = tid; e < CW * kRowTile; e += blockDim.x) {
                            const int rl = e >> 5, l2 = e & 31, r = g0 * kCRB + rl;
                            if (l2 < nrows && r < R) {
                                double qq = cps[rl * kRowTile + l2];
                                for (int k = 1; k < nk; ++k) qq = qq + cps[(k * CW + rl) * kRowTile + l2];
                                p.cpart[(int64_t(m) * rows + i0 + l2) * R + r] = qq;
                            }
                        }
                        __syncthreads();
                    }
                    if (tr && blockIdx.x == 0 && tid == 0 && item == 0) tr[9] = gtimer();
                }
            }
            if (tr && blockIdx.x == 0 && tid == 0) tr[2] = gtimer();
            __syncthreads();
            grid.sync();
            if (tr && blockIdx.x == 0 && tid == 0) tr[5] = gtimer();

            // ---------------- phase B: row solves; idle blocks load the next stage's idx
            {
                const int nb2 = (st + 1 < N) ? b : b + 1, ns2 = (st + 1 < N) ? st + 1 : 0;
                if (int(blockIdx.x) < rows) {
                    double* Ls = sm;  // R x R, L(i,k) at [k*R + i], then D
                    if (tid == 0) {
                        const unsigned bytes = unsigned(((RR + R + 1) & ~1) * 8);
                        fence_proxy_async();
                        tma_load_1d(Ls, p.LD, bytes, &bar);
                        mbar_expect_tx(&bar, bytes);
                    }
                    mbar_wait(&bar, phase);
                    phase ^= 1u;
                    if (tr && blockIdx.x == 0 && tid == 0) tr[16] = gtimer();
                    const int mode = __ldcg(p.mode_flag);
                    double* out = (st == 0) ? u_new : p.U[st - 1];
                    chain_rows_warp(p.cpart, st > 0 ? p.P[st - 1] : nullptr, st, rows, R, nsuper, out, Ls, Ls + RR,
                                    mode);
                    if (tr && blockIdx.x == 0 && tid == 0) tr[17] = gtimer();
                }
                load_idx(nb2, ns2);
            }
            if (tr && blockIdx.x == 0 && tid == 0) tr[6] = gtimer();
            __syncthreads();
            grid.sync();
            if (tr && blockIdx.x == 0 && tid == 0) tr[7] = gtimer();
        }
    }
}

// Sampled residual of every batch's temporal solve in a window,
// after the chain: column partials (warp per column), then hsum per batch.
struct WinResidParams {
    int N, R, S, B, RP, nb;
    const double* temporal;  // row-major; batch b's rows at t_len0 + b*B
    int64_t t_len0;
    const double* X_base;
    const int64_t* xoff;
    const double* zT;        // nb x S x RP
    double* cols;            // nb x 3 x S
    double* out;             // nb x 2 (num, den)
    double* last_out;        // 2: the last batch's (num, den)
};

__global__ void __launch_bounds__(256) k_win_resid_cols(const WinResidParams p) {
    const int b = blockIdx.y;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c = blockIdx.x * 8 + warp;
    if (c >= p.S) return;
    const double* u = p.temporal + (p.t_len0 + int64_t(b) * p.B) * p.R;
    const double* X = p.X_base + p.xoff[b * p.N];
    const double* z = p.zT + (int64_t(b) * p.S + c) * p.RP;
    double qn = 0.0, qd = 0.0;
    for (int i = lane; i < p.B; i += 32) {
        double uz = 0.0;
        for (int r = 0; r < p.R; ++r) uz = __fma_rn(u[int64_t(i) * p.R + r], z[r], uz);
        const double xv = X[xs_offset(i, c, p.S)];
        const double e = xv - uz;
        qn = __fma_rn(e, e, qn);
        qd = __fma_rn(xv, xv, qd);
    }
    qn = butterfly32(qn);
    qd = butterfly32(qd);
    if (lane == 0) {
        p.cols[(int64_t(b) * 3 + 0) * p.S + c] = qn;
        p.cols[(int64_t(b) * 3 + 1) * p.S + c] = qd;
    }
}

__global__ void __launch_bounds__(256) k_win_resid_sum(const WinResidParams p) {
    const int b = blockIdx.x;
    double* base = p.cols + int64_t(b) * 3 * p.S;
    block_hsum_inplace(base, p.S, base + 2 * p.S);
    block_hsum_inplace(base + p.S, p.S, base + 2 * p.S);
    if (threadIdx.x == 0) {
        const double num = __ldcg(base), den = __ldcg(base + p.S);
        p.out[2 * b] = num;
        p.out[2 * b + 1] = den;
        if (b == p.nb - 1) {
            p.last_out[0] = num;
            p.last_out[1] = den;
        }
    }
}

}  // namespace rocpk
