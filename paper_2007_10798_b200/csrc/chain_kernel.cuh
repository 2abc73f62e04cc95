// chain_kernel.cuh -- K6, the persistent factor-dependent chain of a stream
// window (k_chain), and the window residual pass that follows it.
#pragma once

#include "kernels.cuh"

namespace rocpk {

// ===========================================================================
// K6: persistent stream chain.  One cooperative launch (148 blocks x 256) runs
// the whole factor-dependent chain of a window of nb batches
// (RocpStream::consume, rocp.cpp:144-160, after the hoisted draw + gather):
// for every batch the temporal stage (update_last_mode_with, rocp.cpp:71-84),
// then modes 1..N-1 (update_mode_with, rocp.cpp:96-113, Gauss-Seidel).  Per
// stage (DESIGN.md section 5 has the measured phase budget):
//   stage start  contraction blocks start a TMA bulk copy of their X_s tile
//                (row-tiled layout: one contiguous block; X_s never depends on
//                factors); the Gram finisher prefetches its Q entries
//   phase 0      sampled Khatri-Rao Z (S x RP, zero padded), one 32-sample
//                chunk per block, and that chunk's Gram partial       | grid barrier
//   phase 1      concurrently:
//                - contraction blocks: Z tile by TMA; warp w = chunk w of the
//                  superchunk; superchunk partials of X_s Z (register-blocked
//                  variant for R in 33..64, k_chain<true, .>)
//                - the Gram finisher: chunk partials summed in order (one TMA
//                  bulk copy when they fit, else 4 pre-combine blocks), Q += G,
//                  solve_gram in canonical form (the sweep, kernels.cuh gram_solve_block),
//                  publishes G^-1                                        | grid barrier
//   phase B      warp per row: superchunk partials in order, P += X_s Z,
//                forward / diagonal / backward solve -> U(n) or u_new row | grid barrier
// Arithmetic is exactly that of the per-stage kernels (bitwise equal).

__device__ __forceinline__ unsigned long long gtimer_raw() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

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
    unsigned int* zctr;       // phase-0 chunk arrivals: [0] all, [1 + m] superchunk m (cumulative, zeroed per launch)
    unsigned long long* trace;  // optional phase timestamps (globaltimer ns), 16 per stage
    // overlapped window gather (k_gather_warps on reserved SMs): per (b*N + stage) units
    // published / needed; nullptr when the window was gathered before the launch
    const unsigned* gdone;
    const unsigned* gneed;
    // k_flow (flow_kernel.cuh) only
    double* ginv;     // 2 slots of G^-1 (stage parity)
    int* gmode;       // 2 mode flags (0 = zero solution)
    double* wtemp;    // B x R summed temporal right-hand sides of the current batch
    unsigned* fctr;   // dependency counters (flow_kernel.cuh)
    int maxtiles;     // row tiles of the largest stage
    // k_chain<true, .> with streamed items (chain_stream_items): the window's X_s arena as a 2-D
    // tensor map of 128-byte rows (box 64 rows = one 32-sample x 32-row chunk tile, 128-B swizzle),
    // in device memory; nullptr selects the tile-at-a-time items.  zstride: row stride of Z in
    // memory (RP, or RP + 4 for the streamed items so that the tile is bank-conflict free as loaded)
    const void* xmap;
    int zstride;
};

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* a) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
    return v;
}
// Waits until the overlapped gather published every unit of one (batch, stage)
// (seen = a value loaded earlier, usually during the previous phase).  A gather
// that never arrives traps after ~20 s instead of hanging the device (long enough
// for time-slicing with other GPU contexts).
// nap: back-off between polls in ns (0: spin; the chain's own arrivals are microseconds apart).
__device__ __noinline__ void wait_gathered(const unsigned* done, unsigned need, unsigned seen, unsigned nap = 128) {
    if (seen >= need) return;
    const unsigned long long t0 = gtimer_raw();
    while (ld_acquire_u32(done) < need) {
        if (nap) __nanosleep(nap);
        if (gtimer_raw() - t0 > 20000000000ull) {
            printf("rocp: arrival wait timed out (counter %p at %u of %u, block %d)\n", (const void*)done,
                   ld_acquire_u32(done), need, int(blockIdx.x));
            __trap();
        }
    }
}

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
// Trace stamp: every thread of the (uniform) caller reads the timer and only
// 'who' stores, through a predicated store (no branch), so no lane diverges
// from its warp.  A lane-0-only timer read in
// front of a warp-synchronous device call (a warp LDL^T) left the warp split for
// the whole call and made it 4x slower in traced runs.
__device__ __forceinline__ void trace_stamp(unsigned long long* tr, int slot, bool who) {
    const unsigned long long t = gtimer();
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %2, 0;\n @p st.global.u64 [%0], %1;\n}\n" ::"l"(tr + slot), "l"(t),
        "r"(int(who)));
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
// X_s tiles are read exactly once: bulk copy with an L2 evict-first hint
__device__ __forceinline__ void tma_load_1d_once(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
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


constexpr int kMaxSuperRows = 8;  // superchunk partials prefetched per row entry
constexpr int kQPre = 3;          // Q pairs per thread prefetched by the Gram finisher

// Row solves of phase B: warp per row, lanes own entries j and j + 32, u = b G^-1
// against the explicit inverse the finisher published (Ls).  Every load
// of the row (superchunk partials, P, the mode flag) is issued before the wait for
// the bulk copy (bar, phase), which none of them depend on.
__device__ __noinline__ void chain_rows_warp(const double* __restrict__ cpart, double* Prow_base, int st,
                                             int rows, int R, int nsuper, double* out, const double* Ls,
                                             uint64_t* bar, unsigned phase,
                                             const int* mode_flag) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int j0 = lane, j1 = lane + 32;
    const bool v0 = j0 < R, v1 = j1 < R;
    const int mode = __ldcg(mode_flag);
    bool ld_ready = false;
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
        if (!ld_ready) {
            mbar_wait(bar, phase);
            ld_ready = true;
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
        } else {  // u_j = fma chain over k of b_k G^-1(k, j) (Ls holds G^-1, R > 32)
            double a0 = 0.0, a1 = 0.0;
#pragma unroll 4
            for (int k = 0; k < R; ++k) {
                const double bk = __shfl_sync(0xffffffffu, k < 32 ? w0 : w1, k & 31);
                if (v0) a0 = __fma_rn(bk, Ls[k + j0 * R], a0);
                if (v1) a1 = __fma_rn(bk, Ls[k + j1 * R], a1);
            }
            w0 = a0;
            w1 = a1;
        }
        if (v0) out[int64_t(row) * R + j0] = w0;
        if (v1) out[int64_t(row) * R + j1] = w1;
    }
    if (!ld_ready) mbar_wait(bar, phase);  // the phase completes before the barrier's next use
}

// Row solves of phase B for R in 33..64 on the fp64 tensor cores.  A block owns a contiguous
// range of rows.  Per sub-tile of up to 64 rows: every thread sums superchunk partials (in order)
// and P for a few entries with all loads in flight, P += X_s Z is stored, and the right-hand
// sides go to shared memory (row stride RP + 4: conflict-free fragment loads); then each warp
// forms 8 rows of U = W G^-1 as m8n8k4 MMAs, k increasing -- the fma chain u_j = sum_k b_k
// G^-1(k, j) of chain_rows_warp bit for bit (zero padding past R leaves the accumulators
// unchanged; they are never -0).
template <int NT>
__device__ __noinline__ void chain_rows_dmma(const double* __restrict__ cpart, double* Prow_base, int st, int rows,
                                             int R, int nsuper, double* out, const double* Ls, double* wt,
                                             uint64_t* bar, unsigned phase, const int* mode_flag) {
    constexpr int RP = 8 * NT, WS = RP + 4, KS = RP / 4;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int q4 = lane & 3, rr = lane >> 2;
    const int G = gridDim.x;
    const int rpb = (((rows + G - 1) / G) + 7) & ~7;
    const int rb0 = int(blockIdx.x) * rpb, rb1 = min(rows, rb0 + rpb);
    const int mode = __ldcg(mode_flag);
    bool ld_ready = false;
    for (int r0 = rb0; r0 < rb1; r0 += 64) {
        const int nr = min(64, rb1 - r0);
        const int ne = nr * R;
        for (int e = tid; e < 64 * WS; e += blockDim.x) wt[e] = 0.0;
        __syncthreads();
        const double* cp0 = cpart + int64_t(r0) * R;
        double* P0 = Prow_base ? Prow_base + int64_t(r0) * R : nullptr;
        for (int e0 = 0; e0 < ne; e0 += 4 * int(blockDim.x)) {
            double cv[4][kMaxSuperRows], pv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int e = e0 + u * int(blockDim.x) + tid;
                const bool ok = e < ne;
#pragma unroll
                for (int m = 0; m < kMaxSuperRows; ++m)
                    cv[u][m] = (ok && m < nsuper) ? __ldcg(cp0 + int64_t(m) * rows * R + e) : 0.0;
                pv[u] = (ok && st > 0) ? __ldcg(P0 + e) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int e = e0 + u * int(blockDim.x) + tid;
                if (e < ne) {
                    double tot = cv[u][0];
#pragma unroll
                    for (int m = 1; m < kMaxSuperRows; ++m)
                        if (m < nsuper) tot = tot + cv[u][m];
                    for (int m = kMaxSuperRows; m < nsuper; ++m) tot = tot + __ldcg(cp0 + int64_t(m) * rows * R + e);
                    if (st > 0) {
                        tot = pv[u] + tot;
                        P0[e] = tot;
                    }
                    const int rl = e / R, c = e - rl * R;
                    wt[rl * WS + c] = tot;
                }
            }
        }
        __syncthreads();
        if (!ld_ready) {
            mbar_wait(bar, phase);
            ld_ready = true;
        }
        if (warp * 8 < nr) {
            double c0[NT], c1[NT];
#pragma unroll
            for (int n = 0; n < NT; ++n) c0[n] = c1[n] = 0.0;
            if (mode != 0) {
                const double* wb = wt + (warp * 8 + rr) * WS + q4;
#pragma unroll 2
                for (int ks = 0; ks < KS; ++ks) {
                    const int k = 4 * ks + q4;
                    const double a = wb[4 * ks];
#pragma unroll
                    for (int n = 0; n < NT; ++n) {
                        const int col = n * 8 + rr;
                        const double bb = (k < R && col < R) ? Ls[k + col * R] : 0.0;
                        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                                     : "+d"(c0[n]), "+d"(c1[n])
                                     : "d"(a), "d"(bb));
                    }
                }
            }
            const int row = r0 + warp * 8 + rr;
            if (row < rb1) {
#pragma unroll
                for (int n = 0; n < NT; ++n) {
                    const int c = n * 8 + 2 * q4;
                    if (c < R) out[int64_t(row) * R + c] = c0[n];
                    if (c + 1 < R) out[int64_t(row) * R + c + 1] = c1[n];
                }
            }
        }
        __syncthreads();  // wt is rewritten by the next sub-tile
    }
    if (!ld_ready) mbar_wait(bar, phase);  // the phase completes before the barrier's next use
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

// The wide contraction item on the fp64 tensor cores: warp w forms chunk w of
// the (32-row tile, superchunk) item with mma.sync m8n8k4 -- 4 row tiles x
// NT = RP/8 column tiles of 8x8 accumulators, 4 samples per step.  On B200 the
// fp64 MMA rounds exactly like the sequential fma chain in increasing k
// (tools/dmma_order.cu: 4.2M of 4.2M outputs bitwise equal), so each chunk
// partial is bit-identical to chain_contract_blocked's; samples past the chunk
// end enter as 0 x 0, which leaves an accumulator that started at +0.0
// unchanged.  Per 4 samples: 4 + NT shared loads and 4 NT MMAs, against 36
// loads and 16 NT fmas (x4) in the blocked loop.  The chunk partials are then
// summed left to right exactly as in chain_contract_blocked.
template <int NT>
__device__ __noinline__ void chain_contract_dmma(const double* xs, const double* zs, double* red, int cc0, int ccn,
                                                 int nk, int nrows, int R, double* out_rows) {
    constexpr int RP = 8 * NT;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int q = lane & 3, rr = lane >> 2;
    double acc[4][NT][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int n = 0; n < NT; ++n) acc[a][n][0] = acc[a][n][1] = 0.0;
    for (int k0 = 0; k0 < ccn; k0 += 4) {
        const bool valid = k0 + q < ccn;
        const int smp = cc0 + k0 + q;
        double fa[4], fb[NT];
#pragma unroll
        for (int a = 0; a < 4; ++a) fa[a] = valid ? xs[smp * kRowTile + a * 8 + rr] : 0.0;
#pragma unroll
        for (int n = 0; n < NT; ++n) fb[n] = valid ? zs[smp * RP + n * 8 + rr] : 0.0;
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int n = 0; n < NT; ++n)
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                             : "+d"(acc[a][n][0]), "+d"(acc[a][n][1])
                             : "d"(fa[a]), "d"(fb[n]));
    }
    __syncthreads();  // every warp is done with the X tile (the Z tile stays resident)
    constexpr int HC = RP / 2;  // columns per half
    constexpr int RS = (8 * HC * kRedStride <= kSuperSamples * kRowTile) ? kRedStride : kRowTile;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        if (warp < nk) {
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int n = 0; n < NT; ++n)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int col = n * 8 + 2 * q + e, row = a * 8 + rr;
                        if (col >= h * HC && col < (h + 1) * HC)
                            red[(warp * HC + col - h * HC) * RS + row] = acc[a][n][e];
                    }
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

// ---- Streamed wide contraction (R in 33..64, one superchunk per block) ------------------
// The block keeps superchunk zm's Z tile resident and walks its share of the stage's row-tile
// PAIRS (64 rows: tiles 2u, 2u + 1).  A pair's X_s arrives chunk by chunk (two 8 KB tensor-map
// boxes per 32-sample chunk) through a ring of stream_stages(RP) slots, so the loads of the next
// chunks -- and of the block's next pair -- are in flight behind the MMAs.  Warp w owns the
// 16 rows rp = w & 3 of the pair and one half of the column tiles (w >> 2) for EVERY chunk:
// the chunk partial is the fp64 MMA chain over the chunk's samples from +0.0 (rounds like the
// fma chain, tools/dmma_order.cu) and the superchunk partial is the chunk partials summed left
// to right in registers -- the arithmetic of chain_contract_dmma without its shared-memory
// reduction, its block barriers per half, or an exposed tile load per item.
constexpr int kRingStagesMax = 6;
// Shared-memory layouts that keep the MMA fragment loads free of bank conflicts: lane (rr, q4)
// reads row rr of sample k0 + q4, so a sample stride that is a multiple of 128 bytes (X_s: 256)
// would put the four q4 lanes on the same banks.
//   X: each (tile, chunk) = 64 rows of 128 bytes arrives through the tensor map with the 128-byte
//      swizzle (16-byte unit index ^= row index mod 8), so four consecutive samples land on
//      different banks;
//   Z: written to memory with a row stride of RP + 4 doubles (p.zstride), one bulk copy per tile.
constexpr int kRingSlot = 2 * kChunk * kRowTile;  // doubles: two 32-sample x 32-row chunk tiles (16 KB)
// ring stages by padded width: 6 (5 for RP = 64), then the Z tile [256][RP + 4]
__host__ __device__ constexpr int stream_stages(int RP) { return RP >= 64 ? 5 : 6; }

__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void tma_tile_2d_once(void* dst, const void* map, int c0, int c1, uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}

struct StreamPlan {
    int zm, zrank, zcnt;  // the block's superchunk, its rank among that superchunk's blocks, their count
    int units, nk;        // row-tile pairs of this block in the stage, chunks of the superchunk
    int nst;              // ring stages
    unsigned base;        // ring steps this block consumed before the stage (slot / parity bookkeeping)
    int64_t xrow0;        // first 128-byte row of the stage's X_s in the arena
};

// one thread: the tensor copies of ring step (pair index ui, chunk k) = step t of the stage.  A
// box always holds 32 samples; past the end of S it reads the next tile's rows (or zero fill past
// the arena), which the consumer masks.
__device__ __forceinline__ void stream_issue(const StreamPlan& sp, int slot, int ui, int k, const void* xmap, int S,
                                             int tiles, double* ring, uint64_t* rbar, uint64_t pol) {
    const int u = sp.zrank + ui * sp.zcnt;
    const int c0 = sp.zm * kSuperSamples + k * kChunk;
    double* dst = ring + slot * kRingSlot;
    const bool two = 2 * u + 1 < tiles;
    constexpr unsigned kBox = kChunk * kRowTile * 8;
    const int row = int(sp.xrow0) + (2 * u * S + c0) * 2;  // 128-byte rows: below 2^31 (make_xs_map)
    tma_tile_2d_once(dst, xmap, 0, row, &rbar[slot], pol);
    if (two) tma_tile_2d_once(dst + kChunk * kRowTile, xmap, 0, row + 2 * S, &rbar[slot], pol);
    mbar_expect_tx(&rbar[slot], two ? 2 * kBox : kBox);
}

constexpr int kStreamIssuer = 128;  // lane 0 of warp 4: the warps 4..7 carry the smaller column half

template <int NT>
__device__ __noinline__ void chain_stream_items(const StreamPlan sp, int S, int rows, int tiles, int R,
                                                const double* zs, double* ring, uint64_t* rbar, uint64_t* ebar,
                                                double* cpart_m, unsigned long long* tr, const void* xmap) {
    constexpr int RPZ = 8 * NT + 4, NH0 = (NT + 1) / 2, NH1 = NT / 2;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int q4 = lane & 3, rr = lane >> 2;
    const int rp = warp & 3, half = warp >> 2;
    const int n0 = half ? NH0 : 0, nloc = half ? NH1 : NH0;
    const int tsel = rp >> 1, rsub = (rp & 1) * 16, hrow = rp & 1;
    const int T = sp.units * sp.nk;
    // steps in flight: step t + ahead is issued at the start of step t into the slot of step t - 2,
    // once every warp has released it (ebar: one arrival per warp and consumed step), so the warps
    // run up to a step apart without a block barrier
    const int ahead = sp.nst - 2;
    const uint64_t pol = policy_evict_first();
    double acc[2][NH0][2], qv[2][NH0][2];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int n = 0; n < NH0; ++n) qv[a][n][0] = qv[a][n][1] = 0.0;
    // (pair index, chunk) of the step being consumed and of the step being issued
    int ui = 0, k = 0, iu = ahead / sp.nk, ik = ahead - iu * sp.nk;
    unsigned g = sp.base;
    int slot = int(g % unsigned(sp.nst));
    unsigned par = (g / unsigned(sp.nst)) & 1u;
    int islot = int((g + unsigned(ahead)) % unsigned(sp.nst));                 // slot of the step being issued
    unsigned ipar = (((g + unsigned(ahead)) / unsigned(sp.nst)) & 1u) ^ 1u;  // parity of that slot's previous use
    // this lane's fragment offsets inside a swizzled chunk tile (per 4-sample step: + 128 doubles)
    int xo[2];
#pragma unroll
    for (int a = 0; a < 2; ++a) {
        const int r = 2 * q4 + hrow;  // (2 (k0 + q4) + hrow) & 7 == r & 7, k0 a multiple of 4
        xo[a] = r * 16 + (((a * 4 + (rr >> 1)) ^ (r & 7)) << 1) + (rr & 1);
    }
    const int zo = q4 * RPZ + n0 * 8 + rr;
    long long tw_wait = 0, tw_sync = 0, tw_mma = 0;
    (void)tw_sync;  // traced build: cycles waiting for data / for the block, in the MMAs
    for (int t = 0; t < T; ++t) {
        // the slot consumed at step t - 1 is free (block barrier below): refill it
        if (tid == kStreamIssuer && t + ahead < T) {
            mbar_wait(&ebar[islot], ipar);
            stream_issue(sp, islot, iu, ik, xmap, S, tiles, ring, rbar, pol);
        }
        const int u = sp.zrank + ui * sp.zcnt;
        const int cnk = min(kChunk, S - (sp.zm * kSuperSamples + k * kChunk));
        long long tq0 = 0;
        if (tr) tq0 = clock64();
        mbar_wait(&rbar[slot], par);
        if (tr) tw_wait += clock64() - tq0;
        if (tr) trace_stamp(tr, 8, blockIdx.x == 0 && tid == 0 && t == 0);
        const double* xb = ring + slot * kRingSlot + tsel * (kChunk * kRowTile);
        const double* zb = zs + (k * kChunk) * RPZ + zo;
        const bool live = 2 * u + tsel < tiles;
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int n = 0; n < NH0; ++n) acc[a][n][0] = acc[a][n][1] = 0.0;
        if (tr) tq0 = clock64();
        if (live) {
            // the next 4-sample step's fragments are loaded before this step's MMAs
            double fa[2][2], fb[2][NH0];
            auto ld = [&](int ks, int buf) {
                const bool valid = 4 * ks + q4 < cnk;
#pragma unroll
                for (int a = 0; a < 2; ++a) fa[buf][a] = valid ? xb[ks * 128 + xo[a]] : 0.0;
#pragma unroll
                for (int n = 0; n < NH0; ++n) fb[buf][n] = (valid && n < nloc) ? zb[ks * 4 * RPZ + n * 8] : 0.0;
            };
            const int nks = (cnk + 3) >> 2;
            ld(0, 0);
#pragma unroll
            for (int ks = 0; ks < kChunk / 4; ++ks) {
                if (ks < nks) {
                    if (ks + 1 < kChunk / 4) ld(ks + 1, (ks + 1) & 1);  // past the chunk end: masked to zero, unused
#pragma unroll
                    for (int a = 0; a < 2; ++a)
#pragma unroll
                        for (int n = 0; n < NH0; ++n)
                            if (n < nloc)
                                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                                             : "+d"(acc[a][n][0]), "+d"(acc[a][n][1])
                                             : "d"(fa[ks & 1][a]), "d"(fb[ks & 1][n]));
                }
            }
        }
        // superchunk partial = chunk partials in increasing chunk order
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int n = 0; n < NH0; ++n)
#pragma unroll
                for (int e = 0; e < 2; ++e) qv[a][n][e] = (k == 0) ? acc[a][n][e] : qv[a][n][e] + acc[a][n][e];
        if (tr) tw_mma += clock64() - tq0;
        if (k == sp.nk - 1 && live) {
            const int i0 = (2 * u + tsel) * kRowTile + rsub;
#pragma unroll
            for (int a = 0; a < 2; ++a) {
                const int i = i0 + a * 8 + rr;
#pragma unroll
                for (int n = 0; n < NH0; ++n)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int c = (n0 + n) * 8 + 2 * q4 + e;
                        if (n < nloc && i < rows && c < R) cpart_m[int64_t(i) * R + c] = qv[a][n][e];
                    }
            }
        }
        __syncwarp();
        if (lane == 0)  // this warp is done with the slot
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&ebar[slot])) : "memory");
        if (tr) trace_stamp(tr, 9, blockIdx.x == 0 && tid == 0 && t == sp.nk - 1);
        if (++k == sp.nk) {
            k = 0;
            ++ui;
        }
        if (++ik == sp.nk) {
            ik = 0;
            ++iu;
        }
        if (++slot == sp.nst) {
            slot = 0;
            par ^= 1u;
        }
        if (++islot == sp.nst) {
            islot = 0;
            ipar ^= 1u;
        }
    }
    __syncthreads();  // every warp has consumed every step: the ring region is free again
    if (tr && blockIdx.x == 0 && (tid == 0 || tid == kStreamIssuer)) {  // per step, in cycles
        if (tid == 0) {
            tr[20] = (unsigned long long)(tw_wait / max(T, 1));
            tr[21] = (unsigned long long)(tw_sync / max(T, 1));
            tr[22] = (unsigned long long)(tw_mma / max(T, 1));
        } else {
            tr[23] = (unsigned long long)(tw_mma / max(T, 1));
        }
    }
}

// Chunk Gram partial on the fp64 tensor cores (narrow kernel, RP <= 32): the
// lower 8x8 tiles of Z_chunk^T Z_chunk, one warp per tile, 8 MMA steps of 4
// samples over the 32-sample chunk (rows past the chunk end are zero in zc).
// Bit-identical to the per-pair fma chain from +0.0 in sample order (the MMA
// rounds like that chain, tools/dmma_order.cu); out[q] for the lower pair q of
// (i >= j), q = j R - j (j - 1) / 2 + (i - j).
__device__ __noinline__ void chain_chunk_gram_dmma(const double* zc, int RP, int R, double* out) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int q4 = lane & 3, rr = lane >> 2;
    const int nt = RP / 8, ntiles = nt * (nt + 1) / 2;
    for (int t = warp; t < ntiles; t += nw) {
        int ti = 0, tj = t;  // lower tile (ti >= tj) number t, row-major over the lower triangle
        while (tj > ti) {
            tj -= ti + 1;
            ++ti;
        }
        double d0 = 0.0, d1 = 0.0;
#pragma unroll
        for (int k0 = 0; k0 < kChunk; k0 += 4) {
            const double fa = zc[(k0 + q4) * RP + ti * 8 + rr];  // A(i, c) = z[c][i]
            const double fb = zc[(k0 + q4) * RP + tj * 8 + rr];  // B(c, j) = z[c][j]
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                         : "+d"(d0), "+d"(d1)
                         : "d"(fa), "d"(fb));
        }
        const int i = ti * 8 + rr;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int j = tj * 8 + 2 * q4 + e;
            if (i < R && j <= i) out[j * R - j * (j - 1) / 2 + (i - j)] = e ? d1 : d0;
        }
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
constexpr int kSmTotal = 28416;                  // doubles (222 KB; the streamed wide items: 1 KB alignment slack + ring + Z tile)
static_assert(kSuperSamples == 256, "the streamed Z tile is loaded one row per thread");
constexpr int kZU = 4;                           // phase-0 Z elements per thread per round (registers)
constexpr int kGramSplitC = 8;                   // Gram output ranges per superchunk
constexpr int kGramOneBlock = 16384;
constexpr bool kBlockedNarrow = true;  // R <= 32: register-blocked contraction items too
constexpr int kGramBlocksMax = 4;  // Gram pre-combine blocks when one block does not hold every partial
constexpr int kTraceSlots = 24;                  // globaltimer stamps per stage (profiling aid)             // R^2 x chunks combined by one block up to this

// kWide: R in 33..64 (register-blocked contraction); the R <= 32 instance
// carries none of that code, so its register allocation is unaffected.
// kTrace: the profiling build (phase stamps into p.trace); the production
// instance carries no stamp code at all (kTrace = false folds tr to nullptr).
template <bool kWide, bool kTrace>
__global__ void __launch_bounds__(kChainThreads, 1) k_chain(const ChainParams p) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    extern __shared__ __align__(128) double sm[];
    __shared__ unsigned short pairs[64 * 65 / 2];
    __shared__ __align__(8) uint64_t bar;
    __shared__ __align__(8) uint64_t rbar[kRingStagesMax];  // wide: the X_s chunk ring (chain_stream_items): slot filled
    __shared__ __align__(8) uint64_t ebar[kRingStagesMax];  // ... and slot released by the 8 warps
    __shared__ int s_last;
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
        for (int q = 0; q < kRingStagesMax; ++q) {
            mbar_init(&rbar[q], 1);
            mbar_init(&ebar[q], kChainThreads / 32);
        }
    }
    __syncthreads();
    unsigned ring_base = 0;  // ring steps this block has consumed so far (wide, streamed items)
    // the swizzled tensor copies need 1024-byte aligned destinations
    double* ring = sm + ((1024u - (smem_u32(sm) & 1023u)) & 1023u) / 8;
    // Gram: chunk partials are formed in phase 0 by the blocks that build each
    // 32-sample chunk of Z; phase 1 only combines them (canonical superchunk
    // then total order).  Small R^2 x chunks: one block combines everything;
    // otherwise superchunk items pre-combine and the last arrival finishes.
    const int nch = (S + kChunk - 1) / kChunk;
    const int NPp = (npairs + 1) & ~1;  // chunk-partial stride (lower pairs): 16-byte multiple for the bulk copy
    const bool gram_one = int64_t(NPp) * nch <= kGramOneBlock;
    // When one block cannot hold every chunk partial, the superchunk's last chunk block
    // pre-sums them (phase 0), so a single finisher block remains in either case.
    const int gram_blocks = 1;
    const int cblocks = G - gram_blocks;  // contraction blocks [0, cblocks), the Gram finisher after them
    const int gb0 = cblocks;
    const bool is_gram_block = int(blockIdx.x) >= gb0;
    const int cix = int(blockIdx.x);  // contraction index
    double* xs = sm + kSmXs;
    double* zs = sm + kSmZs;
    double* cps = zs + kSuperSamples * RP;
    const int czt = kChunk * RP;  // Z elements of one chunk

    // Phase 0 (chunk Z + chunk Gram partial) runs on the blocks at the TOP of the contraction
    // range (chunk ch -> block cblocks-1-ch), which have no contraction item when items do not
    // fill the grid (configs[1]: 96 items, 19 chunks).  There is no grid barrier after phase 0:
    // each chunk publishes itself (p.zctr), a contraction block waits only for the 8 chunks of
    // its superchunk before its Z bulk copy, the Gram finisher for all of them.
    const int ch_first = (int(blockIdx.x) < cblocks) ? cblocks - 1 - int(blockIdx.x) : nch;
    const bool zreuse = kWide && cblocks >= nsuper;
    const int zm = cix % nsuper, zrank = cix / nsuper, zcnt = (cblocks - zm + nsuper - 1) / nsuper;
    auto first_item_of = [&](int tiles) {
        const int n_contract = tiles * nsuper;
        return is_gram_block ? n_contract : (zreuse ? ((zrank < tiles) ? zm * tiles + zrank : n_contract) : cix);
    };
    // idx of this thread's phase-0 Z elements (chunk ch_first) of stage (b, st), in
    // registers; loaded one phase ahead so the phase-0 critical path is a single L2 gather.
    int32_t nidx[kZU][kMaxOrder - 1];
    auto load_idx = [&](int b, int st) {
        if (b >= p.nb) return;
        const int32_t* idx = p.idx_base + int64_t(b * N + st) * S * n_other;
#pragma unroll
        for (int u = 0; u < kZU; ++u) {
            const int e = tid + u * blockDim.x;
            const int c = ch_first * kChunk + e / RP;
            const bool ok = ch_first < nch && e < czt && c < S;
#pragma unroll
            for (int l = 0; l < kMaxOrder - 1; ++l)
                nidx[u][l] = (ok && l < n_other) ? __ldg(idx + int64_t(c) * n_other + (n_other - 1 - l)) : 0;
        }
    };
    load_idx(0, 0);
    // overlapped gather: the count of the next (batch, stage), loaded a phase ahead
    unsigned gseen = 0;
    if (p.gdone && tid == 0) gseen = ld_acquire_u32(p.gdone);

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
            const int ZS = p.zstride;  // row stride of Z in memory
            double* Z = (st == 0) ? p.zbuf + int64_t(b) * S * ZS : p.gch + int64_t(st) * S * ZS;
            const int tiles = (rows + kRowTile - 1) / kRowTile;
            const int n_contract = tiles * nsuper;
            unsigned long long* tr = (kTrace && p.trace) ? p.trace + (int64_t(b) * N + st) * kTraceSlots : nullptr;
            if (tr) trace_stamp(tr, 0, blockIdx.x == 0 && tid == 0);

            // stage start: TMA the first X_s tile of this block (independent of factors);
            // its arrive.expect_tx is issued with the Z tile in phase 1.
            // item schedule: (tile, superchunk) pairs; the wide kernel gives each block one
            // superchunk (its Z tile, up to 128 KB, is loaded once per stage), the narrow one
            // strides over all items
            // wide with one superchunk per block: the streamed pair items (chain_stream_items);
            // their first ring steps are issued here, ahead of phase 0
            StreamPlan sp{};
            bool stream = false;
            if constexpr (kWide) stream = zreuse && p.xmap != nullptr;
            if (stream) {
                const int npair = (tiles + 1) / 2;
                sp.zm = zm;
                sp.zrank = zrank;
                sp.zcnt = zcnt;
                sp.units = (!is_gram_block && zrank < npair) ? (npair - 1 - zrank) / zcnt + 1 : 0;
                sp.nk = (min(kSuperSamples, S - zm * kSuperSamples) + kChunk - 1) / kChunk;
                sp.base = ring_base;
                sp.nst = stream_stages(RP);
                sp.xrow0 = p.xoff[b * N + st] / 16;
                if (sp.units > 0 && tid == 0) {
                    if (p.gdone) {
                        wait_gathered(p.gdone + b * N + st, __ldg(p.gneed + b * N + st), gseen);
                        asm volatile("fence.proxy.async.global;" ::: "memory");
                    }
                    const int T = sp.units * sp.nk;  // steps 0 .. nst - 3 now, the rest from the item loop
                    fence_proxy_async();  // the ring region was last written through the generic proxy (phase B)
                    const uint64_t pol = policy_evict_first();
                    for (int t = 0; t < min(sp.nst - 2, T); ++t)
                        stream_issue(sp, int((sp.base + unsigned(t)) % unsigned(sp.nst)), t / sp.nk, t % sp.nk, p.xmap, S,
                                     tiles, ring, rbar, pol);
                }
            }
            const int first_item = stream ? n_contract : first_item_of(tiles);
            const bool contract_block = first_item < n_contract;
            if (contract_block && tid == 0) {
                const int tile = first_item % tiles, m = first_item / tiles;
                const int c0 = m * kSuperSamples, cn = min(kSuperSamples, S - c0);
                if (p.gdone) {  // X_s of this (batch, stage) comes from the overlapped gather
                    wait_gathered(p.gdone + b * N + st, __ldg(p.gneed + b * N + st), gseen);
                    asm volatile("fence.proxy.async.global;" ::: "memory");  // generic stores -> bulk copy
                }
                fence_proxy_async();
                tma_load_1d_once(xs, X + (int64_t(tile) * S + c0) * kRowTile, unsigned(cn * kRowTile * 8), &bar);
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
            for (int ch = ch_first; ch < nch; ch += cblocks) {
                const int c0 = ch * kChunk, cn = min(kChunk, S - c0);
                // [32][RP]; scratch, before this block's contraction Z (streamed items: clear of the
                // X ring, whose first steps are already in flight)
                double* zc = stream ? ring + stream_stages(RP) * kRingSlot : zs;
                const int32_t* idx = p.idx_base + int64_t(b * N + st) * S * n_other;
                if (ch == ch_first) {
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
                            if (cc < cn) Z[int64_t(c0 + cc) * ZS + r] = z;
                        }
                    }
                }
                const int e0 = (ch == ch_first) ? kZU * int(blockDim.x) : 0;
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
                    if (cc < cn) Z[int64_t(c0 + cc) * ZS + r] = z;
                }
                __syncthreads();
                if (tr) trace_stamp(tr, 14, tid == 0 && ch == 0);
                if (tid == 0) {  // the chunk's Z rows are in: the contraction does not wait for its Gram partial
                    __threadfence();
                    atomicAdd(p.zctr + 2 + nsuper + ch / kSuper, 1u);
                }
                if constexpr (!kWide) {
                    chain_chunk_gram_dmma(zc, RP, R, p.chpart + int64_t(ch) * NPp);
                } else {
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
                }
                __syncthreads();
                if (tr) trace_stamp(tr, 15, tid == 0 && ch == 0);
                const int msup = ch / kSuper;
                if (tid == 0) {  // the chunk's Z rows and Gram partial are in (bar.sync above)
                    __threadfence();
                    const unsigned prev = atomicAdd(p.zctr + 1 + msup, 1u);
                    const unsigned nck = unsigned(min(kSuper, nch - msup * kSuper));
                    s_last = (!gram_one && prev + 1 == unsigned(b * N + st + 1) * nck) ? 1 : 0;
                    atomicAdd(p.zctr, 1u);
                }
                if (!gram_one) {  // the superchunk's last chunk pre-sums its Gram partials, chunks in order
                    __syncthreads();
                    if (s_last) {
                        __threadfence();
                        const int k0 = msup * kSuper, k1 = min(nch, k0 + kSuper);
                        for (int pp = tid; pp < npairs; pp += blockDim.x) {
                            double v[kSuper];  // every load before the sums
#pragma unroll
                            for (int u = 0; u < kSuper; ++u)
                                v[u] = (k0 + u < k1) ? __ldcg(p.chpart + int64_t(k0 + u) * NPp + pp) : 0.0;
                            double q = v[0];
#pragma unroll
                            for (int u = 1; u < kSuper; ++u)
                                if (k0 + u < k1) q = q + v[u];
                            p.gpart[int64_t(msup) * NPp + pp] = q;
                        }
                        __syncthreads();
                        if (tid == 0) {
                            __threadfence();
                            atomicAdd(p.zctr + 1 + nsuper, 1u);
                        }
                    }
                    __syncthreads();  // s_last is rewritten by the block's next chunk
                }
            }
            if (tr) trace_stamp(tr, 1, blockIdx.x == 0 && tid == 0);

            // ---------------- phase 1
            if (is_gram_block) {
                if (tid == 0) {  // every chunk partial (or every superchunk pre-sum) of this stage published
                    if (gram_one) wait_gathered(p.zctr, unsigned(b * N + st + 1) * unsigned(nch), 0u, 0u);
                    else wait_gathered(p.zctr + 1 + nsuper, unsigned(b * N + st + 1) * unsigned(nsuper), 0u, 0u);
                    asm volatile("fence.proxy.async.global;" ::: "memory");  // generic stores -> bulk copy
                }
                __syncthreads();
                const bool finisher = true;
                if (finisher) {
                    if (tr) trace_stamp(tr, 3, tid == 0);
                    double* A = sm + kSmFact;        // [64][65]
                    double* D = A + 64 * kLdStride;  // 64
                    double* Gs = D + 64;             // R x R column-major
                    double* colb = Gs + 64 * 64;     // 128: the sweep's column buffers
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
                    if (tr) trace_stamp(tr, 18, tid == 0);
                    if (!gram_one) {
                        // the superchunk pre-sums in order; every load of a batch of pairs (the
                        // pre-sums and Q) is issued before the sums and the stores to Q
                        constexpr int kPB = 5;
                        for (int u0 = 0; u0 < kMaxPairsPerThread; u0 += kPB) {
                            if (tid + u0 * int(blockDim.x) >= npairs) break;
                            double gv[kPB][8], qva[kPB], qvb[kPB];
#pragma unroll
                            for (int uu = 0; uu < kPB; ++uu) {
                                const int q = tid + (u0 + uu) * int(blockDim.x);
                                const bool ok = q < npairs;
#pragma unroll
                                for (int m = 0; m < 8; ++m)
                                    gv[uu][m] = (ok && m < nsuper) ? __ldcg(p.gpart + int64_t(m) * NPp + q) : 0.0;
                                qva[uu] = qvb[uu] = 0.0;
                                if (ok && st > 0) {
                                    const int i = pairs[q] >> 8, j = pairs[q] & 0xff;
                                    qva[uu] = __ldcg(p.Q[st - 1] + i + j * R);
                                    qvb[uu] = __ldcg(p.Q[st - 1] + j + i * R);
                                }
                            }
#pragma unroll
                            for (int uu = 0; uu < kPB; ++uu) {
                                const int q = tid + (u0 + uu) * int(blockDim.x);
                                if (q < npairs) {
                                    double tot = gv[uu][0];
#pragma unroll
                                    for (int m = 1; m < 8; ++m)
                                        if (m < nsuper) tot = tot + gv[uu][m];
                                    for (int m = 8; m < nsuper; ++m) tot = tot + __ldcg(p.gpart + int64_t(m) * NPp + q);
                                    const int i = pairs[q] >> 8, j = pairs[q] & 0xff;
                                    double ga = tot, gb = tot;
                                    if (st > 0) {  // Q + G entry by entry (rocp.cpp:108)
                                        ga = qva[uu] + tot;
                                        gb = qvb[uu] + tot;
                                        p.Q[st - 1][i + j * R] = ga;
                                        p.Q[st - 1][j + i * R] = gb;
                                    }
                                    Gs[i + j * R] = ga;
                                    Gs[j + i * R] = gb;
                                }
                            }
                        }
                    }
#pragma unroll
                    for (int u = 0; u < kMaxPairsPerThread; ++u) {
                        const int q = tid + u * int(blockDim.x);
                        if (q >= npairs || !gram_one) break;
                        double tot;
                        {
                            for (int m = 0; m < nsuper; ++m) {
                                const int k0 = m * kSuper, k1 = min(nch, k0 + kSuper);
                                double sq = chs[k0 * NPp + q];
                                for (int k = k0 + 1; k < k1; ++k) sq = sq + chs[k * NPp + q];
                                tot = (m == 0) ? sq : tot + sq;
                            }
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
                    if (tr) trace_stamp(tr, 10, tid == 0);
                    // solve_gram (solve.cpp:9-35) in canonical form: the sweep of G, the
                    // regularisation decision, the regularised sweep when it applies
                    // (kernels.cuh gram_solve_block); G^-1 feeds the row solves of phase B
                    double* gi = sm + 12288;
                    if (tr) trace_stamp(tr, 12, tid == 0);
                    int2 mr;
                    if constexpr (!kWide) {
                        if (npairs <= 224) mr = gram_solve_block<1>(Gs, R, pairs, gi, colb, sm, true);
                        else if (npairs <= 448) mr = gram_solve_block<2>(Gs, R, pairs, gi, colb, sm, true);
                        else mr = gram_solve_block<3>(Gs, R, pairs, gi, colb, sm, true);
                    } else {
                        if (npairs <= 1344) mr = gram_solve_block<6>(Gs, R, pairs, gi, colb, sm, true);
                        else mr = gram_solve_block<10>(Gs, R, pairs, gi, colb, sm, true);
                    }
                    const int s_mode = mr.x, reg = mr.y;
                    if (tr) trace_stamp(tr, 11, tid == 0);
                    if (s_mode == 1)
                        for (int t = tid; t < RR; t += blockDim.x) p.LD[t] = gi[t];
                    if (tid == 0) {
                        p.mode_flag[0] = s_mode;
                        if (reg) atomicOr(p.flags + (st == 0 ? 0 : 2), 1);
                        if (tr) tr[4] = gtimer();
                    }
                    asm volatile("fence.proxy.async.global;" ::: "memory");  // LD is read by TMA
                }
            } else if (stream) {
                if (sp.units > 0) {
                    const int c0 = zm * kSuperSamples, cn = min(kSuperSamples, S - c0);
                    double* zst = ring + stream_stages(RP) * kRingSlot;  // [256][RP + 4], as in memory
                    if (tid == 0) {  // superchunk zm's chunks of Z published (no grid barrier after phase 0)
                        const unsigned nck = unsigned(min(kSuper, nch - zm * kSuper));
                        wait_gathered(p.zctr + 2 + nsuper + zm, unsigned(b * N + st + 1) * nck, 0u, 0u);
                        asm volatile("fence.proxy.async.global;" ::: "memory");  // generic stores -> bulk copy
                        fence_proxy_async();
                        tma_load_1d(zst, Z + int64_t(c0) * ZS, unsigned(cn * ZS * 8), &bar);
                        mbar_expect_tx(&bar, unsigned(cn * ZS * 8));
                    }
                    mbar_wait(&bar, phase);
                    phase ^= 1u;
                    double* cpm = p.cpart + int64_t(zm) * rows * R;
                    if constexpr (kWide) {
                        if (RP == 40) chain_stream_items<5>(sp, S, rows, tiles, R, zst, ring, rbar, ebar, cpm, tr, p.xmap);
                        else if (RP == 48) chain_stream_items<6>(sp, S, rows, tiles, R, zst, ring, rbar, ebar, cpm, tr, p.xmap);
                        else if (RP == 56) chain_stream_items<7>(sp, S, rows, tiles, R, zst, ring, rbar, ebar, cpm, tr, p.xmap);
                        else chain_stream_items<8>(sp, S, rows, tiles, R, zst, ring, rbar, ebar, cpm, tr, p.xmap);
                    }
                    ring_base += unsigned(sp.units * sp.nk);
                }
            } else {
                int zm_cur = -1;
                for (int item = first_item; item < n_contract;
                     item = zreuse ? ((item % tiles) + zcnt < tiles ? item + zcnt : n_contract) : item + cblocks) {
                    const int tile = item % tiles, m = item / tiles;
                    const int c0 = m * kSuperSamples, cn = min(kSuperSamples, S - c0);
                    const int i0 = tile * kRowTile, nrows = min(kRowTile, rows - i0);
                    if (tid == 0) {
                        fence_proxy_async();
                        if (item != first_item)  // later items: X tile now
                            tma_load_1d_once(xs, X + (int64_t(tile) * S + c0) * kRowTile, unsigned(cn * kRowTile * 8), &bar);
                        const bool zload = m != zm_cur;
                        if (zload) {  // superchunk m's chunks of Z published (no grid barrier after phase 0)
                            const unsigned nck = unsigned(min(kSuper, nch - m * kSuper));
                            wait_gathered(p.zctr + 2 + nsuper + m, unsigned(b * N + st + 1) * nck, 0u, 0u);
                            asm volatile("fence.proxy.async.global;" ::: "memory");  // generic stores -> bulk copy
                            tma_load_1d(zs, Z + int64_t(c0) * RP, unsigned(cn * RP * 8), &bar);
                        }
                        mbar_expect_tx(&bar, unsigned(cn * kRowTile * 8 + (zload ? cn * RP * 8 : 0)));
                    }
                    zm_cur = m;
                    mbar_wait(&bar, phase);
                    phase ^= 1u;
                    if (tr) trace_stamp(tr, 8, blockIdx.x == 0 && tid == 0 && item == 0);
                    const int nk = (cn + kChunk - 1) / kChunk;
                    const int cc0 = warp * kChunk;
                    const int ccn = min(kChunk, cn - cc0);
                    if (kWide || kBlockedNarrow) {  // register-blocked item
                        double* orow = p.cpart + (int64_t(m) * rows + i0) * R;
                        const int cn0 = max(ccn, 0);
                        if constexpr (kWide) {  // fp64 tensor cores, bit-identical chunk partials
                            if (RP == 40) chain_contract_dmma<5>(xs, zs, xs, cc0, cn0, nk, nrows, R, orow);
                            else if (RP == 48) chain_contract_dmma<6>(xs, zs, xs, cc0, cn0, nk, nrows, R, orow);
                            else if (RP == 56) chain_contract_dmma<7>(xs, zs, xs, cc0, cn0, nk, nrows, R, orow);
                            else chain_contract_dmma<8>(xs, zs, xs, cc0, cn0, nk, nrows, R, orow);
                        } else {
                            if (RP == 8) chain_contract_blocked<2>(xs, zs, xs, cc0, cn0, nk, nrows, R, orow);
                            else if (RP == 16) chain_contract_blocked<4>(xs, zs, xs, cc0, cn0, nk, nrows, R, orow);
                            else if (RP == 24) chain_contract_blocked<6>(xs, zs, xs, cc0, cn0, nk, nrows, R, orow);
                            else chain_contract_blocked<8>(xs, zs, xs, cc0, cn0, nk, nrows, R, orow);
                        }
                    }
                    for (int g0 = 0; g0 < ng && !kWide && !kBlockedNarrow; g0 += NGP) {
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
                    if (tr) trace_stamp(tr, 9, blockIdx.x == 0 && tid == 0 && item == 0);
                }
            }
            if (tr) trace_stamp(tr, 2, blockIdx.x == 0 && tid == 0);
            __syncthreads();
            grid.sync();
            if (tr) trace_stamp(tr, 5, blockIdx.x == 0 && tid == 0);

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
                    if (tr) trace_stamp(tr, 16, blockIdx.x == 0 && tid == 0);
                    double* out = (st == 0) ? u_new : p.U[st - 1];
                    double* Pst = st > 0 ? p.P[st - 1] : nullptr;
                    if constexpr (kWide) {
                        double* wt = sm + 4608;  // past L/D (R R + R <= 4160 doubles)
                        if (RP == 40) chain_rows_dmma<5>(p.cpart, Pst, st, rows, R, nsuper, out, Ls, wt, &bar, phase, p.mode_flag);
                        else if (RP == 48) chain_rows_dmma<6>(p.cpart, Pst, st, rows, R, nsuper, out, Ls, wt, &bar, phase, p.mode_flag);
                        else if (RP == 56) chain_rows_dmma<7>(p.cpart, Pst, st, rows, R, nsuper, out, Ls, wt, &bar, phase, p.mode_flag);
                        else chain_rows_dmma<8>(p.cpart, Pst, st, rows, R, nsuper, out, Ls, wt, &bar, phase, p.mode_flag);
                    } else {
                        chain_rows_warp(p.cpart, Pst, st, rows, R, nsuper, out, Ls, &bar, phase, p.mode_flag);
                    }
                    phase ^= 1u;
                    if (tr) trace_stamp(tr, 17, blockIdx.x == 0 && tid == 0);
                }
                load_idx(nb2, ns2);
                if (p.gdone && tid == 0 && nb2 < p.nb) gseen = ld_acquire_u32(p.gdone + nb2 * N + ns2);
            }
            if (tr) trace_stamp(tr, 6, blockIdx.x == 0 && tid == 0);
            __syncthreads();
            grid.sync();
            if (tr) trace_stamp(tr, 7, blockIdx.x == 0 && tid == 0);
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
    unsigned int* rctr;      // nb arrival counters (self-resetting)
    int stage_u;             // B x R temporal rows fit in shared memory
};

// One launch for the window: block (x, b) forms the column partials of 8
// columns of batch b (warp per column, lanes over the B rows, the batch's
// temporal rows staged in shared memory when they fit), and the last block of
// batch b to finish (last_arrive_of on rctr[b]) reduces them in the canonical
// hsum order.  Before, the columns read u row by row from L2 inside a runtime-R
// loop (one load pair per fma) and the hsum was a second launch: 36 us per
// configs[1] step, now a few.
__global__ void __launch_bounds__(256) k_win_resid(const WinResidParams p) {
    extern __shared__ double us[];  // [8][R] z rows of the block's columns, then B x R temporal rows (stage_u)
    const int b = blockIdx.y;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c = blockIdx.x * 8 + warp;
    double* zs = us;
    for (int e = threadIdx.x; e < 8 * p.R; e += blockDim.x) {
        const int w = e / p.R, r = e - w * p.R, cw = blockIdx.x * 8 + w;
        zs[e] = (cw < p.S) ? __ldcg(p.zT + (int64_t(b) * p.S + cw) * p.RP + r) : 0.0;
    }
    const double* u = p.temporal + (p.t_len0 + int64_t(b) * p.B) * p.R;
    if (p.stage_u) {
        for (int e = threadIdx.x; e < p.B * p.R; e += blockDim.x) us[8 * p.R + e] = __ldcg(u + e);
        u = us + 8 * p.R;
    }
    __syncthreads();
    if (c < p.S) {
        const double* X = p.X_base + p.xoff[b * p.N];
        const double* z = zs + warp * p.R;
        double qn = 0.0, qd = 0.0;
        for (int i = lane; i < p.B; i += 32) {
            const double xv = __ldcg(X + xs_offset(i, c, p.S));
            double uz = 0.0;
            for (int r = 0; r < p.R; ++r) uz = __fma_rn(u[int64_t(i) * p.R + r], z[r], uz);
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
    if (!last_arrive_of(p.rctr + b, gridDim.x)) return;
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
