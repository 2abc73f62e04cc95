// flow_kernel.cuh -- K6 for R <= 32 as a dataflow kernel (k_flow): the persistent
// factor-dependent chain of a stream window without grid barriers.
#pragma once

#include "chain_kernel.cuh"

namespace rocpk {

// ===========================================================================
// k_flow.  Same work and arithmetic as k_chain<false>
// (RocpStream::consume, rocp.cpp:144-160: per batch the temporal stage, then
// modes 1..N-1, Gauss-Seidel), reorganised around one observation: a stage's
// solve U(n) = solve_gram(Q(n), P(n)) recomputes EVERY row from P and Q
// (rocp.cpp:110), and the next stage reads only the S sampled rows of it.  So a
// stage publishes the explicit inverse G^-1 instead of waiting
// for all of its rows:
//   chunk blocks   (one 32-sample chunk of Z each) compute the sampled rows of
//                  the factor the previous stage just solved themselves, one
//                  length-R dot product per entry against its G^-1, and read
//                  every older factor from memory; then the chunk's Gram partial
//   Gram finisher  (last block) sums the chunk partials, Q += G, forms G^-1 and
//                  the regularisation decision (the sweep, kernels.cuh
//                  gram_solve_block), publishes G^-1 (two slots, by stage
//                  parity) and bumps the finished-stage counter
//   contraction    items of X_s Z as in k_chain; the last item of a 32-row tile
//                  sums the tile's superchunk partials into P in place (or the
//                  temporal right-hand sides into wtemp)
//   materialise    the chunk blocks, once their chunk of the next stage is out,
//                  write every row of the solved factor, off the critical path
// Dependencies are counters (release: block barrier + red.release.gpu by one
// thread; acquire: ld.acquire.gpu polls by one thread, then a block barrier), so the
// critical path per stage is: previous G^-1 -> sampled rows -> Z chunk ->
// chunk Gram -> combine -> sweep (G^-1) -> publish.  Reuse hazards are ordered
// by the same chain: a stage's chunk blocks wait for the previous
// stage's tile sums and the rows of the stage before it, which transitively
// orders every buffer's next writer after its last reader.
// Counters (p.fctr, zeroed per launch, cumulative over the launch's stages):
//   [0] finished stages; [1 + st] tile sums of stage st; [1 + N + st] rows of
//   stage st written; [1 + 2N + st * maxtiles + t] item arrivals of tile t.

constexpr int kGinvSlot = 64 * 64;  // doubles per G^-1 slot (R <= 64)

// One contraction item of k_flow on the fp64 tensor cores: rows [8 a0, 8 (a0 + AT)) of a
// 32-row X_s tile against a superchunk of Z (warp w = chunk w), AT row tiles of 8 x NT column
// tiles of 8x8 accumulators per warp.  The same per-output operation sequence as
// chain_contract_dmma (chunk partial = fma chain over the chunk's samples from +0.0, the
// mma rounding like that chain; superchunk partial = chunk partials left to right), so a
// stage with few items can split each tile's rows over 2 or 4 blocks bit-identically.
template <int NT, int AT>
__device__ __noinline__ void flow_contract_dmma(const double* xs, const double* zs, double* red, int cc0, int ccn,
                                                int nk, int a0, int nrows, int R, double* out_rows) {
    constexpr int RP = 8 * NT;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int q = lane & 3, rr = lane >> 2;
    double acc[AT][NT][2];
#pragma unroll
    for (int a = 0; a < AT; ++a)
#pragma unroll
        for (int n = 0; n < NT; ++n) acc[a][n][0] = acc[a][n][1] = 0.0;
    for (int k0 = 0; k0 < ccn; k0 += 4) {
        const bool valid = k0 + q < ccn;
        const int smp = cc0 + k0 + q;
        double fa[AT], fb[NT];
#pragma unroll
        for (int a = 0; a < AT; ++a) fa[a] = valid ? xs[smp * kRowTile + (a0 + a) * 8 + rr] : 0.0;
#pragma unroll
        for (int n = 0; n < NT; ++n) fb[n] = valid ? zs[smp * RP + n * 8 + rr] : 0.0;
#pragma unroll
        for (int a = 0; a < AT; ++a)
#pragma unroll
            for (int n = 0; n < NT; ++n)
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                             : "+d"(acc[a][n][0]), "+d"(acc[a][n][1])
                             : "d"(fa[a]), "d"(fb[n]));
    }
    __syncthreads();  // every warp is done with the X tile (the Z tile stays resident)
    constexpr int HC = RP / 2;  // columns per half
    constexpr int RS = (8 * HC * kRedStride <= kSuperSamples * kRowTile) ? kRedStride : kRowTile;
    constexpr int NR = 8 * AT;  // rows of this item
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        if (warp < nk) {
#pragma unroll
            for (int a = 0; a < AT; ++a)
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
        for (int e = tid; e < HC * NR; e += blockDim.x) {
            const int c = e / NR, il = e - c * NR, r = h * HC + c, i = a0 * 8 + il;
            if (i < nrows && r < R) {
                double qq = red[c * RS + il];
                for (int k = 1; k < nk; ++k) qq = qq + red[(k * HC + c) * RS + il];
                out_rows[int64_t(i) * R + r] = qq;
            }
        }
        __syncthreads();
    }
}

// MAXR = RP (R padded to a multiple of 8, <= 64): every loop over R is unrolled.  R > 32
// (the wide instances, C4): a lane owns columns lane and lane + 32, the factor lists hold at
// most kMO factors (N <= 5), G^-1 is read from shared memory in the row dot products, the
// items keep one superchunk's Z tile resident (each block takes one superchunk's tiles), and
// the chunk Gram partials are pre-summed per superchunk by the superchunk's last chunk (the
// finisher cannot hold them all).
template <int MAXR, bool kTrace>
__global__ void __launch_bounds__(kChainThreads, 1) k_flow(const ChainParams p) {
    extern __shared__ __align__(128) double sm[];
    constexpr bool kWideF = MAXR > 32;
    constexpr int kCW = kWideF ? 2 : 1;               // columns per lane
    constexpr int kMO = kWideF ? 4 : kMaxOrder - 1;   // factors per list
    __shared__ unsigned short pairs[MAXR * (MAXR + 1) / 2];
    __shared__ __align__(8) uint64_t bar;
    __shared__ int s_last;
    constexpr int RP = MAXR;
    constexpr int kW = kChainThreads / 32;  // warps per block
    constexpr int kSPW = kChunk / kW;       // chunk samples per warp
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int N = p.N, R = p.R, S = p.S, nsuper = p.nsuper, n_other = N - 1;
    const int RR = R * R, npairs = R * (R + 1) / 2;
    const int G = gridDim.x;
    const int nch = (S + kChunk - 1) / kChunk;
    const int NPp = (npairs + 1) & ~1;
    const bool gram_one = int64_t(NPp) * nch <= kGramOneBlock;  // the finisher bulk-copies every chunk partial
    const int cblocks = G - 1;  // block G - 1 is the Gram finisher
    const bool is_fin = int(blockIdx.x) == G - 1;
    // chunk ch on block cblocks - 1 - ch (the host keeps at least 8 blocks without a chunk)
    const int ch = is_fin ? nch : cblocks - 1 - int(blockIdx.x);
    const bool chunk_block = ch >= 0 && ch < nch;
    unsigned* fin_ctr = p.fctr;
    unsigned* tsum_ctr = p.fctr + 1;
    unsigned* rows_ctr = p.fctr + 1 + N;
    unsigned* tile_ctr = p.fctr + 1 + 2 * N;
    unsigned* gsum_ctr = p.fctr + 1 + 2 * N + N * p.maxtiles;  // superchunk Gram sums (!gram_one)
    double* xs = sm + kSmXs;
    double* zs = sm + kSmZs;
    double* wsm = sm + kSmFact;  // per warp: the right-hand-side rows it turns into factor rows [8][4][32 kCW]
    double* gsm = sm + kSmFact + 1024 * kCW;  // G^-1 of the stage whose rows this block forms
    unsigned phase = 0;
    if (tid == 0) {
        int off = 0;
        for (int j = 0; j < R; ++j)
            for (int i = j; i < R; ++i) pairs[off++] = (unsigned short)((i << 8) | j);
        mbar_init(&bar, 1);
    }
    __syncthreads();

    auto rows_of = [&](int st) { return (st == 0) ? p.B : int(p.head[st - 1]); };
    auto tiles_of = [&](int st) { return (rows_of(st) + kRowTile - 1) / kRowTile; };
    auto wrows_of = [&](int st) -> double* { return (st == 0) ? p.wtemp : p.P[st - 1]; };
    auto out_of = [&](int b, int st) -> double* {
        return (st == 0) ? p.temporal + (p.t_len0 + int64_t(b) * p.B) * R : p.U[st - 1];
    };
    // mode of factor l in stage st's list ([u_new,] U(N-1), ..., U(1) without U(st); 0 = temporal)
    auto mode_at = [&](int st, int l) -> int {
        if (st == 0) return N - 1 - l;
        if (l == 0) return 0;
        int k = N - 1 - (l - 1);
        if (k <= st) k -= 1;
        return k;
    };
    auto wait_ge = [&](const unsigned* c, unsigned need) {
        if (tid == 0) wait_gathered(c, need, 0u, 0u);
    };
    auto publish = [&](unsigned* c, unsigned v) {  // after a block barrier, by one thread
        asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(c), "r"(v) : "memory");
    };
    // G^-1 of stage sp into shared memory, once per block (a per-warp load of the same few
    // lines from L2 by every warp of every chunk block queues at the L2 slices); block-uniform,
    // the caller synchronises before use
    auto stage_ginv = [&](int sp) {
        const double* slot = p.ginv + (sp & 1) * kGinvSlot;
        for (int t = tid; t < RR; t += kChainThreads) gsm[t] = __ldcg(slot + t);
    };
    // narrow: column `lane` of G^-1 in registers (symmetric: G^-1(k, lane) = gsm[k R + lane])
    auto load_gcol = [&](double* g) {
#pragma unroll
        for (int k = 0; k < MAXR; ++k) g[k] = (lane < R && k < R) ? gsm[k * R + lane] : 0.0;
    };
    // u_c = fma chain over k of w_k G^-1(k, c) (oracle solve_gram_m), w in shared memory;
    // narrow: G^-1 column in registers (g), wide: from shared memory (column c)
    auto row_dot = [&](const double* w, const double* g, int c) {
        double acc = 0.0;
        if constexpr (!kWideF) {
            // w and g are zero past R, and fma(+0, +0, acc) = acc (acc is never -0 here), so the
            // padded steps change nothing: no select on the chain
#pragma unroll
            for (int k = 0; k < MAXR; ++k) acc = __fma_rn(w[k], g[k], acc);
        } else {  // a rolled loop: hoisting every load of an unrolled one spills
#pragma unroll 4
            for (int k = 0; k < R; ++k) acc = __fma_rn(w[k], gsm[k * R + c], acc);
        }
        return acc;
    };

    // idx of this warp's chunk samples (cc = warp + 8q), loaded a stage ahead
    int32_t nidx[kSPW][kMO];
    auto load_idx = [&](int b, int st) {
        if (b >= p.nb || !chunk_block) return;
        const int32_t* idx = p.idx_base + int64_t(b * N + st) * S * n_other;
#pragma unroll
        for (int q = 0; q < kSPW; ++q) {
            const int c = ch * kChunk + warp + kW * q;
#pragma unroll
            for (int l = 0; l < kMO; ++l)
                nidx[q][l] = (c < S && l < n_other) ? __ldg(idx + int64_t(c) * n_other + (n_other - 1 - l)) : 0;
        }
    };
    load_idx(0, 0);

    // rows of the stage sp = (bp, stp) solved before, by this block's warps: warp-global index
    // gw, rows gw, gw + nw_total, ...; four rows at a time, their loads issued together
    auto materialise = [&](int bp, int stp, int gw, int nw_total) {
        const int rows = rows_of(stp);
        if (gw >= rows) return;
        const double* W = wrows_of(stp);
        double* out = out_of(bp, stp);
        const int md = __ldcg(p.gmode + ((bp * N + stp) & 1));
        double g[kWideF ? 1 : MAXR];
        if constexpr (!kWideF) load_gcol(g);  // gsm holds the G^-1 of (bp, stp)
        double* wr = wsm + warp * (4 * 32 * kCW);
        for (int row0 = gw; row0 < rows; row0 += 4 * nw_total) {
            double w[4][kCW];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int row = row0 + q * nw_total;
#pragma unroll
                for (int cw = 0; cw < kCW; ++cw) {
                    const int c = lane + 32 * cw;
                    w[q][cw] = (c < R && row < rows) ? __ldcg(W + int64_t(row) * R + c) : 0.0;
                }
            }
            __syncwarp();
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
                for (int cw = 0; cw < kCW; ++cw) wr[q * 32 * kCW + lane + 32 * cw] = w[q][cw];
            __syncwarp();
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int row = row0 + q * nw_total;
#pragma unroll
                for (int cw = 0; cw < kCW; ++cw) {
                    const int c = lane + 32 * cw;
                    const double u = row_dot(wr + q * 32 * kCW, g, c);
                    if (c < R && row < rows) out[int64_t(row) * R + c] = md ? u : 0.0;
                }
            }
        }
    };

    for (int b = 0; b < p.nb; ++b) {
        double* u_new = p.temporal + (p.t_len0 + int64_t(b) * p.B) * R;
        for (int st = 0; st < N; ++st) {
            const int sg = b * N + st;
            const int b1 = (st > 0) ? b : b - 1, st1 = (st > 0) ? st - 1 : N - 1;  // stage sg - 1
            const int rows = rows_of(st);
            const double* X = p.X_base + p.xoff[b * N + st];
            double* Z = (st == 0) ? p.zbuf + int64_t(b) * S * RP : p.gch + int64_t(st) * S * RP;
            const int tiles = (rows + kRowTile - 1) / kRowTile;
            const int n_contract = tiles * nsuper;
            unsigned long long* tr = (kTrace && p.trace) ? p.trace + int64_t(sg) * kTraceSlots : nullptr;

            if (!is_fin) {
                if (chunk_block) {
                    // ------------- Z chunk (sampling.cpp:90-103), warp per sample, lane = r (and
                    // r + 32); the sampled rows of the factor solved by stage sg - 1 (list
                    // position lod) are formed here from its summed right-hand sides and G^-1
                    const double* F[kMO];
                    int lod = -1;
#pragma unroll
                    for (int l = 0; l < kMO; ++l) {
                        F[l] = nullptr;
                        if (l < n_other) {
                            const int md = mode_at(st, l);
                            F[l] = (md == 0) ? u_new : p.U[md - 1];
                            if (sg >= 1 && md == st1) lod = l;
                        }
                    }
                    if (sg >= 2) {  // rows of stage sg - 2 (factors read from memory)
                        const int b2 = (st1 > 0) ? b1 : b1 - 1, st2 = (st1 > 0) ? st1 - 1 : N - 1;
                        wait_ge(rows_ctr + st2, unsigned(b2 + 1) * unsigned(rows_of(st2)));
                        __syncthreads();
                    }
                    const int c0 = ch * kChunk, cn = min(kChunk, S - c0);
                    double f[kSPW][kMO][kCW];
#pragma unroll
                    for (int q = 0; q < kSPW; ++q)
#pragma unroll
                        for (int cw = 0; cw < kCW; ++cw) {
                            const int c = lane + 32 * cw;
                            const bool live = warp + kW * q < cn && c < R;
#pragma unroll
                            for (int l = 0; l < kMO; ++l)
                                f[q][l][cw] = (live && l < n_other && l != lod) ? __ldcg(F[l] + int64_t(nidx[q][l]) * R + c) : 1.0;
                        }
                    if (sg >= 1) {
                        wait_ge(fin_ctr, unsigned(sg));
                        wait_ge(tsum_ctr + st1, unsigned(b1 + 1) * unsigned(tiles_of(st1)));
                        __syncthreads();
                        if (tr) trace_stamp(tr, 0, ch == 0 && tid == 0);
                        const double* W = wrows_of(st1);
                        double wq[kSPW][kCW];
#pragma unroll
                        for (int q = 0; q < kSPW; ++q) {
                            int32_t iw = 0;
#pragma unroll
                            for (int l = 0; l < kMO; ++l)
                                if (l == lod) iw = nidx[q][l];
#pragma unroll
                            for (int cw = 0; cw < kCW; ++cw) {
                                const int c = lane + 32 * cw;
                                const bool live = warp + kW * q < cn && c < R;
                                wq[q][cw] = live ? __ldcg(W + int64_t(iw) * R + c) : 0.0;
                            }
                        }
                        const int md = __ldcg(p.gmode + ((sg - 1) & 1));
                        stage_ginv(sg - 1);
                        __syncthreads();
                        if (tr) trace_stamp(tr, 15, ch == 0 && tid == 0);
                        double g[kWideF ? 1 : MAXR];
                        if constexpr (!kWideF) load_gcol(g);
#pragma unroll
                        for (int q = 0; q < kSPW; ++q)
#pragma unroll
                            for (int cw = 0; cw < kCW; ++cw) wsm[(warp * kSPW + q) * 32 * kCW + lane + 32 * cw] = wq[q][cw];
                        __syncwarp();
                        if (tr) trace_stamp(tr, 16, ch == 0 && tid == 0);
                        double uq[kSPW][kCW];
                        if constexpr (!kWideF) {
                            // U(4 samples x RP) = W . G^-1 on the fp64 tensor cores, one m8n8k4 tile
                            // row block (rows 4..7 empty): the mma accumulates in increasing k like
                            // the fma chain (w and G^-1 are zero past R), bit-identical
                            const double* wb = wsm + warp * kSPW * 32;
                            double* ub = sm + kSmFact + 2048 + warp * kSPW * 32;
                            const int rr = lane >> 2, q4 = lane & 3;
                            constexpr int NTc = MAXR / 8, KSc = MAXR / 4;
                            double c0[NTc], c1[NTc];
#pragma unroll
                            for (int n = 0; n < NTc; ++n) c0[n] = c1[n] = 0.0;
#pragma unroll
                            for (int ks = 0; ks < KSc; ++ks) {
                                const int k = 4 * ks + q4;
                                const double a = (rr < kSPW) ? wb[rr * 32 + k] : 0.0;
#pragma unroll
                                for (int n = 0; n < NTc; ++n) {
                                    const int col = n * 8 + rr;
                                    const double bb = (k < R && col < R) ? gsm[k * R + col] : 0.0;
                                    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                                                 : "+d"(c0[n]), "+d"(c1[n])
                                                 : "d"(a), "d"(bb));
                                }
                            }
                            if (rr < kSPW)
#pragma unroll
                                for (int n = 0; n < NTc; ++n) {
                                    ub[rr * 32 + n * 8 + 2 * q4] = c0[n];
                                    ub[rr * 32 + n * 8 + 2 * q4 + 1] = c1[n];
                                }
                            __syncwarp();
#pragma unroll
                            for (int q = 0; q < kSPW; ++q) uq[q][0] = (lane < MAXR) ? ub[q * 32 + lane] : 0.0;
                        } else {
#pragma unroll
                            for (int q = 0; q < kSPW; ++q)
#pragma unroll
                                for (int cw = 0; cw < kCW; ++cw)
                                    uq[q][cw] = row_dot(wsm + (warp * kSPW + q) * 32 * kCW, g, lane + 32 * cw);
                        }
#pragma unroll
                        for (int q = 0; q < kSPW; ++q)
#pragma unroll
                            for (int cw = 0; cw < kCW; ++cw) {
#pragma unroll
                                for (int l = 0; l < kMO; ++l)
                                    if (l == lod) f[q][l][cw] = md ? uq[q][cw] : 0.0;
                            }
                        if (tr) trace_stamp(tr, 12, ch == 0 && tid == 0);
                    }
                    double* zc = zs;  // [32][RP]
#pragma unroll
                    for (int q = 0; q < kSPW; ++q) {
                        const int cc = warp + kW * q;
#pragma unroll
                        for (int cw = 0; cw < kCW; ++cw) {
                            const int c = lane + 32 * cw;
                            if (c < RP) {
                                double z = 0.0;
                                if (cc < cn && c < R) {
                                    z = 1.0;
#pragma unroll
                                    for (int l = 0; l < kMO; ++l)
                                        if (l < n_other) z = z * f[q][l][cw];
                                }
                                zc[cc * RP + c] = z;
                                if (cc < cn) Z[int64_t(c0 + cc) * RP + c] = z;
                            }
                        }
                    }
                    __syncthreads();
                    if (tr) trace_stamp(tr, 14, ch == 0 && tid == 0);
                    chain_chunk_gram_dmma(zc, RP, R, p.chpart + int64_t(ch) * NPp);
                    __syncthreads();
                    const int msup = ch / kSuper;
                    if (tid == 0) {  // one release fence for both counters
                        asm volatile("fence.acq_rel.gpu;" ::: "memory");
                        if (gram_one) {
                            asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(p.zctr + 1 + msup) : "memory");
                        } else {  // the superchunk's last chunk pre-sums its Gram partials
                            unsigned prev;
                            asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(p.zctr + 1 + msup) : "memory");
                            const unsigned nck = unsigned(min(kSuper, nch - msup * kSuper));
                            s_last = (prev + 1 == unsigned(sg + 1) * nck) ? 1 : 0;
                        }
                        asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(p.zctr) : "memory");
                    }
                    if (!gram_one) {
                        __syncthreads();
                        if (s_last) {  // superchunk sum of the chunk partials, chunks in order (k_chain's)
                            const int k0 = msup * kSuper, k1 = min(nch, k0 + kSuper);
                            for (int pp = tid; pp < npairs; pp += kChainThreads) {
                                double cv[kSuper];  // every load before the sums
#pragma unroll
                                for (int k = 0; k < kSuper; ++k)
                                    cv[k] = (k0 + k < k1) ? __ldcg(p.chpart + int64_t(k0 + k) * NPp + pp) : 0.0;
                                double v = cv[0];
#pragma unroll
                                for (int k = 1; k < kSuper; ++k)
                                    if (k0 + k < k1) v = v + cv[k];
                                p.gpart[int64_t(msup) * NPp + pp] = v;
                            }
                            __syncthreads();
                            if (tid == 0) publish(gsum_ctr, 1u);
                        }
                    }
                    if (tr) trace_stamp(tr, 1, ch == 0 && tid == 0);
                    const int nb2 = (st + 1 < N) ? b : b + 1, ns2 = (st + 1 < N) ? st + 1 : 0;
                    load_idx(nb2, ns2);
                }
                // ------------- every row of stage sg - 1, off the critical path, by the chunk
                // blocks (the next stage's chunks need these rows only two stages on, rows_ctr):
                // narrow right after their chunk (they are idle until the next stage), wide
                // after their contraction items (every block has items there)
                auto materialise_prev = [&]() {
                    if (!chunk_block || sg < 1) return;
                    const int nwt = nch * kW;
                    materialise(b1, st1, ch + warp * nch, nwt);
                    __syncthreads();
                    if (tid == 0) {
                        const int rows1 = rows_of(st1);
                        unsigned n = 0;
                        for (int w = 0; w < kW; ++w) {
                            const int g0 = ch + w * nch;
                            if (g0 < rows1) n += unsigned((rows1 - 1 - g0) / nwt + 1);
                        }
                        if (n) publish(rows_ctr + st1, n);
                        if (tr && ch == 0) tr[5] = gtimer();
                    }
                };
                if constexpr (!kWideF) materialise_prev();

                // ------------- contraction items (tile, superchunk[, row part]); a stage with few
                // items splits each tile's rows over F = 2 or 4 blocks.  Narrow: item i on block
                // i mod cblocks.  Wide: block c takes superchunk c mod nsuper and every
                // (cblocks / nsuper)-th tile of it, so its Z tile (up to 128 KB) loads once.
                const int F = (4 * n_contract <= cblocks) ? 4 : ((2 * n_contract <= cblocks) ? 2 : 1);
                const bool zr = kWideF && F == 1 && cblocks >= nsuper;
                const int cix = int(blockIdx.x);
                const int zm = cix % nsuper, zrank = cix / nsuper, zcnt = (cblocks - zm + nsuper - 1) / nsuper;
                int zm_cur = -1;
                for (int it = 0;; ++it) {
                    int tile, m, part;
                    if (zr) {
                        const int t = zrank + it * zcnt;
                        if (t >= tiles) break;
                        tile = t;
                        m = zm;
                        part = 0;
                    } else {
                        const int item = cix + it * cblocks;
                        if (item >= F * n_contract) break;
                        part = item % F;
                        const int base = item / F;
                        tile = base % tiles;
                        m = base / tiles;
                    }
                    const int c0 = m * kSuperSamples, cn = min(kSuperSamples, S - c0);
                    const int i0 = tile * kRowTile, nrows = min(kRowTile, rows - i0);
                    if (tid == 0) {  // X_s tile (from the overlapped gather when it runs) and Z tile
                        if (p.gdone) {
                            wait_gathered(p.gdone + b * N + st, __ldg(p.gneed + b * N + st), 0u);
                            asm volatile("fence.proxy.async.global;" ::: "memory");
                        }
                        if (tr && blockIdx.x == 0 && it == 0) tr[7] = gtimer();
                        fence_proxy_async();
                        tma_load_1d_once(xs, X + (int64_t(tile) * S + c0) * kRowTile, unsigned(cn * kRowTile * 8), &bar);
                        const bool zload = m != zm_cur;
                        if (zload) {  // superchunk m's chunks of Z published
                            const unsigned nck = unsigned(min(kSuper, nch - m * kSuper));
                            wait_gathered(p.zctr + 1 + m, unsigned(sg + 1) * nck, 0u, 0u);
                            asm volatile("fence.proxy.async.global;" ::: "memory");
                            tma_load_1d(zs, Z + int64_t(c0) * RP, unsigned(cn * RP * 8), &bar);
                        }
                        mbar_expect_tx(&bar, unsigned(cn * kRowTile * 8 + (zload ? cn * RP * 8 : 0)));
                    }
                    zm_cur = m;
                    mbar_wait(&bar, phase);
                    phase ^= 1u;
                    if (tr) trace_stamp(tr, 8, blockIdx.x == 0 && tid == 0 && it == 0);
                    const int nk = (cn + kChunk - 1) / kChunk;
                    const int cc0 = warp * kChunk;
                    const int cn0 = max(min(kChunk, cn - cc0), 0);
                    double* orow = p.cpart + (int64_t(m) * rows + i0) * R;
                    // fp64 tensor cores (bit-identical to the register-blocked fma chains:
                    // tools/contract_bench.cu; 7270 -> 5842 cycles per R = 20 item)
                    if (F == 1) flow_contract_dmma<MAXR / 8, 4>(xs, zs, xs, cc0, cn0, nk, 0, nrows, R, orow);
                    else if (F == 2) flow_contract_dmma<MAXR / 8, 2>(xs, zs, xs, cc0, cn0, nk, 2 * part, nrows, R, orow);
                    else flow_contract_dmma<MAXR / 8, 1>(xs, zs, xs, cc0, cn0, nk, part, nrows, R, orow);
                    if (tr) trace_stamp(tr, 19, blockIdx.x == 0 && tid == 0 && it == 0);
                    // the tile's last item sums its superchunk partials (rocp.cpp:107: P += X_s Z)
                    if (tid == 0) {
                        unsigned prev;
                        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;"
                                     : "=r"(prev) : "l"(tile_ctr + st * p.maxtiles + tile) : "memory");
                        s_last = (prev + 1 == unsigned(b + 1) * unsigned(F * nsuper)) ? 1 : 0;
                    }
                    __syncthreads();
                    if (s_last) {
                        // every load of the thread's entries issued before the sums (a load-add
                        // chain per superchunk took ~3 us of L2 round trips)
                        double* W = wrows_of(st);
                        constexpr int kTE = (32 * MAXR + kChainThreads - 1) / kChainThreads;  // entries per thread
                        constexpr int kTU = kWideF ? 8 : 4;  // superchunk partials loaded up front
                        double cv[kTE][kTU], pv[kTE];
#pragma unroll
                        for (int u = 0; u < kTE; ++u) {
                            const int e = tid + u * kChainThreads;
                            const bool ok = e < nrows * R;
                            const int64_t o = int64_t(i0) * R + e;
#pragma unroll
                            for (int mm = 0; mm < kTU; ++mm)
                                cv[u][mm] = (ok && mm < nsuper) ? __ldcg(p.cpart + int64_t(mm) * rows * R + o) : 0.0;
                            pv[u] = (ok && st > 0) ? __ldcg(W + o) : 0.0;
                        }
#pragma unroll
                        for (int u = 0; u < kTE; ++u) {
                            const int e = tid + u * kChainThreads;
                            if (e < nrows * R) {
                                const int64_t o = int64_t(i0) * R + e;
                                double tot = cv[u][0];
#pragma unroll
                                for (int mm = 1; mm < kTU; ++mm)
                                    if (mm < nsuper) tot = tot + cv[u][mm];
                                for (int mm = kTU; mm < nsuper; ++mm) tot = tot + __ldcg(p.cpart + int64_t(mm) * rows * R + o);
                                W[o] = (st > 0) ? pv[u] + tot : tot;
                            }
                        }
                        __syncthreads();
                        if (tid == 0) {
                            publish(tsum_ctr + st, 1u);
                            if (tr) tr[6] = gtimer();  // the last tile sum of the stage overwrites
                        }
                    }
                    if (tr) trace_stamp(tr, 9, blockIdx.x == 0 && tid == 0 && it == 0);
                }
                if constexpr (kWideF) {  // the G^-1 in shared memory was overwritten by Z tiles
                    if (chunk_block && sg >= 1) {
                        stage_ginv(sg - 1);
                        __syncthreads();
                    }
                    materialise_prev();
                }
            } else {
                // ------------- the Gram finisher
                double* D = sm + kSmFact;  // the sweep's pivots (64)
                double* Gs = D + 64;       // R x R column-major
                double* colb = Gs + 64 * 64;  // 128: the sweep's column buffers
                double* gi = sm + 12288;   // G^-1 (row-major, symmetric)
                double qa[kQPre], qb[kQPre];
#pragma unroll
                for (int u = 0; u < kQPre; ++u) {
                    const int q = tid + u * kChainThreads;
                    qa[u] = qb[u] = 0.0;
                    if (st > 0 && q < npairs) {
                        const int i = pairs[q] >> 8, j = pairs[q] & 0xff;
                        qa[u] = __ldcg(p.Q[st - 1] + i + j * R);
                        qb[u] = __ldcg(p.Q[st - 1] + j + i * R);
                    }
                }
                if (gram_one) {
                    if (tid == 0) {  // every chunk partial of this stage published
                        wait_gathered(p.zctr, unsigned(sg + 1) * unsigned(nch), 0u, 0u);
                        asm volatile("fence.proxy.async.global;" ::: "memory");
                        const unsigned bytes = unsigned(nch * NPp * 8);
                        fence_proxy_async();
                        tma_load_1d(sm, p.chpart, bytes, &bar);
                        mbar_expect_tx(&bar, bytes);
                    }
                    if (tr) trace_stamp(tr, 3, tid == 0);
                    mbar_wait(&bar, phase);
                    phase ^= 1u;
                } else {  // every superchunk's Gram sum published
                    wait_ge(gsum_ctr, unsigned(sg + 1) * unsigned(nsuper));
                    __syncthreads();
                    if (tr) trace_stamp(tr, 3, tid == 0);
                }
#pragma unroll
                for (int u = 0; u < kMaxPairsPerThread; ++u) {
                    const int q = tid + u * kChainThreads;
                    if (q >= npairs) break;
                    double tot = 0.0;
                    if (gram_one) {
                        for (int m = 0; m < nsuper; ++m) {
                            const int k0 = m * kSuper, k1 = min(nch, k0 + kSuper);
                            double v[kSuper];
#pragma unroll
                            for (int k = 0; k < kSuper; ++k) v[k] = (k0 + k < k1) ? sm[(k0 + k) * NPp + q] : 0.0;
                            double sq = v[0];
#pragma unroll
                            for (int k = 1; k < kSuper; ++k)
                                if (k0 + k < k1) sq = sq + v[k];
                            tot = (m == 0) ? sq : tot + sq;
                        }
                    } else {  // the superchunk sums in order, every load first
                        double gv[kSuper];
#pragma unroll
                        for (int m = 0; m < kSuper; ++m) gv[m] = (m < nsuper) ? __ldcg(p.gpart + int64_t(m) * NPp + q) : 0.0;
                        tot = gv[0];
#pragma unroll
                        for (int m = 1; m < kSuper; ++m)
                            if (m < nsuper) tot = tot + gv[m];
                        for (int m = kSuper; m < nsuper; ++m) tot = tot + __ldcg(p.gpart + int64_t(m) * NPp + q);
                    }
                    const int i = pairs[q] >> 8, j = pairs[q] & 0xff;
                    double ga = tot, gb = tot;
                    if (st > 0) {  // Q + G entry by entry (rocp.cpp:108)
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
                // solve_gram (solve.cpp:9-35) in canonical form (kernels.cuh gram_solve_block)
                int2 mr;
                if constexpr (!kWideF) {
                    if (npairs <= 224) mr = gram_solve_block<1>(Gs, R, pairs, gi, colb, sm, true);
                    else if (npairs <= 448) mr = gram_solve_block<2>(Gs, R, pairs, gi, colb, sm, true);
                    else mr = gram_solve_block<3>(Gs, R, pairs, gi, colb, sm, true);
                } else {
                    if (npairs <= 1344) mr = gram_solve_block<6>(Gs, R, pairs, gi, colb, sm, true);
                    else mr = gram_solve_block<10>(Gs, R, pairs, gi, colb, sm, true);
                }
                if (tr) trace_stamp(tr, 11, tid == 0);
                double* slot = p.ginv + (sg & 1) * kGinvSlot;
                for (int t = tid; t < RR; t += kChainThreads) slot[t] = gi[t];
                if (tid == 0) {
                    p.gmode[sg & 1] = mr.x;
                    if (mr.y) atomicOr(p.flags + (st == 0 ? 0 : 2), 1);
                }
                __syncthreads();
                if (tid == 0) publish(fin_ctr, 1u);
                if (tr) trace_stamp(tr, 4, tid == 0);
            }
        }
    }
    // the last stage's rows, by every block
    {
        const int sl = p.nb * N - 1;
        const int bl = p.nb - 1, stl = N - 1;
        wait_ge(fin_ctr, unsigned(sl + 1));
        wait_ge(tsum_ctr + stl, unsigned(bl + 1) * unsigned(tiles_of(stl)));
        __syncthreads();
        stage_ginv(sl);
        __syncthreads();
        materialise(bl, stl, int(blockIdx.x) + warp * G, G * kW);
    }
}

}  // namespace rocpk
