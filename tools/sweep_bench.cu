// Profiling aid: cycles of the Gram-inverse variants of the chain finisher on one warp /
// block (148 independent blocks, block 0 timed with clock64), and a bitwise check of the
// sweep against a host restatement of the canonical order (oracle gram_sweep).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>
#include "../paper_2007_10798_b200/csrc/flow_kernel.cuh"
using namespace rocpk;

static std::vector<double> host_sweep(const std::vector<double>& g, int R) {
    std::vector<double> A = g, gi(size_t(R) * R);  // lower triangle used: A(i, j), i >= j
    for (int k = 0; k < R; ++k) {
        std::vector<double> c(R);
        for (int x = 0; x < R; ++x) c[x] = (x >= k) ? A[x + k * R] : A[k + x * R];
        const double d = c[k];
        const double r = (std::fabs(d) > 2.2250738585072014e-308) ? 1.0 / d : 0.0;
        for (int j = 0; j < R; ++j)
            for (int i = j; i < R; ++i) {
                double& a = A[i + j * R];
                if (j == k) a = (i == k) ? -r : c[i] * r;
                else if (i == k) a = std::fma(c[j], r, 0.0);
                else a = std::fma(-(c[i] * r), c[j], a);
            }
    }
    for (int j = 0; j < R; ++j)
        for (int i = j; i < R; ++i) gi[i * R + j] = gi[j * R + i] = -A[i + j * R];
    return gi;
}

// experiment variants of sweep_warp: V bit0: __drcp_rn; bit1: select instead of divergent
// zeroing; bit2: no reciprocal at all (timing only)
template <int MAXR, int V>
__device__ __noinline__ void sweep_warp_x(const double* G, double lambda, int R, double* gi, double* cbuf) {
    const int lane = threadIdx.x & 31;
    double a[MAXR];
#pragma unroll
    for (int j = 0; j < MAXR; ++j) {
        const bool ok = lane < R && j < R;
        const double g = G[ok ? lane + j * R : 0];
        a[j] = ok ? ((j == lane) ? g + lambda : g) : 0.0;
    }
    cbuf[lane] = a[0];
    __syncwarp();
#pragma unroll
    for (int k = 0; k < MAXR; ++k) {
        if (k < R) {
            const double* c = cbuf + (k & 1) * 32;
            double cv[MAXR];
#pragma unroll
            for (int j = 0; j < MAXR; ++j) cv[j] = c[j];
            const double d = cv[k];
            double r;
            if (V & 4) r = d * 0.5;
            else if (V & 1) r = (fabs(d) > 2.2250738585072014e-308) ? __drcp_rn(d) : 0.0;
            else r = (fabs(d) > 2.2250738585072014e-308) ? 1.0 / d : 0.0;
            const bool me = lane == k;
            const double l = a[k] * r;
            const double mult = me ? r : -l;
            if (!(V & 2)) {
                if (me) {
#pragma unroll
                    for (int j = 0; j < MAXR; ++j) a[j] = 0.0;
                }
            }
            if (k + 1 < MAXR) {
                a[k + 1] = __fma_rn(cv[k + 1], mult, (V & 2) ? (me ? 0.0 : a[k + 1]) : a[k + 1]);
                cbuf[((k + 1) & 1) * 32 + lane] = a[k + 1];
            }
#pragma unroll
            for (int j = 0; j < MAXR; ++j)
                if (j != k && j != k + 1) a[j] = __fma_rn(cv[j], mult, (V & 2) ? (me ? 0.0 : a[j]) : a[j]);
            a[k] = me ? -r : l;
            __syncwarp();
        }
    }
    if (lane < R) {
#pragma unroll
        for (int j = 0; j < MAXR; ++j)
            if (j < R) gi[lane * R + j] = -a[j];
    }
}

// mode 0: ldlt_warp + flow_ginv (current); 1: sweep_warp; 2: sweep_block
template <int MAXR>
__global__ void __launch_bounds__(256, 1) k_bench(const double* G, int R, int mode, int reps, long long* cyc, double* out) {
    extern __shared__ double sm[];
    __shared__ unsigned short pairs[32 * 33 / 2];
    const int tid = threadIdx.x;
    if (tid == 0) {
        int off = 0;
        for (int j = 0; j < R; ++j)
            for (int i = j; i < R; ++i) pairs[off++] = (unsigned short)((i << 8) | j);
    }
    double* A = sm;                       // 64 x 65
    double* D = A + 64 * kLdStride;       // 64
    double* Gs = D + 64;                  // 64 x 64
    double* colb = Gs + 64 * 64;          // 96 + 64
    double* ms = colb + 256;              // 1024
    double* gi = ms + 4096;               // 4096
    for (int t = tid; t < R * R; t += blockDim.x) Gs[t] = G[t];
    __syncthreads();
    for (int rep = 0; rep < reps; ++rep) {
        const long long t0 = clock64();
        if (mode == 0) {
            if (tid < 32) ldlt_warp<MAXR>(Gs, 0.0, R, A, kLdStride, D, colb, D + 61);
            __syncthreads();
            flow_ginv<MAXR>(A, kLdStride, D, R, ms, colb + 96, gi, pairs, R * (R + 1) / 2);
        } else if (mode == 1) {
            if (tid < 32) sweep_warp<MAXR>(Gs, 0.0, R, gi, colb, D + 61, D);
            __syncthreads();
        } else if (mode == 2) {
            const int np = R * (R + 1) / 2;
            if (np <= 256) sweep_block<1>(Gs, 0.0, R, colb, gi, D);
            else if (np <= 512) sweep_block<2>(Gs, 0.0, R, colb, gi, D);
            else if (np <= 768) sweep_block<3>(Gs, 0.0, R, colb, gi, D);
            else sweep_block<5>(Gs, 0.0, R, colb, gi, D);
        } else {
            if (tid < 32) {
                if (mode == 3) sweep_warp_x<MAXR, 1>(Gs, 0.0, R, gi, colb);
                else if (mode == 4) sweep_warp_x<MAXR, 3>(Gs, 0.0, R, gi, colb);
                else if (mode == 5) sweep_warp_x<MAXR, 2>(Gs, 0.0, R, gi, colb);
                else sweep_warp_x<MAXR, 6>(Gs, 0.0, R, gi, colb);
            }
            __syncthreads();
        }
        const long long t1 = clock64();
        if (blockIdx.x == 0 && tid == 0) cyc[rep] = t1 - t0;
        __syncthreads();
    }
    if (blockIdx.x == 0)
        for (int t = tid; t < R * R; t += blockDim.x) out[t] = gi[t];
}

template <int MAXR>
void run(int R, std::mt19937_64& gen) {
    std::normal_distribution<double> nd;
    const int S = 600;
    std::vector<double> z(size_t(S) * R), g(size_t(R) * R, 0.0);
    for (auto& v : z) v = nd(gen);
    for (int i = 0; i < R; ++i)
        for (int j = 0; j < R; ++j) {
            double a = 0.0;
            for (int s = 0; s < S; ++s) a = std::fma(z[s * R + i], z[s * R + j], a);
            g[i + j * R] = a;
        }
    for (int i = 0; i < R; ++i)
        for (int j = 0; j < i; ++j) g[j + i * R] = g[i + j * R];
    const std::vector<double> ref = host_sweep(g, R);
    double *dG, *dout;
    long long* dc;
    cudaMalloc(&dG, g.size() * 8);
    cudaMalloc(&dout, 64 * 64 * 8);
    cudaMalloc(&dc, 64 * 8);
    cudaMemcpy(dG, g.data(), g.size() * 8, cudaMemcpyHostToDevice);
    const int smem = (64 * 65 + 64 + 4096 + 256 + 4096 + 4096) * 8;
    cudaFuncSetAttribute(k_bench<MAXR>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const char* names[7] = {"ldlt_warp+flow_ginv", "sweep_warp", "sweep_block", "sweep drcp", "sweep drcp+sel", "sweep sel", "sweep sel no-rcp"};
    for (int mode = 0; mode < 7; ++mode) {
        if (R > 32 && mode != 2) continue;
        k_bench<MAXR><<<148, 256, smem>>>(dG, R, mode, 6, dc, dout);
        cudaError_t e = cudaDeviceSynchronize();
        long long c[6];
        cudaMemcpy(c, dc, sizeof(c), cudaMemcpyDeviceToHost);
        std::vector<double> o(size_t(R) * R);
        cudaMemcpy(o.data(), dout, o.size() * 8, cudaMemcpyDeviceToHost);
        double maxrel = 0.0;
        bool bit = true;
        for (int t = 0; t < R * R; ++t) {
            if (std::memcmp(&o[t], &ref[t], 8) != 0) bit = false;
            maxrel = std::fmax(maxrel, std::fabs(o[t] - ref[t]) / std::fabs(ref[t] + 1e-300));
        }
        printf("R=%d %-22s cold %6lld  warm %6lld %6lld cycles  bitwise-vs-sweep=%d maxrel=%.2e %s\n", R, names[mode], c[0],
               c[3], c[5], int(bit), maxrel, cudaGetErrorString(e));
    }
    cudaFree(dG);
    cudaFree(dout);
    cudaFree(dc);
}

int main() {
    std::mt19937_64 gen(7);
    run<16>(10, gen);
    run<16>(16, gen);
    run<24>(20, gen);
    run<32>(32, gen);
    run<32>(50, gen);
    return 0;
}
