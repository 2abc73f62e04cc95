// Profiling aid: cycles of the Gram-inverse sweep of the chain finisher (kernels.cuh sweep_block)
// on one block (148 independent blocks, block 0 timed with clock64), and a bitwise check of the
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

// the block sweep (kernels.cuh sweep_block), block 0 timed
template <int MAXR>
__global__ void __launch_bounds__(256, 1) k_bench(const double* G, int R, int mode, int reps, long long* cyc, double* out) {
    extern __shared__ double sm[];
    const int tid = threadIdx.x;
    double* Gs = sm;               // 64 x 64
    double* colb = Gs + 64 * 64;   // 128
    double* gi = colb + 128;       // 4096
    double* dd = gi + 4096;        // 2
    for (int t = tid; t < R * R; t += blockDim.x) Gs[t] = G[t];
    __syncthreads();
    for (int rep = 0; rep < reps; ++rep) {
        const long long t0 = clock64();
        const int np = R * (R + 1) / 2;
        if (mode == 1) {
            double* jscr = dd + 8;
            if (np <= 224) gram_solve_block<1>(Gs, R, nullptr, gi, colb, jscr, false);
            else if (np <= 448) gram_solve_block<2>(Gs, R, nullptr, gi, colb, jscr, false);
            else if (np <= 672) gram_solve_block<3>(Gs, R, nullptr, gi, colb, jscr, false);
            else gram_solve_block<6>(Gs, R, nullptr, gi, colb, jscr, false);
        } else if (np <= 224) sweep_block<1>(Gs, 0.0, R, nullptr, colb, gi, dd, dd + 1);
        else if (np <= 448) sweep_block<2>(Gs, 0.0, R, nullptr, colb, gi, dd, dd + 1);
        else if (np <= 672) sweep_block<3>(Gs, 0.0, R, nullptr, colb, gi, dd, dd + 1);
        else sweep_block<6>(Gs, 0.0, R, nullptr, colb, gi, dd, dd + 1);
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
    const int smem = (4096 + 128 + 4096 + 8 + 4096 + 128) * 8;
    cudaFuncSetAttribute(k_bench<MAXR>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const char* names[2] = {"sweep_block", "gram_solve_block"};
    for (int mode = 0; mode < 2; ++mode) {
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
