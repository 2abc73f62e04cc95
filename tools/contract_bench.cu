// Profiling aid: cycles of one contraction item (32 rows x 256 samples x RP) in shared memory,
// register-blocked DFMA (chain_contract_blocked) vs fp64 mma.sync (chain_contract_dmma), and a
// bitwise comparison of their outputs.
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>
#include "../paper_2007_10798_b200/csrc/chain_kernel.cuh"
using namespace rocpk;


// the MMA loop of chain_contract_dmma alone (no cross-warp reduction), timing aid
template <int NT>
__device__ __noinline__ void mma_only(const double* xs, const double* zs, int cc0, int ccn, double* sink) {
    constexpr int RP = 8 * NT;
    const int lane = threadIdx.x & 31;
    const int q = lane & 3, rr = lane >> 2;
    double acc[4][NT][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int n = 0; n < NT; ++n) acc[a][n][0] = acc[a][n][1] = 0.0;
    for (int k0 = 0; k0 < ccn; k0 += 4) {
        const int smp = cc0 + k0 + q;
        double fa[4], fb[NT];
#pragma unroll
        for (int a = 0; a < 4; ++a) fa[a] = xs[smp * 32 + a * 8 + rr];
#pragma unroll
        for (int n = 0; n < NT; ++n) fb[n] = zs[smp * RP + n * 8 + rr];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int n = 0; n < NT; ++n)
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                             : "+d"(acc[a][n][0]), "+d"(acc[a][n][1])
                             : "d"(fa[a]), "d"(fb[n]));
    }
    double t = 0.0;
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int n = 0; n < NT; ++n) t += acc[a][n][0] + acc[a][n][1];
    if (t == 1.2345) *sink = t;
}

template <int RP>
__global__ void __launch_bounds__(256, 1) k_item(const double* X, const double* Z, int R, int mode, int reps, long long* cyc,
                                                 double* out) {
    extern __shared__ double sm[];
    double* xs = sm;          // [256][32]
    double* zs = sm + 8192;   // [256][RP]
    const int tid = threadIdx.x, warp = tid >> 5;
    double* o = out + blockIdx.x * 32 * R;
    for (int rep = 0; rep < reps; ++rep) {
        for (int t = tid; t < 8192; t += 256) xs[t] = X[t];
        for (int t = tid; t < 256 * RP; t += 256) zs[t] = Z[t];
        __syncthreads();
        const long long t0 = clock64();
        if (mode == 0) chain_contract_blocked<RP / 4>(xs, zs, xs, warp * 32, 32, 8, 32, R, o);
        else if (mode == 1) chain_contract_dmma<RP / 8>(xs, zs, xs, warp * 32, 32, 8, 32, R, o);
        else mma_only<RP / 8>(xs, zs, warp * 32, 32, o);
        __syncthreads();
        const long long t1 = clock64();
        if (blockIdx.x == 0 && tid == 0) cyc[rep] = t1 - t0;
    }
}

template <int RP>
void run(int R) {
    std::mt19937_64 g(3);
    std::normal_distribution<double> nd;
    std::vector<double> x(8192), z(256 * RP, 0.0);
    for (auto& v : x) v = nd(g);
    for (int s = 0; s < 256; ++s)
        for (int r = 0; r < R; ++r) z[s * RP + r] = nd(g);
    double *dx, *dz, *dout;
    long long* dc;
    cudaMalloc(&dx, x.size() * 8);
    cudaMalloc(&dz, z.size() * 8);
    cudaMalloc(&dout, 148 * 32 * 64 * 8);
    cudaMalloc(&dc, 8 * 8);
    cudaMemcpy(dx, x.data(), x.size() * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dz, z.data(), z.size() * 8, cudaMemcpyHostToDevice);
    const int smem = (8192 + 256 * RP) * 8;
    cudaFuncSetAttribute(k_item<RP>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    std::vector<double> o0(32 * R), o1(32 * R);
    for (int mode = 0; mode < 3; ++mode) {
        k_item<RP><<<148, 256, smem>>>(dx, dz, R, mode, 5, dc, dout);
        cudaError_t e = cudaDeviceSynchronize();
        long long c[5];
        cudaMemcpy(c, dc, sizeof(c), cudaMemcpyDeviceToHost);
        if (mode < 2) cudaMemcpy(mode ? o1.data() : o0.data(), dout, 32 * R * 8, cudaMemcpyDeviceToHost);
        const double fl = 2.0 * 32 * 256 * R;
        printf("R=%d RP=%d %s: %lld cycles (%.1f flop/clk/SM) %s\n", R, RP, mode == 2 ? "mma-only" : (mode ? "dmma   " : "blocked"), c[4], fl / c[4],
               cudaGetErrorString(e));
    }
    printf("  bitwise equal: %d\n", int(std::memcmp(o0.data(), o1.data(), o0.size() * 8) == 0));
}

int main() {
    run<16>(16);
    run<24>(20);
    run<32>(32);
    run<56>(50);
    return 0;
}
