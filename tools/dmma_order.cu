// Profiling aid: does the fp64 tensor-core MMA (mma.sync m8n8k4 f64) round like
// the canonical sample order of the contraction (a sequential fma
// chain over samples)?  Each trial draws A (8x4), B (4x8), C (8x8) and compares
// D = mma(A, B, C) bitwise with fma(a3,b3, fma(a2,b2, fma(a1,b1, fma(a0,b0,c))))
// (k increasing) and with the reverse order.  If the increasing chain matches on
// every trial, DMMA can carry the chunk partials without changing a bit.
#include <cuda_runtime.h>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <random>
#include <vector>

__global__ void k_mma(const double* A, const double* B, const double* C, double* D, int trials) {
    const int lane = threadIdx.x & 31;
    for (int t = blockIdx.x; t < trials; t += gridDim.x) {
        const double* a = A + t * 32;  // 8x4 row-major
        const double* b = B + t * 32;  // 4x8 row-major
        const double* c = C + t * 64;  // 8x8 row-major
        double* d = D + t * 64;
        const int r = lane >> 2, q = lane & 3;
        const double fa = a[r * 4 + q];            // A(r, q)
        const double fb = b[q * 8 + r];            // B(q, r)
        const double c0 = c[r * 8 + 2 * q], c1 = c[r * 8 + 2 * q + 1];
        double d0, d1;
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%4, %5};"
                     : "=d"(d0), "=d"(d1)
                     : "d"(fa), "d"(fb), "d"(c0), "d"(c1));
        d[r * 8 + 2 * q] = d0;
        d[r * 8 + 2 * q + 1] = d1;
    }
}

// throughput: each warp runs `iters` rounds of 8 independent m8n8k4 DMMAs (accumulator chains)
__global__ void k_dmma_tp(double* out, int iters) {
    const int lane = threadIdx.x & 31;
    double a = 1.0 + lane * 1e-3, b = 1.0 - lane * 1e-3;
    double d[8][2];
#pragma unroll
    for (int j = 0; j < 8; ++j) d[j][0] = d[j][1] = 0.0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                         : "+d"(d[j][0]), "+d"(d[j][1])
                         : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += d[j][0] + d[j][1];
    if (s == 1.2345) out[0] = s;
}
// the same flops as DFMA: 8 chains x 2 outputs x 4 products per lane per round = 64 fmas
__global__ void k_dfma_tp(double* out, int iters) {
    const int lane = threadIdx.x & 31;
    double a = 1.0 + lane * 1e-3, b = 1.0 - lane * 1e-3;
    double d[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) d[j] = 0.0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
            for (int j = 0; j < 16; ++j) d[j] = fma(a, b, d[j]);
    }
    double s = 0;
#pragma unroll
    for (int j = 0; j < 16; ++j) s += d[j];
    if (s == 1.2345) out[0] = s;
}

int main() {
    const int trials = 1 << 16;
    std::mt19937_64 g(5);
    std::normal_distribution<double> n01;
    std::vector<double> A(trials * 32), B(trials * 32), C(trials * 64), D(trials * 64);
    for (auto& x : A) x = n01(g);
    for (auto& x : B) x = n01(g);
    for (auto& x : C) x = n01(g) * 1e-3;
    double *dA, *dB, *dC, *dD;
    cudaMalloc(&dA, A.size() * 8);
    cudaMalloc(&dB, B.size() * 8);
    cudaMalloc(&dC, C.size() * 8);
    cudaMalloc(&dD, D.size() * 8);
    cudaMemcpy(dA, A.data(), A.size() * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dC, C.data(), C.size() * 8, cudaMemcpyHostToDevice);
    k_mma<<<592, 32>>>(dA, dB, dC, dD, trials);
    cudaMemcpy(D.data(), dD, D.size() * 8, cudaMemcpyDeviceToHost);
    printf("kernel: %s\n", cudaGetErrorString(cudaGetLastError()));
    long inc = 0, dec = 0, near = 0, total = 0;
    for (int t = 0; t < trials; ++t)
        for (int i = 0; i < 8; ++i)
            for (int j = 0; j < 8; ++j) {
                const double* a = &A[t * 32];
                const double* b = &B[t * 32];
                double s1 = C[t * 64 + i * 8 + j], s2 = s1;
                for (int k = 0; k < 4; ++k) s1 = std::fma(a[i * 4 + k], b[k * 8 + j], s1);
                for (int k = 3; k >= 0; --k) s2 = std::fma(a[i * 4 + k], b[k * 8 + j], s2);
                const double d = D[t * 64 + i * 8 + j];
                inc += d == s1;
                dec += d == s2;
                near += std::fabs(d - s1) <= 1e-12 * (1 + std::fabs(s1));
                ++total;
            }
    printf("outputs %ld: equal to the increasing fma chain %ld, to the decreasing chain %ld, within 1e-12 %ld\n", total,
           inc, dec, near);
    // throughput (148 SMs x 8 warps per block x 4 blocks)
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 20000;
    for (int v = 0; v < 2; ++v)
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            if (v == 0) k_dmma_tp<<<148 * 4, 256>>>(dD, iters);
            else k_dfma_tp<<<148 * 4, 256>>>(dD, iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double flops = 2.0 * 148 * 4 * 256 * double(iters) * 64;  // 64 fma per lane per round
            if (rep) printf("%s: %.3f ms, %.1f TFLOP/s fp64\n", v ? "DFMA" : "DMMA", ms, flops / ms / 1e9);
        }
    return 0;
}
