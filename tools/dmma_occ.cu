// Profiling aid: fp64 mma.sync m8n8k4 throughput per SM against the number of resident warps
// and of independent accumulator chains per warp (one block per SM, register operands).
#include <cstdio>
#include <cuda_runtime.h>

template <int NACC>
__global__ void k_dmma(double* out, int iters) {
    const int lane = threadIdx.x & 31;
    double a = 1.0 + lane * 1e-3, b = 1.0 - lane * 1e-3;
    double d[NACC][2];
#pragma unroll
    for (int j = 0; j < NACC; ++j) d[j][0] = d[j][1] = 0.0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < NACC; ++j)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                         : "+d"(d[j][0]), "+d"(d[j][1])
                         : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int j = 0; j < NACC; ++j) s += d[j][0] + d[j][1];
    if (s == 1.2345) out[0] = s;
}

template <int NACC>
void run(double* d, int warps) {
    const int total = 1 << 16;  // DMMAs per warp
    const int iters = total / NACC;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_dmma<NACC><<<148, warps * 32>>>(d, iters);
    cudaEventRecord(e0);
    k_dmma<NACC><<<148, warps * 32>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 148.0 * warps * double(iters) * NACC * 512.0;
    printf("warps/SM %2d acc/warp %2d: %.1f TFLOP/s (%.1f clk per DMMA per SMSP at 1.965 GHz)\n", warps, NACC,
           flops / ms / 1e9, ms * 1e-3 * 1.965e9 / (double(iters) * NACC * warps / 4.0));
}

int main() {
    double* d;
    cudaMalloc(&d, 64);
    for (int w : {4, 8, 16, 32}) {
        run<1>(d, w);
        run<2>(d, w);
        run<4>(d, w);
        run<8>(d, w);
        run<14>(d, w);
    }
    return 0;
}
