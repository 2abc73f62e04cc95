// Profiling aid: GPU zero-copy gather rate from pinned host memory over PCIe.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k_rand(const double* __restrict__ t, int64_t n_total, int64_t stride, double* out, int64_t n) {
    const int64_t tid = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    double acc = 0;
    for (int64_t e = tid; e < n; e += int64_t(gridDim.x) * blockDim.x) {
        uint64_t h = (uint64_t)e * 0x9E3779B97F4A7C15ull;
        int64_t off = int64_t((h >> 20) % uint64_t(n_total / stride)) * stride;
        acc += __ldcs(t + off);
    }
    if (acc == 1.2345) out[0] = acc;
}
__global__ void k_seq(const double* __restrict__ t, int64_t n, double* out) {
    const int64_t tid = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    double acc = 0;
    for (int64_t e = tid; e < n; e += int64_t(gridDim.x) * blockDim.x) acc += __ldcs(t + e);
    if (acc == 1.2345) out[0] = acc;
}
int main() {
    const int64_t total = int64_t(1) << 28;  // 2 GB host
    double* h; double* o;
    cudaHostAlloc(&h, total * 8, cudaHostAllocMapped);
    for (int64_t i = 0; i < total; i += 512) h[i] = 0;
    cudaMalloc(&o, 8);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int grid : {148 * 4, 148 * 16, 148 * 32}) {
        const int64_t n = 1 << 22;
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            k_rand<<<grid, 256>>>(h, total, 128, o, n);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            if (rep) printf("host random 8B reads (grid %d): %.3f ms, %.1f M reads/s (%s)\n", grid, ms, n / ms / 1e3, cudaGetErrorString(cudaGetLastError()));
        }
    }
    {
        const int64_t n = int64_t(1) << 27;
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            k_seq<<<148 * 16, 256>>>(h, n, o);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            if (rep) printf("host sequential reads: %.3f ms, %.1f GB/s\n", ms, n * 8 / ms / 1e6);
        }
        double* d; cudaMalloc(&d, n * 8);
        cudaEventRecord(a);
        cudaMemcpyAsync(d, h, n * 8, cudaMemcpyHostToDevice);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("cudaMemcpy H2D pinned: %.3f ms, %.1f GB/s\n", ms, n * 8 / ms / 1e6);
    }
    return 0;
}
