// Latency micro-benchmarks on the B200 (profiling aid, not product code).
#include <cstdio>
#include <cuda_runtime.h>
#include <cooperative_groups.h>

__global__ void k_fma_chain(double* out, double a, double b, int n, long long* cyc) {
    double x = out[threadIdx.x];
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = __fma_rn(x, a, b);
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_div_chain(double* out, double d, int n, long long* cyc) {
    double x = out[threadIdx.x] + 1.0;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = d / x;
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_sync(int n, long long* cyc) {
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_shfl(double* out, int n, long long* cyc) {
    double x = out[threadIdx.x];
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = __shfl_sync(0xffffffffu, x, (i + 1) & 31) + 1.0;
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_lds_chain(int n, long long* cyc, int* outp) {
    __shared__ int buf[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) buf[i] = (i + 1) & 1023;
    __syncthreads();
    int x = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = buf[x];
    long long t1 = clock64();
    outp[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_gridsync(int n, long long* cyc) {
    namespace cg = cooperative_groups;
    cg::grid_group g = cg::this_grid();
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) g.sync();
    long long t1 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_fma_tput(double* out, double a, double b, int n, long long* cyc) {
    double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        x0 = __fma_rn(x0, a, b); x1 = __fma_rn(x1, a, b); x2 = __fma_rn(x2, a, b); x3 = __fma_rn(x3, a, b);
        x4 = __fma_rn(x4, a, b); x5 = __fma_rn(x5, a, b); x6 = __fma_rn(x6, a, b); x7 = __fma_rn(x7, a, b);
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
    if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}

int main1() {
    double* d; long long* c; int* ip; long long h;
    cudaMalloc(&d, 1 << 24); cudaMalloc(&c, 64); cudaMalloc(&ip, 1 << 16);
    cudaMemset(d, 0, 1 << 24);
    const int n = 4096;
    k_fma_chain<<<1, 32>>>(d, 0.999, 0.5, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("DFMA dependent latency: %.2f cycles\n", double(h) / n);
    k_div_chain<<<1, 32>>>(d, 1.7, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("fp64 division dependent latency: %.2f cycles\n", double(h) / n);
    k_sync<<<1, 256>>>(n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("__syncthreads (256 thr): %.2f cycles\n", double(h) / n);
    k_shfl<<<1, 32>>>(d, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("shfl+dadd dependent: %.2f cycles\n", double(h) / n);
    k_lds_chain<<<1, 32>>>(n, c, ip); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("LDS dependent latency: %.2f cycles\n", double(h) / n);
    for (int warps : {1, 2, 4, 8, 16}) {
        k_fma_tput<<<1, 32 * warps>>>(d, 0.999, 0.5, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("DFMA throughput, %2d warps/SM: %.2f warp-DFMA/cycle\n", warps, 8.0 * n * warps / double(h));
    }
    int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    int m = 256; void* args[] = {&m, &c};
    cudaLaunchCooperativeKernel((void*)k_gridsync, nsm, 256, args, 0, 0);
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("grid.sync (%d blocks x 256): %.2f cycles\n", nsm, double(h) / m);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("clock rate attr: %d kHz; err=%s\n", clk, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
// (appended) fence / atomic latency
__global__ void k_fence(int n, long long* cyc, unsigned* ctr) {
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) { __threadfence(); }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
    t0 = clock64();
    unsigned v = 0;
    for (int i = 0; i < n; ++i) { v += atomicAdd(ctr, 1u); }
    t1 = clock64();
    if (threadIdx.x == 0) { cyc[1] = t1 - t0; cyc[2] = v; }
}
int main2() {
    long long* c; unsigned* u; long long h[3];
    cudaMalloc(&c, 64); cudaMalloc(&u, 64); cudaMemset(u, 0, 64);
    k_fence<<<1, 32>>>(256, c, u);
    cudaMemcpy(h, c, 24, cudaMemcpyDeviceToHost);
    printf("__threadfence: %.1f cycles, atomicAdd (returning) %.1f cycles\n", h[0] / 256.0, h[1] / 256.0);
    k_fence<<<148, 256>>>(64, c, u);
    cudaMemcpy(h, c, 24, cudaMemcpyDeviceToHost);
    printf("under load (148x256): __threadfence %.1f cycles, atomicAdd %.1f cycles\n", h[0] / 64.0, h[1] / 64.0);
    return 0;
}
int main() { main1(); return main2(); }
