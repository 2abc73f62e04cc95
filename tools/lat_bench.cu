// Profiling aid: dependent-chain latencies on this GPU (one warp): DFMA, DFMA+FSEL, LDS->DFMA.
#include <cstdio>
__global__ void k_lat(double* out, long long* cyc, int n, double x0) {
    __shared__ double s[64];
    if (threadIdx.x < 64) s[threadIdx.x] = 1.0 + threadIdx.x * 1e-3;
    __syncthreads();
    double a = x0, b = 1.0000001;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) a = __fma_rn(a, b, 1e-9);
    }
    long long t1 = clock64();
    double c = x0;
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            const double v = __fma_rn(c, b, 1e-9);
            c = (u < n) ? v : c;
        }
    }
    long long t2 = clock64();
    double d = x0;
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) d = __fma_rn(s[(u + i) & 63], d, 1e-9);
    }
    long long t3 = clock64();
    float f = float(x0);
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) f = __fmaf_rn(f, 1.0000001f, 1e-9f);
    }
    long long t4 = clock64();
    if (threadIdx.x == 0) {
        cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3;
    }
    out[threadIdx.x] = a + c + d + f;
}
int main() {
    double* o; long long* c;
    cudaMalloc(&o, 1024 * 8); cudaMalloc(&c, 64);
    const int n = 64;
    for (int rep = 0; rep < 2; ++rep) {
        k_lat<<<1, 32>>>(o, c, n, 1.0);
        cudaDeviceSynchronize();
        long long h[4];
        cudaMemcpy(h, c, 32, cudaMemcpyDeviceToHost);
        const double m = 16.0 * n;
        printf("per dependent op: DFMA %.1f  DFMA+FSEL %.1f  LDS->DFMA %.1f  FFMA %.1f cycles\n", h[0] / m, h[1] / m, h[2] / m, h[3] / m);
    }
    return 0;
}
