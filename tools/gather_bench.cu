// Profiling aid: DRAM fetch granularity of isolated 8-byte loads per PTX load flavour.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int V>
__device__ __forceinline__ double ld(const double* p) {
    double v;
    if (V == 0) asm volatile("ld.global.f64 %0, [%1];" : "=d"(v) : "l"(p));
    if (V == 1) asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(v) : "l"(p));
    if (V == 2) asm volatile("ld.global.cs.f64 %0, [%1];" : "=d"(v) : "l"(p));
    if (V == 3) asm volatile("ld.global.L2::64B.f64 %0, [%1];" : "=d"(v) : "l"(p));
    if (V == 4) asm volatile("ld.global.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
    if (V == 5) asm volatile("ld.global.lu.f64 %0, [%1];" : "=d"(v) : "l"(p));
    if (V == 6) asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}

template <int V>
__global__ void k_g(const double* __restrict__ t, int64_t n_elems_total, int64_t stride, double* out, int64_t n) {
    const int64_t tid = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    double acc = 0;
    for (int64_t e = tid; e < n; e += int64_t(gridDim.x) * blockDim.x) {
        // pseudo-random 8-byte element, far apart (like strided fibre elements)
        uint64_t h = (uint64_t)e * 0x9E3779B97F4A7C15ull;
        int64_t off = int64_t((h >> 20) % uint64_t(n_elems_total / stride)) * stride;
        acc += ld<V>(t + off);
    }
    if (acc == 1.2345) out[0] = acc;
}

int main() {
    const int64_t total = int64_t(1) << 29;  // 4 GB of doubles
    double* t; double* o;
    cudaMalloc(&t, total * 8); cudaMalloc(&o, 8);
    cudaMemset(t, 0, total * 8);
    const int64_t n = 1 << 24;  // 16M loads
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const char* names[] = {"ld.global", "ld.global.nc", "ld.global.cs", "ld.global.L2::64B", "ld.global.L1::no_allocate", "ld.global.lu", "ld.global.cg"};
    for (int v = 0; v < 7; ++v) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            switch (v) {
                case 0: k_g<0><<<148 * 8, 256>>>(t, total, 16, o, n); break;
                case 1: k_g<1><<<148 * 8, 256>>>(t, total, 16, o, n); break;
                case 2: k_g<2><<<148 * 8, 256>>>(t, total, 16, o, n); break;
                case 3: k_g<3><<<148 * 8, 256>>>(t, total, 16, o, n); break;
                case 4: k_g<4><<<148 * 8, 256>>>(t, total, 16, o, n); break;
                case 5: k_g<5><<<148 * 8, 256>>>(t, total, 16, o, n); break;
                case 6: k_g<6><<<148 * 8, 256>>>(t, total, 16, o, n); break;
            }
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            if (rep) printf("%-28s %8.3f ms  %7.2f G loads/s  (%s)\n", names[v], ms, n / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
