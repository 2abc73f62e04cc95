// Profiling aid: cost of a grid-wide barrier in a persistent kernel (148 blocks x 256).
//   V=0 cooperative_groups grid.sync()
//   V=1 sense-free counter barrier: thread 0 of each block does an atom.add.release.gpu on a
//       per-barrier-generation counter, then spins with ld.acquire.gpu until it reaches G
//   V=2 as V=1 with the arrival through red.release (no return value) and __nanosleep-free spin
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/barrier_bench.cu -o tools/barrier_bench
#include <cooperative_groups.h>
#include <cstdio>

namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

template <int V>
__global__ void __launch_bounds__(256, 1) k_bar(unsigned* counters, int iters, long long* out) {
    cg::grid_group grid = cg::this_grid();
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        if (V == 0) {
            grid.sync();
        } else {
            __syncthreads();
            if (threadIdx.x == 0) {
                unsigned* c = counters + (it & 1023);
                if (V == 1) {
                    unsigned old;
                    asm volatile("atom.add.release.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(c) : "memory");
                } else {
                    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(c) : "memory");
                }
                while (ld_acq(c) < gridDim.x) {
                }
            }
            __syncthreads();
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
}

template <int V>
void run(const char* name, unsigned* counters, long long* out, int G) {
    const int iters = 1000;
    for (int rep = 0; rep < 3; ++rep) {
        cudaMemset(counters, 0, 1024 * sizeof(unsigned));
        int it = iters;
        void* args[] = {&counters, &it, &out};
        cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(k_bar<V>), dim3(G), dim3(256), args, 0, 0);
        cudaDeviceSynchronize();
    }
    long long c;
    cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost);
    printf("%-40s %8.0f cycles per barrier  err=%s\n", name, double(c) / iters, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    int G = 0;
    cudaDeviceGetAttribute(&G, cudaDevAttrMultiProcessorCount, 0);
    unsigned* counters;
    long long* out;
    cudaMalloc(&counters, 1024 * sizeof(unsigned));
    cudaMalloc(&out, 8);
    run<0>("cooperative_groups grid.sync", counters, out, G);
    run<1>("atom.add.release + ld.acquire spin", counters, out, G);
    run<2>("red.release + ld.acquire spin", counters, out, G);
    return 0;
}
