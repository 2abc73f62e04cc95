// Profiling aid: cold (first call in the kernel) vs warm (second call) cycles of
// the chain's straight-line device functions, to size instruction-fetch cost.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -fmad=false tools/icache_bench.cu -o tools/icache_bench
#include <cstdio>
#include "../paper_2007_10798_b200/csrc/chain_kernel.cuh"
using namespace rocpk;

__global__ void k_cold_warm(const double* G, int R, long long* cyc) {
    extern __shared__ double sm[];
    double* Gs = sm + 64 * kLdStride + 64;
    for (int t = threadIdx.x; t < R * R; t += blockDim.x) Gs[t] = G[t];
    __syncthreads();
    for (int rep = 0; rep < 2; ++rep) {
        __syncthreads();
        long long t0 = clock64();
        if (threadIdx.x < 32) ldlt_warp<32>(Gs, 0.0, R, sm, kLdStride, sm + 64 * kLdStride, Gs + R * R, nullptr);
        __syncthreads();
        long long t1 = clock64();
        if (threadIdx.x == 0) cyc[rep] = t1 - t0;
    }
}

// ncu source-level sampling target: ldlt_warp<24> at R = 20, 2000 times in one launch
__global__ void k_ldlt_loop(const double* G, int R, double* out) {
    extern __shared__ double sm[];
    double* Gs = sm + 64 * kLdStride + 64;
    for (int t = threadIdx.x; t < R * R; t += blockDim.x) Gs[t] = G[t];
    __syncwarp();
    double acc = 0.0;
    for (int rep = 0; rep < 2000; ++rep) {
        ldlt_warp<24>(Gs, 1e-3 * rep, R, sm, kLdStride, sm + 64 * kLdStride, Gs + R * R, nullptr);
        __syncwarp();
        acc += sm[64 * kLdStride + R - 1];
    }
    if (threadIdx.x == 0) out[0] = acc;
}

int run_loop() {
    const int R = 20;
    double h[64 * 64];
    for (int i = 0; i < R; ++i)
        for (int j = 0; j < R; ++j) h[i + j * R] = (i == j ? R + 1.0 : 0.5 / (1 + i + j));
    double *G, *o;
    cudaMalloc(&G, sizeof(h));
    cudaMalloc(&o, 8);
    cudaMemcpy(G, h, sizeof(h), cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(k_ldlt_loop, cudaFuncAttributeMaxDynamicSharedMemorySize, 120000);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k_ldlt_loop<<<1, 32, 120000>>>(G, R, o);
    cudaEventRecord(a);
    k_ldlt_loop<<<1, 32, 120000>>>(G, R, o);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    printf("ldlt_warp<24> R=%d: %.1f ns per factorization (%.1f ns per pivot)\n", R, ms * 1e6 / 2000,
           ms * 1e6 / 2000 / R);
    return 0;
}

// The Gram finisher's shape: warp 0 factors, warp 1 lane 0 scans the diagonal,
// block barrier; 'stamp' adds the trace build's tid-0 global store before it.
__global__ void k_finisher(const double* G, int R, long long* cyc, double* gtr, int stamp) {
    extern __shared__ double sm[];
    __shared__ double s_tr;
    __shared__ int s_mode;
    double* A = sm;
    double* D = A + 64 * kLdStride;
    double* Gs = D + 64;
    double* colb = Gs + 64 * 64;
    for (int t = threadIdx.x; t < R * R; t += blockDim.x) Gs[t] = G[t];
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int rep = 0; rep < 2; ++rep) {
        __syncthreads();
        long long t0 = clock64();
        if (stamp && threadIdx.x == 0) gtr[rep] = double(t0);
        __syncwarp();
        if (warp == 0) {
            ldlt_warp<24>(Gs, 0.0, R, A, kLdStride, D, colb, D + 62);
        } else if (warp == 1) {
            if (lane == 0) {
                double maxdiag = Gs[0], trc = Gs[0];
                for (int k = 1; k < R; ++k) {
                    const double dg = Gs[k * R + k];
                    if (dg > maxdiag) maxdiag = dg;
                    trc = trc + dg;
                }
                s_tr = trc;
                s_mode = (maxdiag <= 0.0) ? 0 : 1;
            }
            __syncwarp();
        }
        __syncthreads();
        long long t1 = clock64();
        if (threadIdx.x == 0) cyc[rep] = t1 - t0;
    }
}

int run_finisher() {
    const int R = 20;
    double h[64 * 64];
    for (int i = 0; i < R; ++i)
        for (int j = 0; j < R; ++j) h[i + j * R] = (i == j ? R + 1.0 : 0.5 / (1 + i + j));
    double *G, *gtr;
    long long* c;
    cudaMalloc(&G, sizeof(h));
    cudaMalloc(&gtr, 16);
    cudaMalloc(&c, 16);
    cudaMemcpy(G, h, sizeof(h), cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(k_finisher, cudaFuncAttributeMaxDynamicSharedMemorySize, 120000);
    for (int stamp = 0; stamp < 2; ++stamp) {
        k_finisher<<<1, 256, 120000>>>(G, R, c, gtr, stamp);
        long long cyc[2];
        cudaMemcpy(cyc, c, sizeof(cyc), cudaMemcpyDeviceToHost);
        printf("finisher shape, stamp=%d: %lld / %lld cycles  err=%s\n", stamp, cyc[0], cyc[1],
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}

int run_loop();
int run_finisher();
int main(int argc, char** argv) {
    if (argc > 1 && argv[1][0] == 'f') return run_finisher();
    if (argc > 1) return run_loop();
    const int R = 20;
    double h[64 * 64];
    for (int i = 0; i < R; ++i)
        for (int j = 0; j < R; ++j) h[i + j * R] = (i == j ? R + 1.0 : 0.5 / (1 + i + j));
    double* G;
    long long* c;
    cudaMalloc(&G, sizeof(h));
    cudaMalloc(&c, 2 * 8);
    cudaMemcpy(G, h, sizeof(h), cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(k_cold_warm, cudaFuncAttributeMaxDynamicSharedMemorySize, 120000);
    for (int launch = 0; launch < 3; ++launch) {
        k_cold_warm<<<1, 256, 120000>>>(G, R, c);
        long long cyc[2];
        cudaMemcpy(cyc, c, sizeof(cyc), cudaMemcpyDeviceToHost);
        printf("launch %d R=%d ldlt_warp<32>: cold %lld warm %lld cycles  err=%s\n", launch, R, cyc[0], cyc[1],
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}


