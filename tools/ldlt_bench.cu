// Profiling aid: cycles of the canonical LDL^T variants on one block.
#include <cstdio>
#include "../paper_2007_10798_b200/csrc/chain_kernel.cuh"
using namespace rocpk;

__global__ void k_ldlt(const double* G, int R, long long* cyc, double* out) {
    extern __shared__ double sm[];
    __shared__ unsigned short pairs[64 * 65 / 2];
    if (threadIdx.x == 0) {
        int off = 0;
        for (int j = 0; j < R; ++j)
            for (int i = j; i < R; ++i) pairs[off++] = (unsigned short)((i << 8) | j);
    }
    double* Gs = sm + 64 * kLdStride + 64;
    for (int t = threadIdx.x; t < R * R; t += blockDim.x) Gs[t] = G[t];
    __syncthreads();
    long long t0 = clock64();
    ldlt_one_sync(sm, sm + 64 * kLdStride, R, 0.0, Gs, pairs, R * (R + 1) / 2);
    long long t1 = clock64();
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; out[0] = sm[64 * kLdStride + R - 1]; }
}

__global__ void k_ldlt_warp(const double* G, int R, long long* cyc, double* out) {
    extern __shared__ double sm[];
    double* Gs = sm + 64 * kLdStride + 64;
    for (int t = threadIdx.x; t < R * R; t += blockDim.x) Gs[t] = G[t];
    __syncthreads();
    long long t0 = clock64();
    if (threadIdx.x < 32) {
        if (R <= 16) ldlt_warp<16>(Gs, 0.0, R, sm, kLdStride, sm + 64 * kLdStride, Gs + R * R, nullptr);
        else ldlt_warp<32>(Gs, 0.0, R, sm, kLdStride, sm + 64 * kLdStride, Gs + R * R, nullptr);
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; out[0] = sm[64 * kLdStride + R - 1]; }
}

int main() {
    for (int R : {10, 16, 20, 50}) {
        double h[64 * 64];
        for (int i = 0; i < R; ++i)
            for (int j = 0; j < R; ++j) h[i + j * R] = (i == j ? R + 1.0 : 0.5 / (1 + i + j));
        double* G; long long* c; double* o;
        cudaMalloc(&G, sizeof(h)); cudaMalloc(&c, 8); cudaMalloc(&o, 8);
        cudaMemcpy(G, h, sizeof(h), cudaMemcpyHostToDevice);
        cudaFuncSetAttribute(k_ldlt, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
        for (int rep = 0; rep < 3; ++rep) k_ldlt<<<1, 256, 80000>>>(G, R, c, o);
        long long cyc; cudaMemcpy(&cyc, c, 8, cudaMemcpyDeviceToHost);
        printf("R=%d ldlt_one_sync: %lld cycles (%.1f per step) err=%s\n", R, cyc, double(cyc) / R,
               cudaGetErrorString(cudaGetLastError()));
        double d1; cudaMemcpy(&d1, o, 8, cudaMemcpyDeviceToHost);
        if (R <= 32) {
            cudaFuncSetAttribute(k_ldlt_warp, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
            for (int rep = 0; rep < 3; ++rep) k_ldlt_warp<<<1, 256, 80000>>>(G, R, c, o);
            cudaMemcpy(&cyc, c, 8, cudaMemcpyDeviceToHost);
            double d2; cudaMemcpy(&d2, o, 8, cudaMemcpyDeviceToHost);
            printf("R=%d ldlt_warp: %lld cycles (%.1f per step) same_last_d=%d err=%s\n", R, cyc, double(cyc) / R,
                   int(d1 == d2), cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
