// Profiling aid: cycles of the on-demand row formation of a k_flow chunk block (per warp: one
// G^-1 column per lane from L2, four right-hand-side rows, four length-R dot products).
#include <cstdio>
#include <vector>
#include "../paper_2007_10798_b200/csrc/kernels.cuh"

template <int MAXR, int VAR>
__global__ void __launch_bounds__(256, 1) k_od(const double* ginv, const double* W, const int* idx, int R, long long* cyc,
                                               double* out) {
    __shared__ double wsm[8 * 4 * 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const bool lr = lane < R;
    __syncthreads();
    const long long t0 = clock64();
    double g[MAXR];
#pragma unroll
    for (int k = 0; k < MAXR; ++k) g[k] = (lr && k < R) ? __ldcg(ginv + k * R + lane) : 0.0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int iw = idx[warp * 4 + q];
        wsm[(warp * 4 + q) * 32 + lane] = lr ? __ldcg(W + int64_t(iw) * R + lane) : 0.0;
    }
    __syncwarp();
    double res[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const double* w = wsm + (warp * 4 + q) * 32;
        double acc = 0.0;
        if (VAR == 0) {
#pragma unroll
            for (int k = 0; k < MAXR; ++k) {
                const double v = __fma_rn(w[k], g[k], acc);
                acc = (k < R) ? v : acc;
            }
        } else {  // padded: g[k] = 0 and w[k] finite past R, no select
#pragma unroll
            for (int k = 0; k < MAXR; ++k) acc = __fma_rn(w[k], g[k], acc);
        }
        res[q] = acc;
    }
    const long long t1 = clock64();
    __syncthreads();
    const long long t2 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        cyc[0] = t1 - t0;
        cyc[1] = t2 - t0;
    }
    out[blockIdx.x * 256 + threadIdx.x] = res[0] + res[1] + res[2] + res[3];
}

int main() {
    const int R = 20;
    std::vector<double> gi(R * R, 0.5), w(1000 * R, 1.0);
    std::vector<int> idx(32);
    for (int i = 0; i < 32; ++i) idx[i] = (i * 37) % 1000;
    double *dg, *dw, *dout;
    int* di;
    long long* dc;
    cudaMalloc(&dg, gi.size() * 8);
    cudaMalloc(&dw, w.size() * 8);
    cudaMalloc(&dout, 148 * 256 * 8);
    cudaMalloc(&di, 32 * 4);
    cudaMalloc(&dc, 16);
    cudaMemcpy(dg, gi.data(), gi.size() * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dw, w.data(), w.size() * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(di, idx.data(), 32 * 4, cudaMemcpyHostToDevice);
    for (int var = 0; var < 2; ++var)
        for (int rep = 0; rep < 3; ++rep) {
            if (var == 0) k_od<24, 0><<<148, 256>>>(dg, dw, di, R, dc, dout);
            else k_od<24, 1><<<148, 256>>>(dg, dw, di, R, dc, dout);
            cudaDeviceSynchronize();
            long long c[2];
            cudaMemcpy(c, dc, 16, cudaMemcpyDeviceToHost);
            printf("var %d rep %d: warp0 %lld cycles, block %lld cycles (%s)\n", var, rep, c[0], c[1],
                   cudaGetErrorString(cudaGetLastError()));
        }
    return 0;
}
