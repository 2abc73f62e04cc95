// Profiling aid: per-step cycle breakdown of the warp LDL^T variants.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int kLdStride = 65;
template <int MAXR, int VARIANT>
__global__ void k_exp(const double* G, int R, long long* cyc, double* out) {
    __shared__ double A[64 * kLdStride], D[64];
    __shared__ long long ts[65];
    const int lane = threadIdx.x & 31;
    double r[MAXR];
#pragma unroll
    for (int j = 0; j < MAXR; ++j) r[j] = (lane < R && j <= lane) ? G[lane + j * R] : 0.0;
    __syncwarp();
    long long t0 = clock64();
#pragma unroll
    for (int k = 0; k < MAXR; ++k) {
        if (k < R) {
            const double dk = __shfl_sync(0xffffffffu, r[k], k);
            double ajk[MAXR];
#pragma unroll
            for (int j = k + 1; j < MAXR; ++j) ajk[j] = __shfl_sync(0xffffffffu, r[k], j);
            double l;
            if (VARIANT == 0) {  // plain IEEE division on all lanes
                const double q = r[k] / dk;
                l = (lane > k && dk != 0.0) ? q : 0.0;
            } else if (VARIANT == 1) {  // division with a safe dividend on inactive lanes
                const double num = (lane > k) ? r[k] : 1.0;
                const double q = num / dk;
                l = (lane > k && dk != 0.0) ? q : 0.0;
            } else {  // reciprocal multiply (timing reference only)
                l = (lane > k && dk != 0.0) ? r[k] * (1.0 / dk) : 0.0;
            }
            if (lane == 0) D[k] = dk;
            if (lane > k && lane < R) A[k * kLdStride + lane] = l;
#pragma unroll
            for (int j = k + 1; j < MAXR; ++j) r[j] = __fma_rn(-l, ajk[j], r[j]);
            if (lane == 0) ts[k] = clock64();
        }
    }
    long long t1 = clock64();
    if (lane == 0) { cyc[0] = t1 - t0; for (int k = 0; k < R; ++k) cyc[1 + k] = ts[k] - (k ? ts[k - 1] : t0); out[0] = D[R - 1]; }
}
template <int MAXR, int V = 0>
__global__ void k_exp2(const double* G, int R, long long* cyc, double* out) {
    __shared__ double A[64 * kLdStride], D[64];
    __shared__ double col[2][64];
    __shared__ long long ts[65];
    const int lane = threadIdx.x & 31;
    double r[MAXR];
#pragma unroll
    for (int j = 0; j < MAXR; ++j) r[j] = (lane < R && j <= lane) ? G[lane + j * R] : 0.0;
    __syncwarp();
    long long t0 = clock64();
#pragma unroll
    for (int k = 0; k < MAXR; ++k) {
        if (k < R) {
            double* cb = col[k & 1];
            cb[lane] = r[k];
            __syncwarp();
            const double dk = cb[k];
            double ajk[MAXR];
#pragma unroll
            for (int j = k + 1; j < MAXR; ++j) ajk[j] = cb[j];
            const double num = (lane > k) ? r[k] : 1.0;
            const double q = (V & 1) ? num * dk : num / dk;
            const double l = (lane > k && dk != 0.0) ? q : 0.0;
            if (lane == 0) D[k] = dk;
            if (lane > k && lane < R) A[k * kLdStride + lane] = l;
            if (V & 2) {
                if (k + 1 < MAXR) r[k + 1] = __fma_rn(-l, ajk[k + 1], r[k + 1]);
            } else {
#pragma unroll
                for (int j = k + 1; j < MAXR; ++j) r[j] = __fma_rn(-l, ajk[j], r[j]);
            }
            if (lane == 0) ts[k] = clock64();
        }
    }
    long long t1 = clock64();
    if (lane == 0) { cyc[0] = t1 - t0; for (int k = 0; k < R; ++k) cyc[1 + k] = ts[k] - (k ? ts[k - 1] : t0); out[0] = D[R - 1]; }
}
int main() {
    const int R = 20;
    double h[64 * 64];
    for (int i = 0; i < R; ++i) for (int j = 0; j < R; ++j) h[i + j * R] = (i == j ? R + 1.0 : 0.5 / (1 + i + j));
    double* G; long long* c; double* o; cudaMalloc(&G, sizeof(h)); cudaMalloc(&c, 8 * 80); cudaMalloc(&o, 8);
    cudaMemcpy(G, h, sizeof(h), cudaMemcpyHostToDevice);
    long long hc[80];
    for (int v = 0; v < 7; ++v) {
        for (int rep = 0; rep < 3; ++rep) {
            if (v == 0) k_exp<32, 0><<<1, 32>>>(G, R, c, o);
            if (v == 1) k_exp<32, 1><<<1, 32>>>(G, R, c, o);
            if (v == 2) k_exp<32, 2><<<1, 32>>>(G, R, c, o);
            if (v == 3) k_exp2<32><<<1, 32>>>(G, R, c, o);
            if (v == 4) k_exp2<32, 1><<<1, 32>>>(G, R, c, o);
            if (v == 5) k_exp2<32, 2><<<1, 32>>>(G, R, c, o);
            if (v == 6) k_exp2<32, 3><<<1, 32>>>(G, R, c, o);
        }
        cudaMemcpy(hc, c, 8 * 80, cudaMemcpyDeviceToHost);
        printf("variant %d: total %lld cycles; per step:", v, hc[0]);
        for (int k = 0; k < R; ++k) printf(" %lld", hc[1 + k]);
        printf("\n");
    }
    return 0;
}
