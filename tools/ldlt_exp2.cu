// Profiling aid: where the cycles of one warp-LDL^T pivot step go.
// Variants of the ldlt_warp step (kernels.cuh): V=0 as shipped, V=1 divide
// replaced by a multiply, V=2 no shuffle (pivot from shared memory), V=3 no
// deferred updates, V=4 divide via reciprocal + one Newton step.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false tools/ldlt_exp2.cu -o tools/ldlt_exp2
#include <cstdio>

constexpr int kLd = 65;

template <int MAXR, int V>
__device__ __noinline__ void ldlt_v(const double* G, int R, double* A, double* D, double* col, long long* steps) {
    const int lane = threadIdx.x & 31;
    double r[MAXR];
#pragma unroll
    for (int j = 0; j < MAXR; ++j) r[j] = (lane < R && j <= lane) ? G[lane + j * R] : 0.0;
    col[lane] = r[0];
    __syncwarp();
    double dk = __shfl_sync(0xffffffffu, r[0], 0);
    double lp = 0.0;
    long long t = clock64();
#pragma unroll
    for (int k = 0; k < MAXR; ++k) {
        if (k < R) {
            const double* cb = col + (k % 3) * 32;
            if (V != 3 && k > 0) {
                const double* cp = col + ((k + 2) % 3) * 32;
#pragma unroll
                for (int j = k + 1; j < MAXR; ++j) r[j] = __fma_rn(-lp, cp[j], r[j]);
            }
            const bool act = lane > k && lane < R;
            const double num = act ? r[k] : 1.0;
            double q;
            if (V == 1) q = num * dk;
            else if (V == 4) {
                double y = __drcp_rn(dk);
                q = num * y;
                q = __fma_rn(__fma_rn(-dk, q, num), y, q);
            } else q = num / dk;
            const double l = (act && dk != 0.0) ? q : 0.0;
            double dn = 0.0;
            if (k + 1 < MAXR) {
                r[k + 1] = __fma_rn(-l, cb[k + 1], r[k + 1]);
                col[((k + 1) % 3) * 32 + lane] = r[k + 1];
                if (V == 2) {
                    __syncwarp();
                    dn = col[((k + 1) % 3) * 32 + ((k + 1) & 31)];
                } else {
                    dn = __shfl_sync(0xffffffffu, r[k + 1], (k + 1) & 31);
                }
            }
            if (lane == 0) D[k] = dk;
            if (act) A[k * kLd + lane] = l;
            __syncwarp();
            lp = l;
            dk = dn;
            if (lane == 0) {
                long long t2 = clock64();
                steps[k] = t2 - t;
                t = t2;
            }
        }
    }
}

template <int MAXR, int V>
__global__ void k_run(const double* G, int R, long long* steps, double* out) {
    __shared__ double A[64 * kLd], D[64], col[96];
    if (threadIdx.x < 32) ldlt_v<MAXR, V>(G, R, A, D, col, steps);
    __syncthreads();
    if (threadIdx.x == 0) out[0] = D[R - 1];
}

template <int MAXR, int V>
void run(const char* name, const double* G, int R, long long* steps, double* out) {
    for (int rep = 0; rep < 3; ++rep) k_run<MAXR, V><<<1, 32>>>(G, R, steps, out);
    long long h[64];
    cudaMemcpy(h, steps, sizeof(long long) * R, cudaMemcpyDeviceToHost);
    long long tot = 0;
    for (int k = 1; k < R; ++k) tot += h[k];
    printf("R=%d %-28s mean %.0f cycles/step (k=1..R-1), k=1: %lld, k=R/2: %lld  err=%s\n", R, name,
           double(tot) / (R - 1), h[1], h[R / 2], cudaGetErrorString(cudaGetLastError()));
}

int main() {
    const int R = 20;
    double h[64 * 64];
    for (int i = 0; i < R; ++i)
        for (int j = 0; j < R; ++j) h[i + j * R] = (i == j ? 600.0 + i : 3.0 / (1 + i + j));
    double *G, *o;
    long long* s;
    cudaMalloc(&G, sizeof(h));
    cudaMalloc(&s, 64 * 8);
    cudaMalloc(&o, 8);
    cudaMemcpy(G, h, sizeof(h), cudaMemcpyHostToDevice);
    run<24, 0>("as shipped", G, R, s, o);
    run<24, 1>("divide -> multiply", G, R, s, o);
    run<24, 2>("pivot via smem, no shfl", G, R, s, o);
    run<24, 3>("no deferred updates", G, R, s, o);
    run<24, 4>("rcp + newton", G, R, s, o);
    run<32, 0>("as shipped, MAXR 32", G, R, s, o);
    return 0;
}
