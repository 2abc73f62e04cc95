// Profiling aid: the inner loop of chain_stream_items (one 32-sample chunk step of a 64-row pair,
// RP = 56) on shared-memory-resident data -- fp64 MMA rate against the loop shape.
//   variant 0: rolled k loop (loads, then MMAs, per 4 samples)
//   variant 1: every fragment of the chunk loaded first, then 8 x (2 x nloc) MMAs
//   variant 2: k loop with the next step's fragments loaded before this step's MMAs
#include <cstdio>
#include <cuda_runtime.h>

constexpr int NT = 7, RPZ = 8 * NT + 4, NH0 = 4, NH1 = 3;

#define DMMA(c0, c1, a, b) \
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};" : "+d"(c0), "+d"(c1) : "d"(a), "d"(b))

template <int V>
__global__ void __launch_bounds__(256, 1) k_step(const double* X, const double* Z, int steps, long long* cyc, double* out, const int* cnkp) {
    extern __shared__ __align__(1024) double sm[];
    double* ring = sm;            // 2 tiles x 64 rows x 16
    double* zs = sm + 2048;       // 32 x RPZ
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (V == 3) for (int t = tid; t < 6 * 2048 + 256 * RPZ; t += 256) sm[t] = X[t % 2048];
    __syncthreads();
    for (int t = tid; t < 2048; t += 256) ring[t] = X[t];
    for (int t = tid; t < 32 * RPZ; t += 256) zs[t] = Z[t];
    __syncthreads();
    const int q4 = lane & 3, rr = lane >> 2;
    const int rp = warp & 3, half = warp >> 2;
    const int n0 = half ? NH0 : 0, nloc = half ? NH1 : NH0;
    const int tsel = rp >> 1, hrow = rp & 1;
    const double* xb = ring + tsel * 1024;
    const double* zb = zs + n0 * 8;
    double acc[2][NH0][2], qv[2][NH0][2];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int n = 0; n < NH0; ++n) qv[a][n][0] = qv[a][n][1] = 0.0;
    const long long t0 = clock64();
    for (int s = 0; s < steps; ++s) {
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int n = 0; n < NH0; ++n) acc[a][n][0] = acc[a][n][1] = 0.0;
        if (V == 0) {
            for (int k0 = 0; k0 < 32; k0 += 4) {
                const int smp = k0 + q4;
                double fa[2], fb[NH0];
#pragma unroll
                for (int a = 0; a < 2; ++a) {
                    const int r = 2 * smp + hrow;
                    fa[a] = xb[r * 16 + (((a * 4 + (rr >> 1)) ^ (r & 7)) << 1) + (rr & 1)];
                }
#pragma unroll
                for (int n = 0; n < NH0; ++n) fb[n] = (n < nloc) ? zb[smp * RPZ + n * 8 + rr] : 0.0;
#pragma unroll
                for (int a = 0; a < 2; ++a)
#pragma unroll
                    for (int n = 0; n < NH0; ++n)
                        if (n < nloc) DMMA(acc[a][n][0], acc[a][n][1], fa[a], fb[n]);
            }
        } else if (V == 1) {
            double fa[8][2], fb[8][NH0];
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
                const int smp = 4 * ks + q4;
#pragma unroll
                for (int a = 0; a < 2; ++a) {
                    const int r = 2 * smp + hrow;
                    fa[ks][a] = xb[r * 16 + (((a * 4 + (rr >> 1)) ^ (r & 7)) << 1) + (rr & 1)];
                }
#pragma unroll
                for (int n = 0; n < NH0; ++n) fb[ks][n] = (n < nloc) ? zb[smp * RPZ + n * 8 + rr] : 0.0;
            }
#pragma unroll
            for (int ks = 0; ks < 8; ++ks)
#pragma unroll
                for (int a = 0; a < 2; ++a)
#pragma unroll
                    for (int n = 0; n < NH0; ++n)
                        if (n < nloc) DMMA(acc[a][n][0], acc[a][n][1], fa[ks][a], fb[ks][n]);
        } else if (V == 3) {
            const int cnk = cnkp[s & 7];
            const double* xb2 = sm + (s % 6) * 2048 + tsel * 1024;
            const double* zb2 = sm + 6 * 2048 + ((s & 7) * 32) * RPZ + n0 * 8 + q4 * RPZ + rr;
            int xo[2];
#pragma unroll
            for (int a = 0; a < 2; ++a) {
                const int r = 2 * q4 + hrow;
                xo[a] = r * 16 + (((a * 4 + (rr >> 1)) ^ (r & 7)) << 1) + (rr & 1);
            }
            double fa[2][2], fb[2][NH0];
            auto ld = [&](int ks, int buf) {
                const bool valid = 4 * ks + q4 < cnk;
#pragma unroll
                for (int a = 0; a < 2; ++a) fa[buf][a] = valid ? xb2[ks * 128 + xo[a]] : 0.0;
#pragma unroll
                for (int n = 0; n < NH0; ++n) fb[buf][n] = (valid && n < nloc) ? zb2[ks * 4 * RPZ + n * 8] : 0.0;
            };
            const int nks = (cnk + 3) >> 2;
            ld(0, 0);
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
                if (ks < nks) {
                    if (ks + 1 < 8) ld(ks + 1, (ks + 1) & 1);
#pragma unroll
                    for (int a = 0; a < 2; ++a)
#pragma unroll
                        for (int n = 0; n < NH0; ++n)
                            if (n < nloc) DMMA(acc[a][n][0], acc[a][n][1], fa[ks & 1][a], fb[ks & 1][n]);
                }
            }
            __syncthreads();
        } else {
            double fa[2][2], fb[2][NH0];
            auto ld = [&](int ks, int buf) {
                const int smp = 4 * ks + q4;
#pragma unroll
                for (int a = 0; a < 2; ++a) {
                    const int r = 2 * smp + hrow;
                    fa[buf][a] = xb[r * 16 + (((a * 4 + (rr >> 1)) ^ (r & 7)) << 1) + (rr & 1)];
                }
#pragma unroll
                for (int n = 0; n < NH0; ++n) fb[buf][n] = (n < nloc) ? zb[smp * RPZ + n * 8 + rr] : 0.0;
            };
            ld(0, 0);
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
                if (ks + 1 < 8) ld(ks + 1, (ks + 1) & 1);
#pragma unroll
                for (int a = 0; a < 2; ++a)
#pragma unroll
                    for (int n = 0; n < NH0; ++n)
                        if (n < nloc) DMMA(acc[a][n][0], acc[a][n][1], fa[ks & 1][a], fb[ks & 1][n]);
            }
        }
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int n = 0; n < NH0; ++n)
#pragma unroll
                for (int e = 0; e < 2; ++e) qv[a][n][e] = qv[a][n][e] + acc[a][n][e];
        if (V >= 10) __syncthreads();
    }
    __syncthreads();
    const long long t1 = clock64();
    if (blockIdx.x == 0 && tid == 0) cyc[0] = t1 - t0;
    double t = 0;
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int n = 0; n < NH0; ++n) t += qv[a][n][0] + qv[a][n][1];
    if (t == 1.2345) out[0] = t;
}

template <int V>
void run(const double* dx, const double* dz, long long* dc, double* dout, const int* dn) {
    const int smem = (V == 3 ? 6 * 2048 + 256 * RPZ : 2048 + 32 * RPZ) * 8, steps = 16384;
    cudaFuncSetAttribute(k_step<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_step<V><<<148, 256, smem>>>(dx, dz, steps, dc, dout, dn);
    cudaEventRecord(e0);
    k_step<V><<<148, 256, smem>>>(dx, dz, steps, dc, dout, dn);
    cudaEventRecord(e1);
    cudaError_t e = cudaDeviceSynchronize();
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    long long c;
    cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
    const double fl = 2.0 * 64 * 32 * 56 * steps;
    printf("variant %d: %.0f cycles per step, %.1f flop/clk/SM of 128, %.3f ms -> %.3f GHz effective, %.1f TFLOP/s (%s)\n", V,
           double(c) / steps, fl / c, ms, double(c) / (ms * 1e6), fl * 148 / ms / 1e9, cudaGetErrorString(e));
}

int main() {
    double *dx, *dz, *dout;
    long long* dc;
    cudaMalloc(&dx, 2048 * 8);
    cudaMalloc(&dz, 32 * RPZ * 8);
    cudaMalloc(&dout, 64);
    cudaMalloc(&dc, 64);
    {
        double hx[2048], hz[32 * RPZ];
        unsigned long long sd = 88172645463325252ull;
        auto rnd = [&]() { sd ^= sd << 13; sd ^= sd >> 7; sd ^= sd << 17; return double(sd % 20001) / 10000.0 - 1.0; };
        for (double& v : hx) v = rnd();
        for (double& v : hz) v = rnd();
        cudaMemcpy(dx, hx, sizeof(hx), cudaMemcpyHostToDevice);
        cudaMemcpy(dz, hz, sizeof(hz), cudaMemcpyHostToDevice);
    }
    int hn[8] = {32, 32, 32, 32, 32, 32, 32, 32};
    int* dn;
    cudaMalloc(&dn, sizeof(hn));
    cudaMemcpy(dn, hn, sizeof(hn), cudaMemcpyHostToDevice);
    run<0>(dx, dz, dc, dout, dn);
    run<1>(dx, dz, dc, dout, dn);
    run<2>(dx, dz, dc, dout, dn);
    run<3>(dx, dz, dc, dout, dn);
    return 0;
}
