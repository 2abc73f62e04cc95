// Profiling aid: strided fibre-gather throughput on a FEW SMs (the overlapped
// window gather runs on SMs reserved beside the chain kernel).
// Workload = the C2 mode-2 stage: fibres X[i1, :, i3] of a 1000^3 fp64 tensor
// (stride 8 KB), sorted by base, 256 elements per warp unit.
// Variants: LSU loads (8 or 16 per lane) vs a TMA tile box {2, 256, 1} per
// unit (16-byte rows; the element is picked by i1 parity) into shared memory.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <vector>
#include <algorithm>
#include <random>

constexpr int I = 1000;
constexpr int kUnit = 256;

template <int U>
__global__ void __launch_bounds__(1024, 1) k_lsu(const double* t, const int64_t* base, int nfib, double* out) {
    const int lane = threadIdx.x & 31;
    const int W = gridDim.x * 32, w = blockIdx.x * 32 + (threadIdx.x >> 5);
    constexpr int span = 32 * U;
    const int nblk = (I + span - 1) / span;
    for (int u = w; u < nfib * nblk; u += W) {
        const int ib = u / nfib, q = u - ib * nfib;
        const double* a = t + base[q];
        double v[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
            const int i = ib * span + lane + 32 * k;
            if (i < I) asm volatile("ld.global.cs.L2::64B.f64 %0, [%1];" : "=d"(v[k]) : "l"(a + int64_t(i) * I));
        }
#pragma unroll
        for (int k = 0; k < U; ++k) {
            const int i = ib * span + lane + 32 * k;
            if (i < I) out[int64_t(q) * I + i] = v[k];
        }
    }
}

__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(unsigned(__cvta_generic_to_shared(b))), "r"(n));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(unsigned(__cvta_generic_to_shared(b))),
                 "r"(bytes));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned ph) {
    asm volatile(
        "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(
            unsigned(__cvta_generic_to_shared(b))),
        "r"(ph));
}

// TMA: each warp owns kStages smem slots of 256 x 2 doubles; lane 0 keeps
// kStages boxes in flight, the warp drains slot by slot.
template <int kStages, int kWarps>
__global__ void __launch_bounds__(kWarps * 32, 1) k_tma(const __grid_constant__ CUtensorMap tm, const int* i1s,
                                                        const int* i3s, int nfib, double* out) {
    extern __shared__ __align__(128) double sm[];
    __shared__ __align__(8) uint64_t bars[kWarps][kStages];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int W = gridDim.x * kWarps, w = blockIdx.x * kWarps + wid;
    const int nblk = (I + kUnit - 1) / kUnit;
    const int total = nfib * nblk;
    double* slot0 = sm + wid * kStages * kUnit * 2;
    if (lane == 0)
        for (int s = 0; s < kStages; ++s) mbar_init(&bars[wid][s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    auto issue = [&](int u, int s) {
        const int ib = u / nfib, q = u - ib * nfib;
        const int c0 = i1s[q] & ~1, c1 = ib * kUnit, c2 = i3s[q];
        uint64_t* b = &bars[wid][s];
        mbar_expect(b, kUnit * 16);
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
            "[%5];" ::"r"(unsigned(__cvta_generic_to_shared(slot0 + s * kUnit * 2))),
            "l"(&tm), "r"(c0), "r"(c1), "r"(c2), "r"(unsigned(__cvta_generic_to_shared(b)))
            : "memory");
    };
    unsigned phase = 0;
    int k = 0;
    if (lane == 0)
        for (int s = 0; s < kStages && w + s * W < total; ++s) issue(w + s * W, s);
    for (int u = w; u < total; u += W, ++k) {
        const int s = k % kStages;
        mbar_wait(&bars[wid][s], (phase >> s) & 1u);
        phase ^= 1u << s;
        const int ib = u / nfib, q = u - ib * nfib;
        const int par = i1s[q] & 1;
        const double* sl = slot0 + s * kUnit * 2;
        double v[kUnit / 32];
#pragma unroll
        for (int j = 0; j < kUnit / 32; ++j) v[j] = sl[(lane + 32 * j) * 2 + par];
        __syncwarp();
        const int un = u + kStages * W;
        if (lane == 0 && un < total) issue(un, s);
#pragma unroll
        for (int j = 0; j < kUnit / 32; ++j) {
            const int i = ib * kUnit + lane + 32 * j;
            if (i < I) out[int64_t(q) * I + i] = v[j];
        }
    }
}

__global__ void k_fill(double* t, int64_t n) {
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n; e += int64_t(gridDim.x) * blockDim.x)
        t[e] = double(e);
}

int main() {
    const int64_t I3 = 1000;
    const int64_t numel = int64_t(I) * I * I3;
    double* t;
    cudaMalloc(&t, numel * 8);
    k_fill<<<148 * 8, 256>>>(t, numel);
    const int nfib = 600 * 36;  // one C2 window of mode-2 stages
    std::mt19937_64 g(7);
    std::vector<int> i1(nfib), i3(nfib);
    std::vector<int64_t> base(nfib);
    for (int b = 0; b < 36; ++b) {
        std::vector<std::pair<int64_t, int>> v;
        for (int c = 0; c < 600; ++c) {
            const int a1 = int(g() % I), a3 = int(b * 25 + g() % 25);
            v.push_back({a1 + int64_t(a3) * I * I, a1});
        }
        std::sort(v.begin(), v.end());
        for (int c = 0; c < 600; ++c) {
            base[b * 600 + c] = v[c].first;
            i1[b * 600 + c] = v[c].second;
            i3[b * 600 + c] = int(v[c].first / (int64_t(I) * I));
        }
    }
    int64_t* dbase;
    int *di1, *di3;
    double* out;
    cudaMalloc(&dbase, nfib * 8);
    cudaMalloc(&di1, nfib * 4);
    cudaMalloc(&di3, nfib * 4);
    cudaMalloc(&out, int64_t(nfib) * I * 8);
    cudaMemcpy(dbase, base.data(), nfib * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(di1, i1.data(), nfib * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(di3, i3.data(), nfib * 4, cudaMemcpyHostToDevice);

    CUtensorMap tm;
    cuuint64_t dims[3] = {cuuint64_t(I), cuuint64_t(I), cuuint64_t(I3)};
    cuuint64_t strides[2] = {cuuint64_t(I) * 8, cuuint64_t(I) * I * 8};
    cuuint32_t box[3] = {2, kUnit, 1}, estr[3] = {1, 1, 1};
    CUresult r = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, t, dims, strides, box, estr,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                        CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) printf("tensor map encode failed %d\n", int(r));

    constexpr int kS = 4, kW = 12;
    const size_t tma_smem = size_t(kW) * kS * kUnit * 2 * 8;  // 192 KB
    cudaFuncSetAttribute(k_lsu<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024);
    cudaFuncSetAttribute(k_lsu<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024);
    {
        cudaFuncAttributes fa;
        cudaError_t e1 = cudaFuncGetAttributes(&fa, k_tma<kS, kW>);
        int optin = 0;
        cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0);
        printf("getattr %s maxthreads %d regs %d static %zu maxdyn %d optin %d\n", cudaGetErrorString(e1), fa.maxThreadsPerBlock,
               fa.numRegs, fa.sharedSizeBytes, fa.maxDynamicSharedSizeBytes, optin);
        cudaError_t e2 = cudaFuncSetAttribute(k_tma<kS, kW>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(tma_smem));
        printf("setattr(%zu) %s\n", tma_smem, cudaGetErrorString(e2));
        cudaGetLastError();
    }
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    std::vector<double> ref(size_t(nfib) * I), got(size_t(nfib) * I);
    const double elems = double(nfib) * I;
    for (int G : {8, 16, 24, 32, 64, 148}) {
        for (int v = 0; v < 3; ++v) {
            float best = 1e9f;
            for (int rep = 0; rep < 3; ++rep) {
                cudaEventRecord(a);
                if (v == 0) k_lsu<8><<<G, 1024, 120 * 1024>>>(t, dbase, nfib, out);
                if (v == 1) k_lsu<16><<<G, 1024, 120 * 1024>>>(t, dbase, nfib, out);
                if (v == 2) k_tma<kS, kW><<<G, kW * 32, tma_smem>>>(tm, di1, di3, nfib, out);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                best = std::min(best, ms);
            }
            cudaMemcpy(got.data(), out, size_t(nfib) * I * 8, cudaMemcpyDeviceToHost);
            long bad = 0;
            for (int q = 0; q < nfib; q += 7)
                for (int i = 0; i < I; ++i)
                    if (got[size_t(q) * I + i] != double(base[q] + int64_t(i) * I)) ++bad;
            if (bad) printf("  MISMATCH %ld\n", bad);
            cudaMemset(out, 0, size_t(nfib) * I * 8);
            const char* nm[] = {"lsu x8 ", "lsu x16", "tma box"};
            printf("G=%3d %s %8.3f ms  %7.2f G elem/s  %6.3f G/s/SM  (%s)\n", G, nm[v], best, elems / best / 1e6,
                   elems / best / 1e6 / G, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
