// gather_kernel.cuh -- K2 overlapped with the persistent chain.
//
// The window gather (sample_unfolding, sampling.cpp:57-79, for every batch and
// stage of a stream window) runs as a persistent grid on a few SMs reserved
// beside k_chain, on its own stream.  Work is cut into warp units dealt round
// robin in (batch, stage) job order; a warp counts the units it finished per
// job and publishes the count (fence + atomicAdd) when it moves on, and the
// chain waits for done[job] == units(job) before its first bulk copy of that
// (batch, stage) (chain_kernel.cuh, wait_gathered).
//
// Two unit kinds:
//  * strided fibres (modes >= 2 and the temporal mode) with a tensor-map view:
//    ONE TMA tile copy per unit, box {2, 1, L, 1} of the 4-D view
//    (I1, Ma, In, Mb) -- 16-byte rows at the fibre's mode-1 position, L fibre
//    elements -- into the warp's shared-memory slot; the warp picks the
//    element of each row by i1 parity and writes the row-tiled X_s.  The TMA
//    unit issues a strided element about 1.7x faster per SM than LSU loads do
//    (tools/gather_sm_bench.cu: 1.5 vs 0.86 G elements/s/SM), so fewer SMs
//    keep pace with the chain.
//  * contiguous mode-1 fibres: one TMA box of L consecutive elements per unit
//    (view (I1, 1, 1, rest)); the LSU version of these units read only
//    ~10 GB/s per SM (kGatherUnroll loads of 8 B per lane, a division per
//    element).
//  * views TMA cannot express (odd I1, a misaligned range, ROCP_GATHER_TMA=0):
//    LSU loads, kGatherUnroll per lane, as in k_gather.
#pragma once

#include <cuda.h>  // CUtensorMap (type only)

namespace rocpk {

constexpr int kGWThreads = 768;  // 85 registers per thread: no spills
constexpr int kGWWarps = kGWThreads / 32;
constexpr int kGWUnit = 32 * kGatherUnroll;  // LSU unit: elements per warp (kGatherUnroll per lane)
constexpr int kGWBox = 256;                  // TMA unit: fibre elements per box (hardware box limit)
// one 4 KB slot per warp (96 KB), padded past half an SM's shared memory so a gather block never
// shares an SM with another gather block or a chain block
constexpr size_t kGWSmem = 120 * 1024;
static_assert(size_t(kGWWarps) * kGWBox * 2 * sizeof(double) <= kGWSmem, "gather slots");

// 4-D view of the window's tensor range for one strided mode n: (I1, Ma =
// I2..I_{n-1}, In, Mb = the rest, time included); the temporal mode uses In =
// the window's slice count and Mb = 1.
struct GatherView {
    int64_t I1, Ma, In;
    int contig;  // mode 1: view (I1, 1, 1, rest), box {L, 1, 1, 1} -- one contiguous fibre segment
};
struct GatherTmaParams {
    CUtensorMap map[kMaxOrder];  // by mode - 1
    GatherView view[kMaxOrder];
};

__host__ __device__ __forceinline__ uint32_t gather_units(const GatherJob& J) {
    if (J.tmap1) return uint32_t((J.I + J.tlen - 1) / J.tlen) * uint32_t(J.s);
    return J.perm ? uint32_t((J.I + kGWUnit - 1) / kGWUnit) * uint32_t(J.s)
                  : uint32_t((int64_t(J.I) * J.s + kGWUnit - 1) / kGWUnit);
}

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
        "%5}], [%6];" ::"r"(smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
        : "memory");
}

__global__ void __launch_bounds__(kGWThreads, 1) k_gather_warps(const __grid_constant__ GatherTmaParams tp,
                                                                 const GatherJob* __restrict__ jobs, int njobs,
                                                                 const uint32_t* __restrict__ ustart,
                                                                 unsigned* __restrict__ done) {
    extern __shared__ __align__(128) double gsm[];
    __shared__ __align__(8) uint64_t bars[kGWWarps];
    const int lane = int(threadIdx.x & 31), wid = int(threadIdx.x >> 5);
    double* slot = gsm + wid * kGWBox * 2;
    uint64_t* bar = &bars[wid];
    if (lane == 0) mbar_init(bar, 1);
    __syncwarp();
    unsigned phase = 0;
    const uint32_t W = gridDim.x * kGWWarps;
    const uint32_t total = __ldg(ustart + njobs);
    int j = 0;
    uint32_t j_end = __ldg(ustart + 1), cnt = 0;
    auto publish = [&]() {
        if (cnt == 0) return;
        __threadfence();  // every lane's stores, then one count
        __syncwarp();
        if (lane == 0) atomicAdd(done + j, cnt);
        cnt = 0;
    };
    for (uint32_t u = blockIdx.x * kGWWarps + uint32_t(wid); u < total; u += W) {
        if (u >= j_end) {
            publish();
            while (u >= j_end) {
                ++j;
                j_end = __ldg(ustart + j + 1);
            }
        }
        const GatherJob& J = jobs[j];
        const uint32_t ul = u - __ldg(ustart + j);
        if (J.tmap1) {  // strided fibre, one TMA box
            const int m = J.tmap1 - 1;
            const uint32_t ib = ul / uint32_t(J.s), q = ul - ib * uint32_t(J.s);
            const int c = J.perm ? __ldg(J.perm + q) : int(q);
            const int i0 = int(ib) * J.tlen, n = min(J.tlen, J.I - i0);
            const GatherView& v = tp.view[m];
            const int tw = v.contig ? 1 : 2;  // doubles per box row
            int par = 0;
            if (lane == 0) {
                const int64_t w = __ldg(J.base + c) + J.toff;
                const int64_t qq = w / v.I1, i1 = w - qq * v.I1;
                const int64_t q2 = qq / v.Ma, a = qq - q2 * v.Ma;
                const int64_t c3 = q2 / v.In, c2 = q2 - c3 * v.In;
                par = v.contig ? 0 : int(i1 & 1);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // slot reads of the last unit
                mbar_expect_tx(bar, unsigned(J.tlen) * 8u * unsigned(tw));
                if (v.contig) tma_load_4d(slot, &tp.map[m], i0, 0, 0, int(qq), bar);
                else tma_load_4d(slot, &tp.map[m], int(i1 & ~int64_t(1)), int(a), int(c2) + i0, int(c3), bar);
            }
            par = __shfl_sync(0xffffffffu, par, 0);
            mbar_wait(bar, phase);
            phase ^= 1u;
            for (int i = lane; i < n; i += 32) {
                const double x = slot[tw * i + par];
                if (J.tiled) J.out[xs_offset(i0 + i, c, J.s)] = x;
                else J.out[int64_t(c) * J.I + i0 + i] = x;
            }
            __syncwarp();
        } else if (J.perm) {  // strided fibre, LSU loads
            const uint32_t ib = ul / uint32_t(J.s), q = ul - ib * uint32_t(J.s);
            const int c = __ldg(J.perm + q);
            const double* a = J.t + __ldg(J.base + c);
            const int i0 = int(ib) * kGWUnit + lane;
            double v[kGatherUnroll];
#pragma unroll
            for (int k = 0; k < kGatherUnroll; ++k) {
                const int i = i0 + 32 * k;
                if (i < J.I) asm volatile("ld.global.cs.L2::64B.f64 %0, [%1];" : "=d"(v[k]) : "l"(a + int64_t(i) * J.ms));
            }
#pragma unroll
            for (int k = 0; k < kGatherUnroll; ++k) {
                const int i = i0 + 32 * k;
                if (i < J.I) J.out[xs_offset(i, c, J.s)] = v[k];
            }
        } else {  // flattened elements (contiguous mode-1 fibres: coalesced)
            const uint32_t I = uint32_t(J.I), tot = I * uint32_t(J.s);
            const uint32_t e0 = ul * kGWUnit + uint32_t(lane);
            double v[kGatherUnroll];
#pragma unroll
            for (int k = 0; k < kGatherUnroll; ++k) {
                const uint32_t e = e0 + 32u * k;
                if (e < tot) {
                    const uint32_t c = e / I, i = e - c * I;
                    const double* a = J.t + __ldg(J.base + c) + int64_t(i) * J.ms;
                    if (J.ms == 1) v[k] = __ldcs(a);
                    else asm volatile("ld.global.cs.L2::64B.f64 %0, [%1];" : "=d"(v[k]) : "l"(a));
                }
            }
#pragma unroll
            for (int k = 0; k < kGatherUnroll; ++k) {
                const uint32_t e = e0 + 32u * k;
                if (e < tot) {
                    const uint32_t c = e / I, i = e - c * I;
                    if (J.tiled) J.out[xs_offset(i, c, J.s)] = v[k];
                    else J.out[e] = v[k];
                }
            }
        }
        ++cnt;
    }
    publish();
}

}  // namespace rocpk
