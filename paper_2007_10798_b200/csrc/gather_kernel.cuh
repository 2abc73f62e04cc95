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

constexpr int kGWThreads = 640;  // 96 registers per thread: no spills
constexpr int kGWWarps = kGWThreads / 32;
constexpr int kGWUnit = 32 * kGatherUnroll;  // LSU unit: elements per warp (kGatherUnroll per lane)
constexpr int kGWBox = 256;                  // TMA unit: fibre elements per box (hardware box limit)
constexpr int kGWDepth = 2;                  // boxes in flight per warp (the next units' coordinates and
                                             // copies overlap the current unit's consumption)
// kGWDepth 4 KB slots per warp (192 KB): more than half an SM's shared memory, so a gather block
// never shares an SM with another gather block or a chain block
constexpr size_t kGWSmem = size_t(kGWWarps) * kGWDepth * kGWBox * 2 * sizeof(double);
static_assert(kGWSmem > 114 * 1024 && kGWSmem <= 200 * 1024, "gather slots");

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

// tensor elements are read once: evict-first, so the random fibre reads do not push the chain's
// working set out of L2 (configs[1]: chain 1.64 -> 1.61 ms beside the gather).  An evict-last hint
// on the X_s stores, for the chain to read them from L2, measured no different (dropped).
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                            uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, "
        "{%2, %3, %4, %5}], [%6], %7;" ::"r"(smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}


// One warp unit, decoded at issue time (lane 0 computes the TMA coordinates).
struct GWUnit {
    int j;       // job (-1: none)
    uint32_t ul; // unit index within the job
    int c, i0, n, par, tw;
};

__global__ void __launch_bounds__(kGWThreads, 1) k_gather_warps(const __grid_constant__ GatherTmaParams tp,
                                                                 const GatherJob* __restrict__ jobs, int njobs,
                                                                 const uint32_t* __restrict__ ustart,
                                                                 unsigned* __restrict__ done) {
    extern __shared__ __align__(128) double gsm[];
    __shared__ __align__(8) uint64_t bars[kGWWarps][kGWDepth];
    const int lane = int(threadIdx.x & 31), wid = int(threadIdx.x >> 5);
    double* slots = gsm + wid * kGWDepth * kGWBox * 2;
    if (lane == 0)
        for (int d = 0; d < kGWDepth; ++d) mbar_init(&bars[wid][d], 1);
    __syncwarp();
    unsigned phase = 0;  // bit d: parity of slot d
    uint64_t pol_first;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_first));
    const uint32_t W = gridDim.x * kGWWarps;
    const uint32_t total = __ldg(ustart + njobs);
    // issue side: decode unit u (job cursor ji only moves forward) and start its box
    int ji = 0;
    uint32_t ji_end = __ldg(ustart + 1);
    auto issue = [&](uint32_t u, int d) -> GWUnit {
        GWUnit x{-1, 0, 0, 0, 0, 0, 1};
        if (u >= total) return x;
        while (u >= ji_end) {
            ++ji;
            ji_end = __ldg(ustart + ji + 1);
        }
        const GatherJob& J = jobs[ji];
        x.j = ji;
        x.ul = u - __ldg(ustart + ji);
        if (!J.tmap1) return x;  // LSU unit: loads at consume time
        const int m = J.tmap1 - 1;
        const uint32_t ib = x.ul / uint32_t(J.s), q = x.ul - ib * uint32_t(J.s);
        x.c = J.perm ? __ldg(J.perm + q) : int(q);
        x.i0 = int(ib) * J.tlen;
        x.n = min(J.tlen, J.I - x.i0);
        const GatherView& v = tp.view[m];
        x.tw = v.contig ? 1 : 2;  // doubles per box row
        if (lane == 0) {
            const int64_t w = __ldg(J.base + x.c) + J.toff;
            const int64_t qq = w / v.I1, i1 = w - qq * v.I1;
            const int64_t q2 = qq / v.Ma, a = qq - q2 * v.Ma;
            const int64_t c3 = q2 / v.In, c2 = q2 - c3 * v.In;
            x.par = v.contig ? 0 : int(i1 & 1);
            uint64_t* bar = &bars[wid][d];
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // earlier generic reads of the slot
            mbar_expect_tx(bar, unsigned(J.tlen) * 8u * unsigned(x.tw));
            double* slot = slots + d * kGWBox * 2;
            if (v.contig) tma_load_4d(slot, &tp.map[m], x.i0, 0, 0, int(qq), bar, pol_first);
            else tma_load_4d(slot, &tp.map[m], int(i1 & ~int64_t(1)), int(a), int(c2) + x.i0, int(c3), bar, pol_first);
        }
        x.par = __shfl_sync(0xffffffffu, x.par, 0);
        return x;
    };
    // consume side: per-job unit counts, published (fence + atomicAdd) on job change
    int jc = -1;
    uint32_t cnt = 0;
    auto publish = [&]() {
        if (cnt == 0) return;
        __threadfence();  // every lane's stores, then one count
        __syncwarp();
        if (lane == 0) atomicAdd(done + jc, cnt);
        cnt = 0;
    };
    const uint32_t u0 = blockIdx.x * kGWWarps + uint32_t(wid);
    GWUnit pend[kGWDepth];
#pragma unroll
    for (int d = 0; d < kGWDepth; ++d) pend[d] = issue(u0 + uint32_t(d) * W, d);
    for (uint32_t u = u0, k = 0; u < total; u += W, ++k) {
        const int d = int(k % kGWDepth);
        GWUnit x = pend[0];
#pragma unroll
        for (int e = 1; e < kGWDepth; ++e)
            if (e == d) x = pend[e];
        if (x.j != jc) {
            publish();
            jc = x.j;
        }
        const GatherJob& J = jobs[x.j];
        if (J.tmap1) {  // strided or mode-1 fibre segment, landed in slot d
            mbar_wait(&bars[wid][d], (phase >> d) & 1u);
            phase ^= 1u << d;
            const double* slot = slots + d * kGWBox * 2;
            for (int i = lane; i < x.n; i += 32) {
                const double v = slot[x.tw * i + x.par];
                if (J.tiled) J.out[xs_offset(x.i0 + i, x.c, J.s)] = v;
                else J.out[int64_t(x.c) * J.I + x.i0 + i] = v;
            }
            __syncwarp();
        } else if (J.perm) {  // strided fibre, LSU loads
            const uint32_t ib = x.ul / uint32_t(J.s), q = x.ul - ib * uint32_t(J.s);
            const int c = __ldg(J.perm + q);
            const double* a = J.t + __ldg(J.base + c);
            const int i0 = int(ib) * kGWUnit + lane;
            double v[kGatherUnroll];
#pragma unroll
            for (int t = 0; t < kGatherUnroll; ++t) {
                const int i = i0 + 32 * t;
                if (i < J.I) asm volatile("ld.global.cs.L2::64B.f64 %0, [%1];" : "=d"(v[t]) : "l"(a + int64_t(i) * J.ms));
            }
#pragma unroll
            for (int t = 0; t < kGatherUnroll; ++t) {
                const int i = i0 + 32 * t;
                if (i < J.I) J.out[xs_offset(i, c, J.s)] = v[t];
            }
        } else {  // flattened elements (contiguous mode-1 fibres: coalesced)
            const uint32_t I = uint32_t(J.I), tot = I * uint32_t(J.s);
            const uint32_t e0 = x.ul * kGWUnit + uint32_t(lane);
            double v[kGatherUnroll];
#pragma unroll
            for (int t = 0; t < kGatherUnroll; ++t) {
                const uint32_t e = e0 + 32u * t;
                if (e < tot) {
                    const uint32_t c = e / I, i = e - c * I;
                    const double* a = J.t + __ldg(J.base + c) + int64_t(i) * J.ms;
                    if (J.ms == 1) v[t] = __ldcs(a);
                    else asm volatile("ld.global.cs.L2::64B.f64 %0, [%1];" : "=d"(v[t]) : "l"(a));
                }
            }
#pragma unroll
            for (int t = 0; t < kGatherUnroll; ++t) {
                const uint32_t e = e0 + 32u * t;
                if (e < tot) {
                    const uint32_t c = e / I, i = e - c * I;
                    if (J.tiled) J.out[xs_offset(i, c, J.s)] = v[t];
                    else J.out[e] = v[t];
                }
            }
        }
        ++cnt;
        // slot d is free again: start the unit kGWDepth rounds ahead in it
        const GWUnit nx = issue(u + uint32_t(kGWDepth) * W, d);
#pragma unroll
        for (int e = 0; e < kGWDepth; ++e)
            if (e == d) pend[e] = nx;
    }
    publish();
}

}  // namespace rocpk
