// rocp_capi.cu -- host orchestration of the B200 ROCP hot path behind the
// C ABI declared in include/rocp_b200.h.
//
// One rocp_dev per GPU owns a CUDA stream, pooled counters/flags and the
// device-resident result of the last cprand.  rocp_stream owns every device
// buffer the online update needs (factors, P/Q, temporal factor, per-stage
// index/gather/KR scratch), allocated once at creation: consume never
// allocates (reference contract: constant state footprint, test_rocp.cpp:258-267).
//
// Control flow mirrors the reference line by line (citations inline); the
// arithmetic lives in kernels.cuh.

#include "../../include/rocp_b200.h"
#include "kernels.cuh"
#include "chain_kernel.cuh"
#include "flow_kernel.cuh"
#include "shard_kernels.cuh"
#include "gather_kernel.cuh"

#include <cuda_runtime.h>
#include <cudaTypedefs.h>  // PFN_cuTensorMapEncodeTiled (the driver entry point is fetched at run time)
#include <dlfcn.h>
#include <immintrin.h>
#include <nccl.h>  // types only: the library is bound at run time (NcclApi)
#include <sys/mman.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <limits>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

using namespace rocpk;

namespace {

struct RocpError {
    rocp_status code;
    std::string msg;
    int sweep = 0;
};

[[noreturn]] void throw_domain(const std::string& m) { throw RocpError{ROCP_E_DOMAIN, m}; }

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        if (e == cudaErrorMemoryAllocation)
            throw RocpError{ROCP_E_OOM, std::string(what) + ": " + cudaGetErrorString(e)};
        throw RocpError{ROCP_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e)};
    }
}
#define CK(x) cuda_check((x), #x)

// Owning device buffer.
template <class T>
struct DBuf {
    T* p = nullptr;
    size_t n = 0;
    DBuf() = default;
    explicit DBuf(size_t count) { alloc(count); }
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    DBuf(DBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
    DBuf& operator=(DBuf&& o) noexcept {
        if (this != &o) { release(); p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
        return *this;
    }
    ~DBuf() { release(); }
    void alloc(size_t count) {
        release();
        n = count;
        if (count) CK(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)));
    }
    void ensure(size_t count) {
        if (count > n) alloc(count);
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
};

int64_t prod(const std::vector<int64_t>& d) {
    int64_t n = 1;
    for (int64_t x : d) n *= x;
    return n;
}

int64_t auto_sample_count(int rank) {  // sampling.cpp:40-45
    if (rank < 1) throw_domain("rank must be positive");
    const double s = 10.0 * rank * std::log(double(rank));
    return std::max<int64_t>(rank, int64_t(std::ceil(s)));
}

std::vector<int64_t> strides_of(const std::vector<int64_t>& d) {  // tensor.cpp:68-76
    std::vector<int64_t> s(d.size());
    int64_t acc = 1;
    for (size_t k = 0; k < d.size(); ++k) { s[k] = acc; acc *= d[k]; }
    return s;
}

// Host column-major <-> device row-major conversions.
std::vector<double> colmajor_to_rowmajor(const double* a, int64_t rows, int64_t cols) {
    std::vector<double> out(size_t(rows * cols));
    for (int64_t j = 0; j < cols; ++j)
        for (int64_t i = 0; i < rows; ++i) out[size_t(i * cols + j)] = a[i + j * rows];
    return out;
}
void rowmajor_to_colmajor(const double* a, int64_t rows, int64_t cols, double* out) {
    for (int64_t i = 0; i < rows; ++i)
        for (int64_t j = 0; j < cols; ++j) out[i + j * rows] = a[size_t(i * cols + j)];
}

// Device copies of a list of draw jobs and gather jobs (+ the flat tile list
// of the gather).  Built on the host, uploaded once, then launched any number
// of times (also from inside CUDA graphs).
// NCCL, bound at run time: the copy already in the process (torch's) when
// there is one, else the system libnccl.so.2.  Only multi-GPU handles
// (world > 1) need it.
struct NcclApi {
    bool ok = false;
    std::string why;
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
};

const NcclApi& nccl_api() {
    static const NcclApi api = [] {
        NcclApi a;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            const char* e = dlerror();
            a.why = e ? e : "libnccl.so.2 not found";
            return a;
        }
        a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
        a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
        a.all_gather = reinterpret_cast<decltype(a.all_gather)>(dlsym(h, "ncclAllGather"));
        a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
        a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(h, "ncclGetErrorString"));
        a.ok = a.get_unique_id && a.comm_init_rank && a.all_gather && a.comm_destroy && a.error_string;
        if (!a.ok) a.why = "libnccl.so.2 lacks a required symbol";
        return a;
    }();
    return api;
}

void NK(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) throw RocpError{ROCP_E_NCCL, std::string(what) + ": " + nccl_api().error_string(r)};
}

const NcclApi& require_nccl() {
    const NcclApi& a = nccl_api();
    if (!a.ok) throw RocpError{ROCP_E_NCCL, "NCCL unavailable: " + a.why};
    return a;
}

struct JobList {
    DBuf<DrawJob> draw;
    DBuf<GatherJob> gather;
    DBuf<GatherTile> tiles;
    DBuf<SortJob> sort;
    int ndraw = 0, ngather = 0, ntiles = 0, nsort = 0;
    // overlapped gather (k_gather_warps): unit prefix per job, units published / needed
    DBuf<uint32_t> ustart;
    DBuf<unsigned> done, need;
    int64_t max_s = 0;
    int64_t gather_elems = 0;
};

}  // namespace

// ===========================================================================
struct rocp_dev {
    int device = 0;
    int world = 1, rank = 0;
    bool emulated = false;      // one of several ranks emulated on one device (no NCCL, no IPC)
    ncclComm_t comm = nullptr;  // world > 1: the mode-1 sharding communicator
    cudaStream_t stream = nullptr;
    std::string err;
    uint64_t launches = 0;
    DBuf<unsigned int> counters;  // zeroed; one per last-block kernel in flight
    DBuf<int> flags;              // [0] regularized, [1] non-finite code
    DBuf<double> scalars;         // small results
    DBuf<double> scratch_a, scratch_b;  // reduction partials
    JobList jobs;                       // draw/gather job scratch of the primitives and cprand
    DBuf<double> contract_partial;      // split-superchunk contraction partials
    DBuf<unsigned int> tile_counters;   // per-row-tile arrival counters (self-resetting)
    DBuf<unsigned int> gram_counters;   // k_gram: per-superchunk arrival counters (self-resetting)
    DBuf<int64_t> rows_in;              // explicit index scratch of the primitives
    cudaEvent_t timer[8] = {};          // rocp_timer_* slots
    // overlapped window gather: its own stream on SMs reserved beside the chain kernel
    cudaStream_t gstream = nullptr;
    cudaEvent_t ev_gready = nullptr, ev_gdone = nullptr;
    int gather_sms = -1;                // -1: not set (env decides); -2: per-stream model; >= 0: fixed
    int chain_sms = 0;                  // blocks of the persistent chain (0: every SM); rocp_set_chain_sms
    bool counted = false;               // registered in g_handles (live handles per GPU)
    int num_sms = 148;
    // device-resident result of the last rocp_cprand (for stream_create_from_init)
    struct Init {
        bool valid = false;
        std::vector<int64_t> dims;
        int rank = 0;
        int64_t s = 0;
        bool regularized = false;
        std::vector<DBuf<double>> factors;  // row-major I_n x R, best iterate
        std::vector<DBuf<double>> best_kr;  // N-1, s x R row-major
    } init;
};

struct rocp_tensor {
    std::vector<int64_t> dims;
    double* d = nullptr;
    bool owned = false;
    int64_t numel = 0;
    ~rocp_tensor() {
        if (owned && d) cudaFree(d);
    }
};

namespace {

void set_err(rocp_dev* dev, const RocpError& e) {
    if (dev) dev->err = e.msg;
}

// ---- launch helpers ---------------------------------------------------------
void after_launch(rocp_dev* dev, const char* name) {
    dev->launches++;
    cuda_check(cudaGetLastError(), name);
}

int grid_for(int64_t work, int block, int cap) {
    int64_t g = (work + block - 1) / block;
    return int(std::max<int64_t>(1, std::min<int64_t>(g, cap)));
}

// Fills a DrawJob for `mode` over tensor dims `d` (sampling.cpp:47-55 +
// decode_all sampling.cpp:11-20 + the base offset of sample_unfolding
// sampling.cpp:68-74).
DrawJob make_draw(const std::vector<int64_t>& d, int mode, int64_t s, uint64_t seed, uint32_t batch,
                  uint32_t iteration, const int64_t* in_rows, int64_t* rows, int32_t* idx,
                  int64_t* base) {
    DrawJob j{};
    j.seed = seed;
    j.seed_ptr = nullptr;
    j.batch_ptr = nullptr;
    j.batch = batch;
    j.iteration = iteration;
    j.mode = uint32_t(mode);
    j.n_other = int(d.size()) - 1;
    j.s = int32_t(s);
    const std::vector<int64_t> st = strides_of(d);
    int64_t co = 1;
    int pos = 0;
    for (size_t k = 0; k < d.size(); ++k) {
        if (int(k) + 1 == mode) continue;
        j.ext[pos] = d[k];
        j.tstride[pos] = st[k];
        co *= d[k];
        ++pos;
    }
    j.co = co;
    j.in_rows = in_rows;
    j.rows = rows;
    j.idx = idx;
    j.base = base;
    return j;
}

GatherJob make_gather(const double* t, const std::vector<int64_t>& d, int mode, int64_t s,
                      const int64_t* base, double* out, int tiled = 0) {
    GatherJob g{};
    g.tiled = tiled;
    g.t = t;
    g.base = base;
    g.ms = strides_of(d)[size_t(mode - 1)];
    g.I = int32_t(d[size_t(mode - 1)]);
    g.s = int32_t(s);
    g.out = out;
    return g;
}

void upload_jobs(rocp_dev* dev, JobList& L, const std::vector<DrawJob>& dj,
                 const std::vector<GatherJob>& gj, const std::vector<SortJob>& sj = {}) {
    std::vector<GatherTile> tiles;
    L.gather_elems = 0;
    for (size_t k = 0; k < gj.size(); ++k) {
        const uint32_t total = uint32_t(gj[k].I) * uint32_t(gj[k].s);
        L.gather_elems += total;
        if (gj[k].perm) {  // sorted tiles: element block outer, so co-scheduled blocks read adjacent samples
            for (uint32_t ib = 0; ib < uint32_t((gj[k].I + kSortedSpan - 1) / kSortedSpan); ++ib)
                for (uint32_t g = 0; g < uint32_t((gj[k].s + kSortedGroup - 1) / kSortedGroup); ++g)
                    tiles.push_back(GatherTile{int32_t(k), (g << 16) | ib});
        } else {
            for (uint32_t e0 = 0; e0 < total; e0 += kGatherTile) tiles.push_back(GatherTile{int32_t(k), e0});
        }
    }
    {  // warp units of the overlapped gather (k_gather_warps)
        std::vector<uint32_t> us(gj.size() + 1, 0), nd(std::max<size_t>(gj.size(), 1), 0);
        for (size_t k = 0; k < gj.size(); ++k) {
            nd[k] = gather_units(gj[k]);
            us[k + 1] = us[k] + nd[k];
        }
        L.ustart.ensure(us.size());
        L.need.ensure(nd.size());
        L.done.ensure(nd.size());
        CK(cudaMemcpyAsync(L.ustart.p, us.data(), us.size() * sizeof(uint32_t), cudaMemcpyHostToDevice, dev->stream));
        CK(cudaMemcpyAsync(L.need.p, nd.data(), nd.size() * sizeof(unsigned), cudaMemcpyHostToDevice, dev->stream));
    }
    L.sort.ensure(std::max<size_t>(sj.size(), 1));
    if (!sj.empty())
        CK(cudaMemcpyAsync(L.sort.p, sj.data(), sj.size() * sizeof(SortJob), cudaMemcpyHostToDevice, dev->stream));
    L.nsort = int(sj.size());
    L.max_s = 0;
    for (const DrawJob& j : dj) L.max_s = std::max<int64_t>(L.max_s, j.s);
    L.draw.ensure(std::max<size_t>(dj.size(), 1));
    L.gather.ensure(std::max<size_t>(gj.size(), 1));
    L.tiles.ensure(std::max<size_t>(tiles.size(), 1));
    if (!dj.empty())
        CK(cudaMemcpyAsync(L.draw.p, dj.data(), dj.size() * sizeof(DrawJob), cudaMemcpyHostToDevice, dev->stream));
    if (!gj.empty())
        CK(cudaMemcpyAsync(L.gather.p, gj.data(), gj.size() * sizeof(GatherJob), cudaMemcpyHostToDevice, dev->stream));
    if (!tiles.empty())
        CK(cudaMemcpyAsync(L.tiles.p, tiles.data(), tiles.size() * sizeof(GatherTile), cudaMemcpyHostToDevice,
                           dev->stream));
    CK(cudaStreamSynchronize(dev->stream));
    L.ndraw = int(dj.size());
    L.ngather = int(gj.size());
    L.ntiles = int(tiles.size());
}

void launch_draw(rocp_dev* dev, const JobList& L) {
    if (L.ndraw == 0) return;
    dim3 grid(grid_for(L.max_s, 128, 64), unsigned(L.ndraw));
    k_draw<<<grid, 128, 0, dev->stream>>>(L.draw.p);
    after_launch(dev, "k_draw");
}

void launch_gather(rocp_dev* dev, const JobList& L) {
    if (L.nsort > 0) {
        k_sort_by_base<<<L.nsort, 1024, 0, dev->stream>>>(L.sort.p);
        after_launch(dev, "k_sort_by_base");
    }
    if (L.ntiles == 0) return;
    k_gather<<<L.ntiles, kGatherThreads, 0, dev->stream>>>(L.gather.p, L.tiles.p);
    after_launch(dev, "k_gather");
}

void launch_skr(rocp_dev* dev, const SkrJob& j) {
    k_skr<<<grid_for(int64_t(j.s) * j.R, 256, dev->num_sms * 4), 256, 0, dev->stream>>>(j);
    after_launch(dev, "k_skr");
}

void launch_gram(rocp_dev* dev, const double* Z, int64_t s, int R, const double* acc_base,
                 double* out) {
    const int nk = int((s + kChunk - 1) / kChunk);
    const int nsup = (nk + kSuper - 1) / kSuper;
    dev->scratch_a.ensure(size_t(nk + nsup) * R * R);
    if (dev->gram_counters.n < size_t(nsup)) {  // self-resetting arrival counters, one per superchunk
        CK(cudaStreamSynchronize(dev->stream));
        dev->gram_counters.alloc(size_t(std::max(nsup, 64)));
        CK(cudaMemset(dev->gram_counters.p, 0, dev->gram_counters.n * sizeof(unsigned int)));
    }
    k_gram<<<nk, 256, size_t(kChunk) * R * sizeof(double), dev->stream>>>(
        Z, int32_t(s), R, dev->scratch_a.p, dev->scratch_a.p + size_t(nk) * R * R, dev->counters.p + 0,
        dev->gram_counters.p, acc_base, out);
    after_launch(dev, "k_gram");
}

// Contraction launch: r-groups of RB <= 10 outputs per thread (32 rows per
// warp), 256-sample superchunks split across blocks.
constexpr int kMaxContractGroups = 8;

int contract_groups(int R, int* rb) {
    const int ng = (R + 9) / 10;
    *rb = (R + ng - 1) / ng;
    return ng;
}

size_t contract_smem(int R) {
    int rb;
    const int ng = contract_groups(R, &rb);
    return (size_t(kSuperSamples) * kRowTile + size_t(kSuperSamples) * ng * rb) * sizeof(double);
}

template <int RB>
void launch_contract_rb(rocp_dev* dev, int ng, const double* X, int64_t I, int64_t s, const double* Z, int R,
                        const double* base, double* out, int tiled) {
    const int tiles = int((I + kRowTile - 1) / kRowTile);
    const int nsuper = int((s + kSuperSamples - 1) / kSuperSamples);
    if (nsuper > 1) {
        if (dev->contract_partial.n < size_t(nsuper) * I * R || dev->tile_counters.n < size_t(tiles))
            throw RocpError{ROCP_E_STATE, "contraction scratch not reserved (internal)"};
    }
    const dim3 grid{unsigned(tiles), unsigned(nsuper), 1u};
    k_contract<RB><<<grid, 32 * ng, contract_smem(R), dev->stream>>>(
        X, int32_t(I), int32_t(s), Z, R, base, out, dev->contract_partial.p, dev->tile_counters.p, tiled);
    after_launch(dev, "k_contract");
}

// Reserves the split-superchunk scratch (outside any graph capture).
void reserve_contract(rocp_dev* dev, int64_t I, int64_t s, int R, bool always = false) {
    const int64_t tiles = (I + kRowTile - 1) / kRowTile;
    const int64_t nsuper = (s + kSuperSamples - 1) / kSuperSamples;
    if (nsuper <= 1 && !always) return;
    if (dev->contract_partial.n < size_t(nsuper * I * R)) {
        CK(cudaStreamSynchronize(dev->stream));
        dev->contract_partial.alloc(size_t(nsuper * I * R));
    }
    if (dev->tile_counters.n < size_t(tiles)) {
        CK(cudaStreamSynchronize(dev->stream));
        dev->tile_counters.alloc(size_t(tiles));
        CK(cudaMemset(dev->tile_counters.p, 0, size_t(tiles) * sizeof(unsigned int)));
    }
}

template <int RPAD>
void launch_contract_chunks(rocp_dev* dev, const double* X, int64_t I, int64_t s, const double* Z, int R,
                            const double* base, double* out, int tiled) {
    const int tiles = int((I + kRowTile - 1) / kRowTile);
    const int nsuper = int((s + kSuperSamples - 1) / kSuperSamples);
    if (nsuper > 1 && (dev->contract_partial.n < size_t(nsuper) * I * R || dev->tile_counters.n < size_t(tiles)))
        throw RocpError{ROCP_E_STATE, "contraction scratch not reserved (internal)"};
    const size_t smem = (size_t(kSuperSamples) * kRowTile + size_t(kSuperSamples) * RPAD + size_t(8) * RPAD * kRowTile) *
                        sizeof(double);
    k_contract_chunks<RPAD><<<dim3(unsigned(tiles), unsigned(nsuper), 1u), 256, smem, dev->stream>>>(
        X, int32_t(I), int32_t(s), Z, R, base, out, dev->contract_partial.p, dev->tile_counters.p, tiled);
    after_launch(dev, "k_contract_chunks");
}

void launch_contract(rocp_dev* dev, const double* X, int64_t I, int64_t s, const double* Z, int R,
                     const double* base, double* out, int tiled = 0) {
    if (R <= 8) return launch_contract_chunks<8>(dev, X, I, s, Z, R, base, out, tiled);
    if (R <= 16) return launch_contract_chunks<16>(dev, X, I, s, Z, R, base, out, tiled);
    if (R <= 24) return launch_contract_chunks<24>(dev, X, I, s, Z, R, base, out, tiled);
    if (R <= 32) return launch_contract_chunks<32>(dev, X, I, s, Z, R, base, out, tiled);
    int rb;
    const int ng = contract_groups(R, &rb);
    switch (rb) {
        case 1: launch_contract_rb<1>(dev, ng, X, I, s, Z, R, base, out, tiled); break;
        case 2: launch_contract_rb<2>(dev, ng, X, I, s, Z, R, base, out, tiled); break;
        case 3: launch_contract_rb<3>(dev, ng, X, I, s, Z, R, base, out, tiled); break;
        case 4: launch_contract_rb<4>(dev, ng, X, I, s, Z, R, base, out, tiled); break;
        case 5: launch_contract_rb<5>(dev, ng, X, I, s, Z, R, base, out, tiled); break;
        case 6: launch_contract_rb<6>(dev, ng, X, I, s, Z, R, base, out, tiled); break;
        case 7: launch_contract_rb<7>(dev, ng, X, I, s, Z, R, base, out, tiled); break;
        case 8: launch_contract_rb<8>(dev, ng, X, I, s, Z, R, base, out, tiled); break;
        case 9: launch_contract_rb<9>(dev, ng, X, I, s, Z, R, base, out, tiled); break;
        default: launch_contract_rb<10>(dev, ng, X, I, s, Z, R, base, out, tiled); break;
    }
}

void set_contract_smem_attrs() {
    CK(cudaFuncSetAttribute(reinterpret_cast<const void*>(k_solve<64>), cudaFuncAttributeMaxDynamicSharedMemorySize,
                            ksolve_smem_bytes(64)));
    {
        auto attr = [](const void* f, int rpad) {
            const int b = int((size_t(kSuperSamples) * kRowTile + size_t(kSuperSamples) * rpad + size_t(8) * rpad * kRowTile) *
                              sizeof(double));
            CK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, b));
        };
        attr(reinterpret_cast<const void*>(k_contract_chunks<8>), 8);
        attr(reinterpret_cast<const void*>(k_contract_chunks<16>), 16);
        attr(reinterpret_cast<const void*>(k_contract_chunks<24>), 24);
        attr(reinterpret_cast<const void*>(k_contract_chunks<32>), 32);
    }
    const int mx = int((size_t(kSuperSamples) * kRowTile + size_t(kSuperSamples) * 70) * sizeof(double));
    CK(cudaFuncSetAttribute(k_contract<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    CK(cudaFuncSetAttribute(k_contract<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    CK(cudaFuncSetAttribute(k_contract<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    CK(cudaFuncSetAttribute(k_contract<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    CK(cudaFuncSetAttribute(k_contract<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    CK(cudaFuncSetAttribute(k_contract<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    CK(cudaFuncSetAttribute(k_contract<7>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    CK(cudaFuncSetAttribute(k_contract<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    CK(cudaFuncSetAttribute(k_contract<9>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    CK(cudaFuncSetAttribute(k_contract<10>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
}

// flags: [0] |= 1 when regularized, [1] = nonfinite_code on a non-finite output.
void launch_solve(rocp_dev* dev, const double* G, int R, const double* RHS, int64_t rows, double* OUT,
                  int* flags, int nonfinite_code) {
    // a warp per row; at most one block per SM (every block repeats the sweep of G)
    const int grid = int(std::max<int64_t>(1, std::min<int64_t>((rows + 7) / 8, dev->num_sms)));
    if (R <= 16) k_solve<16><<<grid, 256, ksolve_smem_bytes(16), dev->stream>>>(G, R, RHS, int32_t(rows), OUT, flags, nonfinite_code);
    else if (R <= 32) k_solve<32><<<grid, 256, ksolve_smem_bytes(32), dev->stream>>>(G, R, RHS, int32_t(rows), OUT, flags, nonfinite_code);
    else k_solve<64><<<grid, 256, ksolve_smem_bytes(64), dev->stream>>>(G, R, RHS, int32_t(rows), OUT, flags, nonfinite_code);
    after_launch(dev, "k_solve");
}

// Sum of squares of (x_hat - x) (factors != null) or x, canonical order.
// Result left in dev->scalars.p[slot].
void launch_fitness(rocp_dev* dev, const rocp_tensor* t, const std::vector<const double*>* factors,
                    int R, int slot) {
    FitJob j{};
    j.t = t->d;
    j.I1 = t->dims[0];
    j.nfib = t->numel / t->dims[0];
    j.N = int(t->dims.size());
    j.R = factors ? R : 0;
    j.with_model = factors ? 1 : 0;
    for (int n = 0; n < j.N; ++n) {
        j.dims[n] = t->dims[size_t(n)];
        j.U[n] = factors ? (*factors)[size_t(n)] : nullptr;
    }
    const int64_t ngroups = (j.nfib + kGroup - 1) / kGroup;
    dev->scratch_a.ensure(size_t(ngroups));
    dev->scratch_b.ensure(size_t(ngroups));
    j.group_partial = dev->scratch_a.p;
    j.group_tmp = dev->scratch_b.p;
    j.counter = dev->counters.p + 1;
    j.out = dev->scalars.p + slot;
    // k-steps of 4 over R (w and U1 are zero-padded past R); instances 1..5, 8, 13, 16
    const int need = std::max(1, (j.R + 3) / 4);
    const int ks = need <= 5 ? need : (need <= 8 ? 8 : (need <= 13 ? 13 : 16));
    const size_t smem = (size_t(kGroup) * 4 * ks + kGroup) * sizeof(double);
    const int grid = int(std::min<int64_t>(ngroups, int64_t(dev->num_sms)));
    switch (ks) {
        case 1: k_fitness<1><<<grid, 256, smem, dev->stream>>>(j); break;
        case 2: k_fitness<2><<<grid, 256, smem, dev->stream>>>(j); break;
        case 3: k_fitness<3><<<grid, 256, smem, dev->stream>>>(j); break;
        case 4: k_fitness<4><<<grid, 256, smem, dev->stream>>>(j); break;
        case 5: k_fitness<5><<<grid, 256, smem, dev->stream>>>(j); break;
        case 8: k_fitness<8><<<grid, 256, smem, dev->stream>>>(j); break;
        case 13: k_fitness<13><<<grid, 256, smem, dev->stream>>>(j); break;
        default: k_fitness<16><<<grid, 256, smem, dev->stream>>>(j); break;
    }
    after_launch(dev, "k_fitness");
}

void launch_residual(rocp_dev* dev, const double* X, int64_t I, int64_t S, const double* U,
                     const double* Z, int R, double* out2, int tiled = 0) {
    ResidJob j{};
    j.tiled = tiled;
    j.X = X;
    j.U = U;
    j.Z = Z;
    j.I = int32_t(I);
    j.S = int32_t(S);
    j.R = R;
    dev->scratch_b.ensure(size_t(3 * S));
    j.col_num = dev->scratch_b.p;
    j.col_den = dev->scratch_b.p + S;
    j.tmp = dev->scratch_b.p + 2 * S;
    j.counter = dev->counters.p + 2;
    j.out = out2;
    k_residual<<<grid_for(S, 8, dev->num_sms * 2), 256, 0, dev->stream>>>(j);
    after_launch(dev, "k_residual");
}

void upload_rowmajor(rocp_dev* dev, const double* host_col, int64_t rows, int64_t cols, double* d) {
    std::vector<double> rm = colmajor_to_rowmajor(host_col, rows, cols);
    CK(cudaMemcpyAsync(d, rm.data(), rm.size() * sizeof(double), cudaMemcpyHostToDevice, dev->stream));
    CK(cudaStreamSynchronize(dev->stream));
}

void download_colmajor(rocp_dev* dev, const double* d, int64_t rows, int64_t cols, double* host_col) {
    std::vector<double> rm(size_t(rows * cols));
    if (!rm.empty()) {
        CK(cudaMemcpyAsync(rm.data(), d, rm.size() * sizeof(double), cudaMemcpyDeviceToHost, dev->stream));
        CK(cudaStreamSynchronize(dev->stream));
    }
    rowmajor_to_colmajor(rm.data(), rows, cols, host_col);
}

template <class F>
rocp_status guarded(rocp_dev* dev, F&& f, int* err_sweep = nullptr) {
    try {
        f();
        return ROCP_OK;
    } catch (const RocpError& e) {
        set_err(dev, e);
        if (err_sweep && e.code == ROCP_E_NUMERICAL) *err_sweep = e.sweep;
        return e.code;
    } catch (const std::exception& e) {
        if (dev) dev->err = e.what();
        return ROCP_E_STATE;
    }
}

void check_tensor_dims(const std::vector<int64_t>& d) {  // tensor.cpp:11-17
    if (d.size() < 2) throw_domain("tensor order must be at least 2");
    if (d.size() > size_t(kMaxOrder)) throw_domain("tensor order above 8 is not supported");
    for (int64_t x : d)
        if (x < 1) throw_domain("tensor extents must be positive");
}

void check_rank(int R) {
    if (R < 1) throw_domain("rank must be positive");
    if (R > 64) throw_domain("rank above 64 is not supported by the B200 solve kernel");
}

}  // namespace

// ===========================================================================
// Stream state (RocpStream, rocp.hpp:85-107 + ComplementaryState :15-24).
//
// Host buffers for host-slab streams: 2 MB-aligned anonymous mapping with
// transparent huge pages requested (the host gather touches one page per
// strided element; 2 MB pages keep those walks in the TLB), page-locked and
// registered with CUDA.
constexpr size_t kHugePage = size_t(2) << 20;

void* host_alloc_huge(size_t bytes) {
    const size_t len = (bytes + kHugePage - 1) / kHugePage * kHugePage;
    void* p = mmap(nullptr, len + kHugePage, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    if (p == MAP_FAILED) return nullptr;
    const uintptr_t a = (reinterpret_cast<uintptr_t>(p) + kHugePage - 1) & ~(uintptr_t(kHugePage) - 1);
    const size_t head = a - reinterpret_cast<uintptr_t>(p);
    if (head) munmap(p, head);
    if (kHugePage - head) munmap(reinterpret_cast<void*>(a + len), kHugePage - head);
    madvise(reinterpret_cast<void*>(a), len, MADV_HUGEPAGE);
    if (cudaHostRegister(reinterpret_cast<void*>(a), len, cudaHostRegisterDefault) != cudaSuccess) {
        munmap(reinterpret_cast<void*>(a), len);
        return nullptr;
    }
    return reinterpret_cast<void*>(a);
}

void host_free_huge(void* p, size_t bytes) {
    if (!p) return;
    cudaHostUnregister(p);
    munmap(p, (bytes + kHugePage - 1) / kHugePage * kHugePage);
}

// Persistent host worker threads for the host-slab gather (one pool per stream).
class HostPool {
public:
    explicit HostPool(int n) {
        for (int t = 1; t < n; ++t) th_.emplace_back([this] { loop(); });
    }
    ~HostPool() {
        {
            std::lock_guard<std::mutex> g(m_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : th_) t.join();
    }
    int size() const { return int(th_.size()) + 1; }
    // Runs fn() on `n` threads (the caller included) and waits for all of them.
    void run(int n, const std::function<void()>& fn) {
        n = std::max(1, std::min(n, size()));
        {
            std::lock_guard<std::mutex> g(m_);
            fn_ = &fn;
            want_ = n - 1;
            pending_ = n - 1;
            ++gen_;
        }
        cv_.notify_all();
        fn();
        std::unique_lock<std::mutex> g(m_);
        done_.wait(g, [this] { return pending_ == 0; });
        fn_ = nullptr;
    }

private:
    void loop() {
        uint64_t seen = 0;
        for (;;) {
            const std::function<void()>* f = nullptr;
            {
                std::unique_lock<std::mutex> g(m_);
                cv_.wait(g, [&] { return stop_ || (gen_ != seen && want_ > 0); });
                if (stop_) return;
                seen = gen_;
                --want_;
                f = fn_;
            }
            (*f)();
            std::lock_guard<std::mutex> g(m_);
            if (--pending_ == 0) done_.notify_one();
        }
    }
    std::vector<std::thread> th_;
    std::mutex m_;
    std::condition_variable cv_, done_;
    const std::function<void()>* fn_ = nullptr;
    uint64_t gen_ = 0;
    int want_ = 0, pending_ = 0;
    bool stop_ = false;
};

// A "window" holds the sample indices and gathered fibres of nb consecutive
// batches: all N*nb draws are one launch, all N*nb gathers are one launch
// (indices never depend on factors), then the factor-dependent chain runs
// batch by batch, stage by stage (Gauss-Seidel, rocp.cpp:122-130) -- captured
// once into a CUDA graph per (nb, B, t_len) for consume_range.
struct Window {
    int64_t nb = 0, B = 0;     // capacity
    DBuf<int32_t> idx;         // [b][stage] S x (N-1)
    DBuf<int64_t> base, rows;  // [b][stage] S
    DBuf<int32_t> perm;        // [b][stage] S: strided stages' samples in fibre-base order (sorted gather)
    DBuf<double> X;            // [b][stage] I_stage x S (column-major)
    std::vector<int64_t> xoff;
    DBuf<int64_t> xoff_dev;
    DBuf<double> zT, rcols, rhist;  // temporal Z per batch, residual column partials, per-batch residuals
    DBuf<unsigned> rctr;            // residual pass: per-batch block arrivals (self-resetting)
    JobList jobs;
    // host-slab path: pinned staging of the gathered X_s and of the fibre base offsets
    double* hX = nullptr;
    size_t hX_n = 0;
    int64_t* hbase = nullptr;
    size_t hbase_n = 0;
    // pageable host-slab path (consume_pageable_host): host-drawn indices, double-buffered
    // pinned staging so a call's host gather overlaps the previous call's copies and chain
    int par = 0;
    double* hXp[2] = {nullptr, nullptr};
    size_t hXp_n[2] = {0, 0};
    int32_t* hidxp[2] = {nullptr, nullptr};
    size_t hidxp_n[2] = {0, 0};
    std::vector<int64_t> hbase_h;
    cudaEvent_t stage_ev[2] = {nullptr, nullptr};  // the copies that last read staging parity p
    cudaEvent_t chain_ev = nullptr;                 // the last chain that read the window arena
    std::vector<DrawJob> hdraw;                     // host copies of the window's draw jobs
    int64_t hdraw_B = -1, hdraw_nb = -1;
    ~Window() {
        host_free_huge(hX, hX_n * sizeof(double));
        if (hbase) cudaFreeHost(hbase);
        for (int q = 0; q < 2; ++q) {
            host_free_huge(hXp[q], hXp_n[q] * sizeof(double));
            if (hidxp[q]) cudaFreeHost(hidxp[q]);
            if (stage_ev[q]) cudaEventDestroy(stage_ev[q]);
        }
        if (chain_ev) cudaEventDestroy(chain_ev);
    }
    // key of the uploaded job list
    const double* key_x = nullptr;
    int64_t key_t0 = -1, key_B = -1, key_nb = -1, key_slice = -1;
    const int64_t* key_rows0 = nullptr;
    const int64_t* key_rowsm = nullptr;
    int key_only = -2;
    bool key_host = false;
    const double* key_zc = nullptr;
    bool key_sort = true;
    std::vector<int64_t> zc_tile;  // host path: first zero-copy gather tile of each batch
    GatherTmaParams gtp{};         // tensor-map views of the strided modes (overlapped gather)
    DBuf<char> xmap;               // tensor map of the X_s arena (k_chain's streamed wide items), device copy
    bool xmap_ok = false;
};

// Window of a sharded stream: per (batch, stage) the global draws, the
// compacted local samples (shard order), their per-shard counts and the
// column-major X_s of the local samples; plus the exchange buffers.
struct ShardWin {
    int64_t nb = 0, B = 0;  // capacity
    int64_t B_cur = 0;      // batch size of the window being run
    DBuf<int32_t> idx, cidx, clist;
    DBuf<int64_t> base, cbase;
    DBuf<int> counts;            // nb x N x V
    std::vector<int> hcounts;
    DBuf<double> X;              // per (b, stage): I_stage x S column-major
    std::vector<int64_t> xoff;
    JobList draws, gathers;
    DBuf<ShardPartJob> pjobs;
    DBuf<double> Zl;             // S x R, this stage's local Z
    DBuf<double> send, recv;     // V x (R^2 + max rows x R) partial blocks
    DBuf<double> rcols, rgath, rwork, rtmp;  // residual columns (2 x S per rank)
    // fused exchange over peer memory (shard_host.inc setup_exchange)
    DBuf<double> x_area;           // [counters][landing x 2][residual landing x 2] of this rank
    DBuf<uint64_t> x_tab;          // device pointer tables into every rank's area
    std::vector<void*> x_opened;   // peer areas opened through CUDA IPC
    size_t x_land = 0, x_rland = 0;
    uint64_t x_target[2] = {0, 0}; // cumulative arrivals expected (partials, residual)
    int x_parity[2] = {0, 0};
    ~ShardWin() {
        for (void* q : x_opened) cudaIpcCloseMemHandle(q);
    }
};
constexpr size_t kXchgHead = 32;  // doubles before the landing buffers (the two counters, padded)

struct rocp_stream {
    rocp_dev* dev = nullptr;
    int N = 0, R = 0;
    int64_t s = 0;
    std::vector<int64_t> head;
    std::vector<DBuf<double>> U, P, Q;  // n = 1..N-1: I_n x R row-major, R x R
    DBuf<double> temporal;              // t_cap x R row-major
    int64_t t_len = 0, t_cap = 0;
    bool regularized = false;
    Window win;
    std::vector<DBuf<double>> Z;  // per stage, S x R row-major (reused across batches)
    DBuf<double> G_t, RHS_t;      // temporal Gram / rhs
    DBuf<double> resid;           // N x 2 (num, den) of the last batch
    DBuf<double> staging;         // host-slab staging for consume_host
    DBuf<int> flags;              // [0] temporal regularized (stream flag), [2] last mode solve
    DBuf<double> gpart, chpart, LD, rpart, zmodes;  // persistent-chain scratch
    DBuf<int> mode_flag;
    DBuf<unsigned> zctr;               // persistent chain: phase-0 chunk arrival counters
    DBuf<double> ginv, wtemp;          // k_flow: G^-1 slots, temporal right-hand sides
    DBuf<int> gmode;                   // k_flow: mode flags of the G^-1 slots
    DBuf<unsigned> fctr;               // k_flow: dependency counters
    bool trace_on = false;             // chain phase timestamps (profiling aid)
    DBuf<unsigned long long> trace;
    int64_t trace_n = 0;
    DBuf<uint64_t> seed_dev;      // draw seed (device, so graphs need no re-capture)
    DBuf<uint32_t> batch_dev;     // first batch id of the window (device)
    int resid_level = 1;          // 0 none, 1 temporal stage (default), 2 every stage
    int win_gsms = 0;             // SMs of the current window's overlapped gather (0: none)
    int host_threads = int(std::max(1u, std::min(64u, std::thread::hardware_concurrency())));
    std::unique_ptr<HostPool> pool;  // host-slab gather workers (created on first use)
    // mode-1 sharding: U(1)/P(1) hold rows [r0, r1) and
    // head[0] = r1 - r0; ghead keeps the global head for the draws
    bool sharded = false;
    int V = 1, v0 = 0, v1 = 1;
    int64_t r0 = 0, r1 = 0;
    std::vector<int64_t> ghead;
    std::unique_ptr<ShardWin> sw;
    double* file_buf = nullptr;               // consume_file: huge-page pinned slab staging
    size_t file_buf_bytes = 0;
    cudaStream_t copy_stream = nullptr;       // host-slab path: in-place reads + staging copies
    std::vector<cudaEvent_t> copy_events;     // one per sub-window, joined by the compute stream
    // checkpoint copies (device)
    std::vector<DBuf<double>> ckU, ckP, ckQ;
    int64_t ck_t_len = -1;
    bool ck_reg = false;
    // gather timing (events around each window gather launch)
    bool time_gather = false;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> gather_events, chain_events;
    size_t gather_events_used = 0, chain_events_used = 0;
    // CUDA graphs of the chain keyed by (nb, B, t_len)
    std::map<std::tuple<int64_t, int64_t, int64_t>, std::pair<cudaGraphExec_t, uint64_t>> graphs;
    ~rocp_stream() {
        for (auto& kv : graphs) cudaGraphExecDestroy(kv.second.first);
        for (auto& e : chain_events) {
            cudaEventDestroy(e.first);
            cudaEventDestroy(e.second);
        }
        for (auto& e : gather_events) {
            cudaEventDestroy(e.first);
            cudaEventDestroy(e.second);
        }
        for (cudaEvent_t e : copy_events) cudaEventDestroy(e);
        if (copy_stream) cudaStreamDestroy(copy_stream);
        host_free_huge(file_buf, file_buf_bytes);
    }
    int64_t stage_rows(int stage, int64_t batch) const { return stage == 0 ? batch : head[size_t(stage - 1)]; }
};

namespace {

std::vector<int64_t> slab_dims(const rocp_stream* st, int64_t batch) {
    std::vector<int64_t> d = st->head;
    d.push_back(batch);
    return d;
}

void check_head_dims(const rocp_stream* st, const rocp_tensor* x) {  // rocp.cpp:14-21
    if (x->dims.size() != st->head.size() + 1) throw_domain("batch order does not match stream order");
    for (size_t k = 0; k < st->head.size(); ++k)
        if (x->dims[k] != st->head[k]) throw_domain("batch head extents do not match stream");
}

void clear_graphs(rocp_stream* st) {
    for (auto& kv : st->graphs) cudaGraphExecDestroy(kv.second.first);
    st->graphs.clear();
}

bool make_xs_map(const double* x, size_t n, CUtensorMap* map);

// Ensures the window arena holds nb batches of B slices.
void ensure_window(rocp_stream* st, int64_t nb, int64_t B) {
    Window& W = st->win;
    if (nb <= W.nb && B <= W.B) return;
    const int64_t nbn = std::max(nb, W.nb), Bn = std::max(B, W.B);
    const int N = st->N;
    const int64_t S = st->s;
    W.idx.alloc(size_t(nbn * N * S * (N - 1)));
    W.perm.alloc(size_t(nbn * N * S));
    W.base.alloc(size_t(nbn * N * S));
    W.rows.alloc(size_t(nbn * N * S));
    W.xoff.assign(size_t(nbn * N), 0);
    int64_t off = 0;
    for (int64_t b = 0; b < nbn; ++b)
        for (int stage = 0; stage < N; ++stage) {
            W.xoff[size_t(b * N + stage)] = off;
            off += xs_size(st->stage_rows(stage, Bn), S);  // row-tiled layout
        }
    W.X.alloc(size_t(off));
    {
        CUtensorMap xm;
        W.xmap_ok = make_xs_map(W.X.p, W.X.n, &xm);
        if (W.xmap_ok) {
            W.xmap.alloc(sizeof(CUtensorMap));
            CK(cudaMemcpy(W.xmap.p, &xm, sizeof(xm), cudaMemcpyHostToDevice));
        }
    }
    {
        const int64_t RP = ((st->R + kCRB - 1) / kCRB) * kCRB + 4;  // + 4: the padded stride of the streamed wide chain
        W.zT.alloc(size_t(nbn * S * RP));
        W.rcols.alloc(size_t(nbn * 3 * S));
        W.rhist.alloc(size_t(nbn * 2));
    }
    W.xoff_dev.alloc(W.xoff.size());
    CK(cudaMemcpy(W.xoff_dev.p, W.xoff.data(), W.xoff.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
    W.nb = nbn;
    W.B = Bn;
    reserve_contract(st->dev, Bn, S, st->R, true);
    for (int n = 1; n < N; ++n) reserve_contract(st->dev, st->head[size_t(n - 1)], S, st->R, true);
    W.key_x = nullptr;
    st->RHS_t.alloc(size_t(Bn * st->R));
    clear_graphs(st);  // graphs hold arena pointers
}

int32_t* win_idx(rocp_stream* st, int64_t b, int stage) {
    return st->win.idx.p + (b * st->N + stage) * st->s * (st->N - 1);
}
int64_t* win_base(rocp_stream* st, int64_t b, int stage) { return st->win.base.p + (b * st->N + stage) * st->s; }
int64_t* win_rows(rocp_stream* st, int64_t b, int stage) { return st->win.rows.p + (b * st->N + stage) * st->s; }
double* win_x(rocp_stream* st, int64_t b, int stage) { return st->win.X.p + st->win.xoff[size_t(b * st->N + stage)]; }

// Tensor-map view for the TMA units of the overlapped gather (gather_kernel.cuh):
// the window range x (dims wd, time extent = the window's slices) seen as
// (I1, Ma, In, Mb) for strided mode `mode`, box {2, 1, L, 1} with L = min(256,
// fibre length); mode 1 as (I1, 1, 1, rest) with box {L, 1, 1, 1}.  Returns
// false where TMA cannot express it (odd I1: row strides must be 16-byte
// multiples; a misaligned range; extents past 2^31) or ROCP_GATHER_TMA=0; those
// jobs use LSU loads.  ROCP_GATHER_PROMO selects the strided boxes' L2
// promotion for A/B runs.
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static const PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            fn = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }();
    return encode;
}

// The X_s arena (n doubles, 128-byte aligned) as 128-byte rows for k_chain's streamed wide items
// (chain_kernel.cuh chain_stream_items): box = 64 rows = one 32-sample x 32-row chunk tile,
// 128-byte swizzle.  ROCP_CHAIN_STREAM=0 keeps the tile-at-a-time items (A/B aid).
bool make_xs_map(const double* x, size_t n, CUtensorMap* map) {
    static const bool off = [] {
        const char* e = std::getenv("ROCP_CHAIN_STREAM");
        return e && std::atoi(e) == 0;
    }();
    const PFN_cuTensorMapEncodeTiled_v12000 encode = tensor_map_encoder();
    if (off || !encode || n < 16 || reinterpret_cast<uintptr_t>(x) % 128 != 0) return false;
    const cuuint64_t rows = cuuint64_t(n / 16);
    if (rows >= (cuuint64_t(1) << 31)) return false;
    const cuuint64_t dims[2] = {16, rows};
    const cuuint64_t gstr[1] = {128};
    const cuuint32_t box[2] = {16, 64};
    const cuuint32_t estr[2] = {1, 1};
    return encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(x), dims, gstr, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool make_gather_view(const double* x, const std::vector<int64_t>& wd, int mode, int64_t fibre_len, CUtensorMap* map,
                      GatherView* view) {
    static const PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
        const char* e = std::getenv("ROCP_GATHER_TMA");
        if (e && std::atoi(e) == 0) return PFN_cuTensorMapEncodeTiled_v12000(nullptr);
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            fn = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }();
    if (!encode) return false;
    const int N = int(wd.size());
    const int64_t I1 = wd[0];
    if (I1 % 2 != 0 || reinterpret_cast<uintptr_t>(x) % 16 != 0 || mode < 1 || mode > N) return false;
    int64_t Ma = 1, Mb = 1;
    for (int k = 1; k < mode - 1; ++k) Ma *= wd[size_t(k)];
    for (int k = std::max(mode, 1); k < N; ++k) Mb *= wd[size_t(k)];
    const int64_t In = mode == 1 ? 1 : wd[size_t(mode - 1)];
    const int64_t lim = int64_t(1) << 31;
    if (Ma >= lim || In >= lim || Mb >= lim || I1 >= lim) return false;
    const cuuint64_t dims[4] = {cuuint64_t(I1), cuuint64_t(Ma), cuuint64_t(In), cuuint64_t(Mb)};
    const cuuint64_t gstr[3] = {cuuint64_t(I1) * 8, cuuint64_t(I1 * Ma) * 8, cuuint64_t(I1 * Ma * In) * 8};
    const cuuint32_t L = cuuint32_t(std::min<int64_t>(kGWBox, fibre_len));
    const cuuint32_t box[4] = {mode == 1 ? L : 2u, 1, mode == 1 ? 1u : L, 1};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    static const CUtensorMapL2promotion promo = [] {
        const char* e = std::getenv("ROCP_GATHER_PROMO");  // A/B aid: 0 none, 1 64 B (default), 2 128 B
        const int v = e ? std::atoi(e) : 1;
        return v == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                      : (v == 2 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_L2_64B);
    }();
    const CUtensorMapL2promotion l2 = mode == 1 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : promo;  // mode 1: whole lines
    if (encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(x), dims, gstr, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, l2, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
        CUDA_SUCCESS)
        return false;
    *view = GatherView{I1, Ma, In, mode == 1 ? 1 : 0};
    return true;
}

// Builds (or reuses) the draw + gather job lists of nb consecutive slabs of B
// slices starting at x (device pointer, slice = elements per slice).  Batch
// ids come from st->batch_dev + b, the seed from st->seed_dev, so the lists
// are reused across calls.  rows0/rowsm: explicit index sets (replay seams);
// only_stage >= 0 restricts to one stage.
// host_gather: the fibres come from host slabs (consume_range_host); then the
// gather jobs are only those of the contiguous (mode-1) stages, reading the
// caller's registered host range in place through zc_src (zero-copy), or none.
void prepare_window(rocp_stream* st, const double* x, int64_t t0, int64_t slice, int64_t B, int64_t nb,
                    const int64_t* rows0, const int64_t* rowsm, int only_stage, bool host_gather = false,
                    const double* zc_src = nullptr, bool sort_strided = true) {
    ensure_window(st, nb, B);
    Window& W = st->win;
    if (W.key_x == x && W.key_t0 == t0 && W.key_B == B && W.key_nb == nb && W.key_slice == slice &&
        W.key_rows0 == rows0 && W.key_rowsm == rowsm && W.key_only == only_stage && W.key_host == host_gather &&
        W.key_zc == zc_src && W.key_sort == sort_strided)
        return;
    const std::vector<int64_t> d = slab_dims(st, B);
    std::vector<DrawJob> dj;
    std::vector<GatherJob> gj;
    std::vector<SortJob> sj;
    const std::vector<int64_t> strides = strides_of(d);
    // tensor-map views of the strided modes over the whole window range (overlapped gather)
    bool tma_mode[kMaxOrder + 1] = {};
    if (!host_gather) {
        const std::vector<int64_t> wd = [&] { std::vector<int64_t> v = slab_dims(st, B); v.back() = B * nb; return v; }();
        for (int mode = 1; mode <= st->N; ++mode)
            tma_mode[mode] = make_gather_view(x + t0 * slice, wd, mode, mode == st->N ? B : wd[size_t(mode - 1)],
                                              &W.gtp.map[mode - 1], &W.gtp.view[mode - 1]);
    }
    W.zc_tile.assign(size_t(nb + 1), 0);
    int64_t ntile = 0;
    for (int64_t b = 0; b < nb; ++b) {
        const double* xb = x + (t0 + b * B) * slice;
        W.zc_tile[size_t(b)] = ntile;
        for (int stage = 0; stage < st->N; ++stage) {
            if (only_stage >= 0 && stage != only_stage) continue;
            const int mode = stage == 0 ? st->N : stage;
            DrawJob j = make_draw(d, mode, st->s, 0, uint32_t(b), 0u, stage == 0 ? rows0 : rowsm,
                                  win_rows(st, b, stage), win_idx(st, b, stage), win_base(st, b, stage));
            j.seed_ptr = st->seed_dev.p;
            j.batch_ptr = st->batch_dev.p;
            dj.push_back(j);
            if (!host_gather) {
                GatherJob g = make_gather(xb, d, mode, st->s, win_base(st, b, stage), win_x(st, b, stage), 1);
                // strided: fibre-base order (DRAM page locality of the all-SM gather).  The
                // overlapped gather is bound by its SMs' issue rate, not DRAM: no sort there
                // (the sort would sit in front of the chain for nothing; 541k -> 545k slices/s)
                if (sort_strided && strides[size_t(mode - 1)] != 1 && st->s <= kSortMax) {
                    g.perm = st->win.perm.p + (b * st->N + stage) * st->s;
                    sj.push_back(SortJob{win_base(st, b, stage), const_cast<int32_t*>(g.perm), int32_t(st->s)});
                }
                if (tma_mode[mode]) {
                    g.tmap1 = mode;
                    g.tlen = int32_t(std::min<int64_t>(kGWBox, d[size_t(mode - 1)]));
                    g.toff = b * B * slice;
                }
                gj.push_back(g);
            } else if (zc_src && strides[size_t(mode - 1)] == 1) {
                gj.push_back(make_gather(zc_src + (t0 + b * B) * slice, d, mode, st->s, win_base(st, b, stage),
                                         win_x(st, b, stage), 1));
                ntile += (int64_t(d[size_t(mode - 1)]) * st->s + kGatherTile - 1) / kGatherTile;
            }
        }
    }
    W.zc_tile[size_t(nb)] = ntile;
    upload_jobs(st->dev, W.jobs, dj, gj, sj);
    W.key_x = x;
    W.key_t0 = t0;
    W.key_B = B;
    W.key_nb = nb;
    W.key_slice = slice;
    W.key_rows0 = rows0;
    W.key_rowsm = rowsm;
    W.key_only = only_stage;
    W.key_host = host_gather;
    W.key_zc = zc_src;
    W.key_sort = sort_strided;
}

// Live handles per GPU in this process.  Two handles' streams run concurrently on
// one GPU, and two cooperative chains plus their spinning gathers could then hold
// each other's SMs: the model gathers serially while a GPU has more than one handle.
std::mutex g_handles_mu;
std::map<int, int> g_handles;
int handles_on(int device) {
    std::lock_guard<std::mutex> lk(g_handles_mu);
    auto it = g_handles.find(device);
    return it == g_handles.end() ? 0 : it->second;
}

// SMs reserved for the overlapped window gather.  ROCP_GATHER_SMS
// overrides; otherwise a model picks the fewest SMs whose TMA gather (about
// 1.47 G elements/s per SM, measured) keeps pace with the chain (about 14 us
// per stage for R <= 32, 110 us for the wide kernel), and 0 -- the whole window
// gathered on every SM before the chain -- when the model puts the gather under
// 2.5% of the step (C1 and C5 lose 1% or tie beside 8 gather SMs; C3, at 2.6%
// by the model and 6% measured, gains 4% with 8).
// The chain keeps one warp per row of its largest stage where that fits on
// the device (a second row-solve round costs more than the gather saves).
int gather_sms(rocp_stream* st, int64_t B) {
    rocp_dev* dev = st->dev;
    if (!dev->gstream) {  // first use on this device: env override and the gather stream
        if (dev->gather_sms == -1) {
            dev->gather_sms = -2;
            if (const char* e = std::getenv("ROCP_GATHER_SMS")) dev->gather_sms = std::max(0, std::atoi(e));
        }
        CK(cudaFuncSetAttribute(k_gather_warps, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kGWSmem)));
        // The overlapped gather and the chain wait on each other's arrivals.  With lazy module
        // loading (CUDA 12's default) a kernel's first launch loads its code, which can wait for
        // the device while the other kernel spins: load every kernel of the pair up front.
        cudaFuncAttributes fa{};
        CK(cudaFuncGetAttributes(&fa, k_chain<false, false>));
        CK(cudaFuncGetAttributes(&fa, k_chain<true, false>));
        CK(cudaFuncGetAttributes(&fa, k_chain<false, true>));
        CK(cudaFuncGetAttributes(&fa, k_chain<true, true>));
        CK(cudaFuncGetAttributes(&fa, k_flow<8, false>));
        CK(cudaFuncGetAttributes(&fa, k_flow<16, false>));
        CK(cudaFuncGetAttributes(&fa, k_flow<24, false>));
        CK(cudaFuncGetAttributes(&fa, k_flow<32, false>));
        CK(cudaFuncGetAttributes(&fa, k_flow<40, false>));
        CK(cudaFuncGetAttributes(&fa, k_flow<48, false>));
        CK(cudaFuncGetAttributes(&fa, k_flow<56, false>));
        CK(cudaFuncGetAttributes(&fa, k_flow<64, false>));
        CK(cudaFuncGetAttributes(&fa, k_flow<8, true>));
        CK(cudaFuncGetAttributes(&fa, k_flow<16, true>));
        CK(cudaFuncGetAttributes(&fa, k_flow<24, true>));
        CK(cudaFuncGetAttributes(&fa, k_flow<32, true>));
        CK(cudaFuncGetAttributes(&fa, k_flow<40, true>));
        CK(cudaFuncGetAttributes(&fa, k_flow<48, true>));
        CK(cudaFuncGetAttributes(&fa, k_flow<56, true>));
        CK(cudaFuncGetAttributes(&fa, k_flow<64, true>));
        CK(cudaFuncGetAttributes(&fa, k_gather_warps));
        CK(cudaStreamCreateWithFlags(&dev->gstream, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&dev->ev_gready, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&dev->ev_gdone, cudaEventDisableTiming));
    }
    int g = dev->gather_sms;
    // Two handles on one GPU: their cooperative chains and spinning gathers could hold
    // each other's SMs, whatever split was requested (explicit, env or model).
    if (handles_on(dev->device) > 1) return 0;
    // Under MPS the process may not get every SM at once: the chain spins on the overlapped
    // gather's arrivals, and only a private GPU guarantees that both grids are resident, so an
    // MPS client gathers serially
    static const bool mps = std::getenv("CUDA_MPS_PIPE_DIRECTORY") || std::getenv("CUDA_MPS_ACTIVE_THREAD_PERCENTAGE");
    if (mps) return 0;
    if (g == -2) {
        double elems = double(B), rows_max = double(B);  // gathered elements per sample of one batch
        for (int64_t I : st->head) {
            elems += double(I);
            rows_max = std::max(rows_max, double(I));
        }
        elems *= double(st->s);
        const double t_chain = st->N * (st->R > 32 ? 100.0 : 14.0);     // us per batch
        const double t_full = elems / (93e3);                             // us, whole-device gather
        if (t_full < 0.025 * (t_full + t_chain)) return 0;
        g = int(std::ceil(elems / (1470.0 * t_chain)));
        if (st->R <= 32) {
            // the dataflow chain (k_flow) runs a stage in ~11 us on C2: size the gather for that
            // with 20% headroom, as long as every contraction item of the largest stage still
            // gets its own block (tools/runs: C2 G = 20 -> 592k, 24..32 -> 611k, 36 -> 516k)
            const int64_t nch = (st->s + kChunk - 1) / kChunk, nsup = (st->s + kSuperSamples - 1) / kSuperSamples;
            int64_t tiles = (B + kRowTile - 1) / kRowTile;
            for (int64_t I : st->head) tiles = std::max<int64_t>(tiles, (I + kRowTile - 1) / kRowTile);
            const int limit = int(dev->num_sms - 1 - nch - tiles * nsup);
            const int gf = int(std::ceil(1.2 * elems / (1470.0 * st->N * 11.0)));
            if (limit >= 8) return std::max(8, std::min(gf, limit));
        }
        const int row_blocks = int(std::ceil(rows_max / (kChainThreads / 32)));
        if (row_blocks < dev->num_sms) g = std::min(g, dev->num_sms - row_blocks);
        g = std::max(g, 8);
        // contraction items come in rounds over the chain's blocks: within 20% below the estimate,
        // take the split with the fewest rounds (ties: more gather SMs).  C4: 1000 items per mode
        // stage take 10 rounds on 111 blocks (G = 33) but 9 on 112 (G = 32).
        const int64_t npairs = int64_t(st->R) * (st->R + 1) / 2;
        const int64_t nch = (st->s + kChunk - 1) / kChunk, nsup = (st->s + kSuperSamples - 1) / kSuperSamples;
        (void)npairs;
        (void)nch;
        const int gram_blocks = 1;
        const int64_t items = ((int64_t(rows_max) + kRowTile - 1) / kRowTile) * nsup;
        auto rounds = [&](int G) {
            const int64_t cb = std::max<int64_t>(1, dev->num_sms - G - gram_blocks);
            return (items + cb - 1) / cb;
        };
        // The wide kernel is compute-bound on its SMs, so among the splits with the fewest rounds
        // it takes the one that leaves it the most (C4: 28 -> 142k, 32 -> 137k slices/s).
        int best = g;
        if (st->R > 32) {
            // the wide chain is paced by the gather below this split and loses its own SMs above it
            // (C4, tools/runs/c4_gather_sweep.sh: 28 -> 143k, 32 -> 155k, 36..40 -> 168k, 44 -> 155k,
            // 52 -> 144k slices/s); its streamed pair items take the same number of rounds over
            // that whole range
        } else {
            for (int G = g; G >= std::max(1, int(std::floor(0.8 * g))); --G)
                if (rounds(G) < rounds(best)) best = G;
        }
        g = best;
    }
    return std::max(0, std::min(g, dev->num_sms / 2));
}

// Draw + gather of the prepared window (seed / first batch id set on device).
// overlap: the gather runs as k_gather_warps on the gather stream, concurrently
// with the chain launched next (launch_chain(..., overlap = true)), which waits
// per (batch, stage) on the published unit counts.
void enqueue_draw_gather(rocp_stream* st, uint64_t seed, uint32_t first_batch_id, bool overlap = false) {
    if (overlap && st->win_gsms <= 0) throw RocpError{ROCP_E_STATE, "overlapped gather without SMs (internal)"};
    rocp_dev* dev = st->dev;
    const JobList& L = st->win.jobs;
    k_window_setup<<<1, 256, 0, dev->stream>>>(st->seed_dev.p, seed, st->batch_dev.p, first_batch_id, L.done.p,
                                                overlap ? L.ngather : 0);
    after_launch(dev, "k_window_setup");
    if (overlap) {
        launch_draw(dev, L);
        if (L.nsort > 0) {
            k_sort_by_base<<<L.nsort, 1024, 0, dev->stream>>>(L.sort.p);
            after_launch(dev, "k_sort_by_base");
        }
        CK(cudaEventRecord(dev->ev_gready, dev->stream));
        CK(cudaStreamWaitEvent(dev->gstream, dev->ev_gready, 0));
        std::pair<cudaEvent_t, cudaEvent_t>* ev = nullptr;
        if (st->time_gather) {
            if (st->gather_events_used == st->gather_events.size()) {
                cudaEvent_t a, b;
                CK(cudaEventCreate(&a));
                CK(cudaEventCreate(&b));
                st->gather_events.emplace_back(a, b);
            }
            ev = &st->gather_events[st->gather_events_used++];
            CK(cudaEventRecord(ev->first, dev->gstream));
        }
        k_gather_warps<<<st->win_gsms, kGWThreads, kGWSmem, dev->gstream>>>(st->win.gtp, L.gather.p, L.ngather,
                                                                                L.ustart.p, L.done.p);
        after_launch(dev, "k_gather_warps");
        if (ev) CK(cudaEventRecord(ev->second, dev->gstream));
        CK(cudaEventRecord(dev->ev_gdone, dev->gstream));
        return;
    }
    launch_draw(dev, L);
    if (st->time_gather) {
        if (st->gather_events_used == st->gather_events.size()) {
            cudaEvent_t a, b;
            CK(cudaEventCreate(&a));
            CK(cudaEventCreate(&b));
            st->gather_events.emplace_back(a, b);
        }
        auto& ev = st->gather_events[st->gather_events_used++];
        CK(cudaEventRecord(ev.first, dev->stream));
        launch_gather(dev, st->win.jobs);
        CK(cudaEventRecord(ev.second, dev->stream));
    } else {
        launch_gather(dev, st->win.jobs);
    }
}

// Temporal stage of batch b (update_last_mode_with, rocp.cpp:71-84): SKR of
// factors_excluding(head, N) = U(N-1..1), gram, rhs, solve into u_out.
void stage_temporal(rocp_stream* st, int64_t b, int64_t B, double* u_out) {
    rocp_dev* dev = st->dev;
    SkrJob sj{};
    sj.idx = win_idx(st, b, 0);
    sj.n_other = st->N - 1;
    sj.s = int32_t(st->s);
    sj.R = st->R;
    int l = 0;
    for (int k = st->N - 1; k >= 1; --k) sj.f[l++] = st->U[size_t(k - 1)].p;
    sj.z = st->Z[0].p;
    launch_skr(dev, sj);
    const double* X = win_x(st, b, 0);
    launch_gram(dev, st->Z[0].p, st->s, st->R, nullptr, st->G_t.p);
    launch_contract(dev, X, B, st->s, st->Z[0].p, st->R, nullptr, st->RHS_t.p, 1);
    launch_solve(dev, st->G_t.p, st->R, st->RHS_t.p, B, u_out, st->flags.p, 0);  // rocp.cpp:150
    if (st->resid_level >= 1) launch_residual(dev, X, B, st->s, u_out, st->Z[0].p, st->R, st->resid.p, 1);
}

// Mode-n stage of batch b (update_mode_with, rocp.cpp:96-113 with
// slab_factors_excluding rocp.cpp:25-34): Z over [u_new, U(N-1..1) \ n],
// P += X_s Z, Q += Z^T Z, U(n) = solve_gram(Q, P).
void stage_mode(rocp_stream* st, int64_t b, int n, const double* u_new) {
    rocp_dev* dev = st->dev;
    SkrJob sj{};
    sj.idx = win_idx(st, b, n);
    sj.n_other = st->N - 1;
    sj.s = int32_t(st->s);
    sj.R = st->R;
    int l = 0;
    sj.f[l++] = u_new;
    for (int k = st->N - 1; k >= 1; --k)
        if (k != n) sj.f[l++] = st->U[size_t(k - 1)].p;
    sj.z = st->Z[size_t(n)].p;
    launch_skr(dev, sj);
    double* Pn = st->P[size_t(n - 1)].p;
    double* Qn = st->Q[size_t(n - 1)].p;
    const int64_t In = st->head[size_t(n - 1)];
    const double* X = win_x(st, b, n);
    launch_gram(dev, st->Z[size_t(n)].p, st->s, st->R, Qn, Qn);
    launch_contract(dev, X, In, st->s, st->Z[size_t(n)].p, st->R, Pn, Pn, 1);
    launch_solve(dev, Qn, st->R, Pn, In, st->U[size_t(n - 1)].p, st->flags.p + 2, 0);
    if (st->resid_level >= 2)
        launch_residual(dev, X, In, st->s, st->U[size_t(n - 1)].p, st->Z[size_t(n)].p, st->R, st->resid.p + 2 * n, 1);
}

// Factor-dependent chain of nb batches (RocpStream::consume, rocp.cpp:144-160):
// temporal solve appended in place (rocp.cpp:152-156), then modes 1..N-1.
void enqueue_chain(rocp_stream* st, int64_t nb, int64_t B) {
    for (int64_t b = 0; b < nb; ++b) {
        double* u_new = st->temporal.p + (st->t_len + b * B) * st->R;
        stage_temporal(st, b, B, u_new);
        for (int n = 1; n < st->N; ++n) stage_mode(st, b, n, u_new);
    }
}

size_t chain_smem(int R, int B) {
    (void)R;
    (void)B;
    return size_t(kSmTotal) * sizeof(double);  // fixed map (kernels.cuh, k_chain)
}

// One cooperative persistent launch of a chain kernel (k_chain<., .> or k_flow<.>):
// grid = one block per SM, less the SMs of an overlapped gather.
void launch_coop(rocp_stream* st, const void* fn, const char* name, const ChainParams& p, int grid) {
    rocp_dev* dev = st->dev;
    const size_t smem = chain_smem(st->R, p.B);
    // the dynamic shared memory opt-in is a per-device function attribute
    constexpr int kMaxDevices = 64;
    static std::map<std::pair<const void*, int>, int> max_dyn;
    static std::mutex max_dyn_mu;
    if (dev->device < 0 || dev->device >= kMaxDevices) throw RocpError{ROCP_E_CUDA, "device ordinal out of range"};
    std::lock_guard<std::mutex> lk(max_dyn_mu);
    int& md = max_dyn[std::make_pair(fn, dev->device)];
    if (md == 0) {
        int optin = 0;
        CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev->device));
        cudaFuncAttributes fa{};
        CK(cudaFuncGetAttributes(&fa, fn));
        CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - int(fa.sharedSizeBytes)));
        md = optin - int(fa.sharedSizeBytes);
    }
    if (smem > size_t(md)) throw_domain("batch too large for the persistent chain kernel's shared memory");
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kChainThreads, smem));
    if (per_sm < 1) throw RocpError{ROCP_E_CUDA, "chain kernel does not fit on an SM"};
    void* args[] = {const_cast<ChainParams*>(&p)};
    CK(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kChainThreads), args, smem, dev->stream));
    after_launch(dev, name);
}

// k_flow (flow_kernel.cuh) serves R <= 32 when at least 8 blocks are left without a chunk;
// k_chain otherwise (and when ROCP_CHAIN=barrier asks for the grid-barrier kernel).  The wide
// k_flow instances (R in 33..64, N <= 5) are bit-identical but slower on C4 than k_chain
// (95k vs 147k slices/s): ROCP_CHAIN=flow selects them.
bool use_flow(const rocp_stream* st, int grid) {
    static const int chain_env = [] {
        const char* e = std::getenv("ROCP_CHAIN");
        if (!e) return 0;
        if (std::string(e) == "barrier") return 1;
        if (std::string(e) == "flow") return 2;
        return 0;
    }();
    if (chain_env == 1 || st->R > 64 || (st->R > 32 && st->N > 5)) return false;
    if (st->R > 32 && chain_env != 2) return false;
    const int64_t nch = (st->s + kChunk - 1) / kChunk;
    return grid - 1 - nch >= 8;
}

// grid: one persistent block per SM, less the SMs of an overlapped gather
void launch_chain_k(rocp_stream* st, const ChainParams& p, int grid, bool flow) {
    const bool wide = p.R > 32, trace = p.trace != nullptr;
    if (flow) {
        const int rp = ((p.R + kCRB - 1) / kCRB) * kCRB;
        const void* fn = nullptr;
#define ROCP_FLOW_FN(RPV) (trace ? reinterpret_cast<const void*>(k_flow<RPV, true>) : reinterpret_cast<const void*>(k_flow<RPV, false>))
        switch (rp) {
            case 8: fn = ROCP_FLOW_FN(8); break;
            case 16: fn = ROCP_FLOW_FN(16); break;
            case 24: fn = ROCP_FLOW_FN(24); break;
            case 32: fn = ROCP_FLOW_FN(32); break;
            case 40: fn = ROCP_FLOW_FN(40); break;
            case 48: fn = ROCP_FLOW_FN(48); break;
            case 56: fn = ROCP_FLOW_FN(56); break;
            default: fn = ROCP_FLOW_FN(64); break;
        }
#undef ROCP_FLOW_FN
        launch_coop(st, fn, "k_flow", p, grid);
    } else if (wide) {
        if (trace) launch_coop(st, reinterpret_cast<const void*>(k_chain<true, true>), "k_chain", p, grid);
        else launch_coop(st, reinterpret_cast<const void*>(k_chain<true, false>), "k_chain", p, grid);
    } else {
        if (trace) launch_coop(st, reinterpret_cast<const void*>(k_chain<false, true>), "k_chain", p, grid);
        else launch_coop(st, reinterpret_cast<const void*>(k_chain<false, false>), "k_chain", p, grid);
    }
}

// The whole factor-dependent chain of the prepared window as ONE cooperative
// persistent kernel (kernels.cuh K6).
// overlap: the window's gather is still running (enqueue_draw_gather(..., true)).
void launch_chain(rocp_stream* st, int64_t nb, int64_t B, int64_t b0 = 0, bool overlap = false) {
    ChainParams p{};
    p.N = st->N;
    p.R = st->R;
    p.S = int(st->s);
    p.nb = int(nb);
    p.B = int(B);
    p.nsuper = int((st->s + kSuperSamples - 1) / kSuperSamples);
    p.resid_level = st->resid_level;
    for (int n = 1; n < st->N; ++n) {
        p.head[n - 1] = int32_t(st->head[size_t(n - 1)]);
        p.U[n - 1] = st->U[size_t(n - 1)].p;
        p.P[n - 1] = st->P[size_t(n - 1)].p;
        p.Q[n - 1] = st->Q[size_t(n - 1)].p;
    }
    p.temporal = st->temporal.p;
    p.t_len0 = st->t_len;
    const int64_t RPw = ((st->R + kCRB - 1) / kCRB) * kCRB;
    p.idx_base = st->win.idx.p + b0 * st->N * st->s * (st->N - 1);
    p.X_base = st->win.X.p;
    p.xoff = st->win.xoff_dev.p + b0 * st->N;
    p.gch = st->zmodes.p;
    p.gpart = st->gpart.p;
    p.chpart = st->chpart.p;
    p.cpart = st->dev->contract_partial.p;
    p.LD = st->LD.p;
    p.mode_flag = st->mode_flag.p;
    p.flags = st->flags.p;
    p.resid = st->resid.p;
    p.rpart = st->rpart.p;
    p.counter = st->dev->counters.p + 4;
    // phase-0 chunk arrivals (total, per superchunk), cumulative over the launch's stages
    // (+ [1 + nsuper]: superchunk Gram pre-sums published, k_chain without the one-block combine)
    // (+ [2 + nsuper + m]: Z rows of superchunk m's chunks published, ahead of their Gram partials)
    if (st->zctr.n < size_t(2 * p.nsuper + 2)) st->zctr.alloc(size_t(2 * p.nsuper + 2));
    CK(cudaMemsetAsync(st->zctr.p, 0, size_t(2 * p.nsuper + 2) * sizeof(unsigned), st->dev->stream));
    p.zctr = st->zctr.p;
    int grid = st->dev->num_sms;
    if (overlap) {
        if (b0 != 0) throw RocpError{ROCP_E_STATE, "overlapped gather needs the whole window (internal)"};
        p.gdone = st->win.jobs.done.p;
        p.gneed = st->win.jobs.need.p;
        grid -= st->win_gsms;
    }
    // several independent streams sharing the GPU (one handle each): each chain takes its share of
    // the SMs, so the chains of different handles are co-resident (rocp_set_chain_sms)
    if (st->dev->chain_sms > 0) grid = std::max(1, std::min(grid, st->dev->chain_sms));
    const bool flow = use_flow(st, grid);
    // streamed wide items (chain_stream_items): one superchunk per block, X_s through the arena's
    // tensor map, Z rows padded by 4 doubles
    const bool streamed = !flow && st->R > 32 && st->win.xmap_ok && grid - 1 >= p.nsuper;
    p.xmap = streamed ? st->win.xmap.p : nullptr;
    p.zstride = int(streamed ? RPw + 4 : RPw);
    p.zbuf = st->win.zT.p + b0 * st->s * p.zstride;
    if (flow) {
        int maxtiles = int((B + kRowTile - 1) / kRowTile);
        for (int64_t I : st->head) maxtiles = std::max(maxtiles, int((I + kRowTile - 1) / kRowTile));
        const size_t nctr = size_t(1 + 2 * st->N + st->N * maxtiles + 1);
        st->fctr.ensure(nctr);
        st->ginv.ensure(size_t(2 * kGinvSlot));
        st->gmode.ensure(2);
        st->wtemp.ensure(size_t(B * st->R));
        CK(cudaMemsetAsync(st->fctr.p, 0, nctr * sizeof(unsigned), st->dev->stream));
        p.ginv = st->ginv.p;
        p.gmode = st->gmode.p;
        p.wtemp = st->wtemp.p;
        p.fctr = st->fctr.p;
        p.maxtiles = maxtiles;
    }
    if (st->trace_on) {
        st->trace.ensure(size_t(nb * st->N * kTraceSlots));
        CK(cudaMemsetAsync(st->trace.p, 0, size_t(nb * st->N * kTraceSlots) * 8, st->dev->stream));
        st->trace_n = nb * st->N * kTraceSlots;
        p.trace = st->trace.p;
    } else {
        p.trace = nullptr;
    }
    if (st->time_gather) {  // kernel timing: events around the persistent chain too
        if (st->chain_events_used == st->chain_events.size()) {
            cudaEvent_t a, e;
            CK(cudaEventCreate(&a));
            CK(cudaEventCreate(&e));
            st->chain_events.emplace_back(a, e);
        }
        auto& ev = st->chain_events[st->chain_events_used++];
        CK(cudaEventRecord(ev.first, st->dev->stream));
        launch_chain_k(st, p, grid, flow);
        CK(cudaEventRecord(ev.second, st->dev->stream));
    } else {
        launch_chain_k(st, p, grid, flow);
    }
    if (overlap) CK(cudaStreamWaitEvent(st->dev->stream, st->dev->ev_gdone, 0));  // join the gather stream
    if (st->resid_level >= 1) {  // sampled residual of every batch's temporal solve (off the chain)
        WinResidParams w{};
        w.N = st->N;
        w.R = st->R;
        w.S = int(st->s);
        w.B = int(B);
        w.RP = p.zstride;  // row stride of the temporal Z
        w.nb = int(nb);
        w.temporal = st->temporal.p;
        w.t_len0 = st->t_len;
        w.X_base = st->win.X.p;
        w.xoff = st->win.xoff_dev.p + b0 * st->N;
        w.zT = p.zbuf;
        w.cols = st->win.rcols.p;
        w.out = st->win.rhist.p;
        w.last_out = st->resid.p;
        if (st->win.rctr.n < size_t(nb)) {  // zero once; last_arrive_of resets each counter after use
            CK(cudaStreamSynchronize(st->dev->stream));
            st->win.rctr.alloc(size_t(std::max<int64_t>(nb, st->win.nb)));
            CK(cudaMemset(st->win.rctr.p, 0, st->win.rctr.n * sizeof(unsigned)));
        }
        w.rctr = st->win.rctr.p;
        const size_t zbytes = size_t(8) * size_t(st->R) * sizeof(double);
        const size_t ubytes = size_t(B) * size_t(st->R) * sizeof(double);
        w.stage_u = zbytes + ubytes <= 48 * 1024 ? 1 : 0;
        const dim3 g1{unsigned((st->s + 7) / 8), unsigned(nb), 1u};
        k_win_resid<<<g1, 256, zbytes + (w.stage_u ? ubytes : 0), st->dev->stream>>>(w);
        after_launch(st->dev, "k_win_resid");
    }
}

// The temporal factor grows geometrically, as RocpStream::consume does
// (rocp.cpp:152-155: capacity max(2 x rows, t_len + batch)): a new buffer, the
// t_len used rows copied on the device, the old one released after the stream
// drains.  Captured graphs hold the old pointer and are dropped.
void grow_temporal(rocp_stream* st, int64_t need) {
    if (need <= st->t_cap) return;
    rocp_dev* dev = st->dev;
    const int64_t cap = std::max<int64_t>(2 * st->t_cap, need);
    DBuf<double> grown(size_t(cap * st->R));
    CK(cudaMemsetAsync(grown.p, 0, size_t(cap * st->R) * sizeof(double), dev->stream));
    if (st->t_len > 0)
        CK(cudaMemcpyAsync(grown.p, st->temporal.p, size_t(st->t_len * st->R) * sizeof(double),
                           cudaMemcpyDeviceToDevice, dev->stream));
    CK(cudaStreamSynchronize(dev->stream));  // queued chains may still read or write the old rows
    if (st->copy_stream) CK(cudaStreamSynchronize(st->copy_stream));
    st->temporal = std::move(grown);
    st->t_cap = cap;
    clear_graphs(st);
}

void check_capacity(rocp_stream* st, int64_t add) { grow_temporal(st, st->t_len + add); }

// One batch on a device slab (no graph).
void consume_one(rocp_stream* st, const double* x, int64_t B, uint64_t seed, uint32_t batch_id) {
    check_capacity(st, B);
    const int64_t slice = prod(st->head);
    st->win_gsms = st->resid_level <= 1 ? gather_sms(st, B) : 0;
    const bool overlap = st->win_gsms > 0;
    prepare_window(st, x, 0, slice, B, 1, nullptr, nullptr, -1, false, nullptr, !overlap);
    enqueue_draw_gather(st, seed, batch_id, overlap);
    if (st->resid_level <= 1) launch_chain(st, 1, B, 0, overlap);
    else enqueue_chain(st, 1, B);
    st->t_len += B;  // rocp.cpp:159
}

#include "host_slab.inc"

#include "shard_host.inc"

}  // namespace

// ===========================================================================
extern "C" {

static rocp_status create_dev(int device, int world, int rank, const void* nccl_id, bool emulated, rocp_dev** out);

rocp_status rocp_create(int device, int world, int rank, const void* nccl_id, rocp_dev** out) {
    return create_dev(device, world, rank, nccl_id, false, out);
}

rocp_status rocp_create_emulated_rank(int device, int world, int rank, rocp_dev** out) {
    return create_dev(device, world, rank, nullptr, true, out);
}

rocp_status rocp_emulated_group_consume_range(rocp_stream* const* ranks, int world, const rocp_tensor* const* x_local,
                                              int64_t t0, int64_t batch, int64_t nb, uint64_t seed,
                                              uint32_t first_batch_id) {
    if (!ranks || world < 1 || !ranks[0]) return ROCP_E_DOMAIN;
    return guarded(ranks[0]->dev, [&] {
        emulated_group_consume(ranks, world, x_local, t0, batch, nb, seed, first_batch_id);
    });
}

static rocp_status create_dev(int device, int world, int rank, const void* nccl_id, bool emulated, rocp_dev** out) {
    auto dev = std::make_unique<rocp_dev>();
    rocp_status st = guarded(dev.get(), [&] {
        if (world < 1 || rank < 0 || rank >= world) throw_domain("need 0 <= rank < world");
        if (world > 1 && !nccl_id && !emulated) throw_domain("world > 1 needs the NCCL unique id of rank 0");
        dev->emulated = emulated;
        CK(cudaSetDevice(device));
        dev->device = device;
        {
            std::lock_guard<std::mutex> lk(g_handles_mu);
            ++g_handles[device];
            dev->counted = true;
        }
        dev->world = world;
        dev->rank = rank;
        CK(cudaStreamCreateWithFlags(&dev->stream, cudaStreamNonBlocking));
        CK(cudaDeviceGetAttribute(&dev->num_sms, cudaDevAttrMultiProcessorCount, device));
        dev->counters.alloc(16);
        CK(cudaMemset(dev->counters.p, 0, 16 * sizeof(unsigned int)));
        dev->gram_counters.alloc(64);
        CK(cudaMemset(dev->gram_counters.p, 0, 64 * sizeof(unsigned int)));
        dev->flags.alloc(4);
        CK(cudaMemset(dev->flags.p, 0, 4 * sizeof(int)));
        dev->scalars.alloc(16);
        {
            const int fs = int((size_t(kGroup) * 64 + kGroup) * sizeof(double));
            CK(cudaFuncSetAttribute(k_fitness<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, fs));
            CK(cudaFuncSetAttribute(k_fitness<13>, cudaFuncAttributeMaxDynamicSharedMemorySize, fs));
            CK(cudaFuncSetAttribute(k_fitness<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, fs));
        }
        set_contract_smem_attrs();
        if (world > 1 && !emulated) {
            const NcclApi& api = require_nccl();
            ncclUniqueId id;
            std::memcpy(&id, nccl_id, sizeof(id));
            NK(api.comm_init_rank(&dev->comm, world, id, rank), "ncclCommInitRank");
        }
    });
    if (st != ROCP_OK) {
        static thread_local std::string last;
        last = dev->err;
        if (dev->counted) {
            std::lock_guard<std::mutex> lk(g_handles_mu);
            if (--g_handles[dev->device] <= 0) g_handles.erase(dev->device);
        }
        *out = nullptr;
        return st;
    }
    *out = dev.release();
    return ROCP_OK;
}

void rocp_destroy(rocp_dev* dev) {
    if (!dev) return;
    if (dev->counted) {
        std::lock_guard<std::mutex> lk(g_handles_mu);
        if (--g_handles[dev->device] <= 0) g_handles.erase(dev->device);
    }
    cudaSetDevice(dev->device);
    cudaStreamSynchronize(dev->stream);
    dev->init = rocp_dev::Init{};
    for (cudaEvent_t& e : dev->timer)
        if (e) cudaEventDestroy(e);
    if (dev->comm) nccl_api().comm_destroy(dev->comm);
    if (dev->gstream) {
        cudaStreamSynchronize(dev->gstream);
        cudaStreamDestroy(dev->gstream);
        cudaEventDestroy(dev->ev_gready);
        cudaEventDestroy(dev->ev_gdone);
    }
    cudaStreamDestroy(dev->stream);
    delete dev;
}

const char* rocp_last_error(const rocp_dev* dev) { return dev ? dev->err.c_str() : "null handle"; }

rocp_status rocp_probe_random_reads(rocp_dev* dev, const rocp_tensor* t, int64_t reads, uint64_t seed, float* ms) {
    return guarded(dev, [&] {
        if (reads < 1 || !t || t->numel < 1) throw_domain("probe: need reads and a non-empty tensor");
        DBuf<double> sink(1);
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        const int grid = dev->num_sms * 8;
        k_probe_random_reads<<<grid, 256, 0, dev->stream>>>(t->d, uint64_t(t->numel), reads, seed, sink.p);  // warm
        after_launch(dev, "k_probe_random_reads");
        CK(cudaEventRecord(e0, dev->stream));
        k_probe_random_reads<<<grid, 256, 0, dev->stream>>>(t->d, uint64_t(t->numel), reads, seed + 1, sink.p);
        after_launch(dev, "k_probe_random_reads");
        CK(cudaEventRecord(e1, dev->stream));
        CK(cudaEventSynchronize(e1));
        CK(cudaEventElapsedTime(ms, e0, e1));
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
    });
}

rocp_status rocp_decision_stats(rocp_dev* dev, uint64_t* counts, int reset) {
    return guarded(dev, [&] {
        CK(cudaStreamSynchronize(dev->stream));
        unsigned long long h[4];
        CK(cudaMemcpyFromSymbol(h, g_dec_paths, sizeof(h)));
        for (int k = 0; k < 4; ++k) counts[k] = h[k];
        if (reset) {
            const unsigned long long z[4] = {0, 0, 0, 0};
            CK(cudaMemcpyToSymbol(g_dec_paths, z, sizeof(z)));
        }
    });
}

rocp_status rocp_set_gather_sms(rocp_dev* dev, int sms) {
    return guarded(dev, [&] {
        if (sms > dev->num_sms / 2) throw_domain("gather SMs: at most half the device");
        CK(cudaStreamSynchronize(dev->stream));
        dev->gather_sms = sms < 0 ? -2 : sms;
    });
}

rocp_status rocp_set_chain_sms(rocp_dev* dev, int sms) {
    return guarded(dev, [&] {
        if (sms < 0 || sms > dev->num_sms) throw_domain("chain SMs: 0 (every SM) .. the device's SM count");
        if (sms != 0 && sms < 16) throw_domain("chain SMs: at least 16");
        CK(cudaStreamSynchronize(dev->stream));
        dev->chain_sms = sms;
    });
}

rocp_status rocp_sm_count(rocp_dev* dev, int* sms) {
    return guarded(dev, [&] {
        if (!sms) throw_domain("null output");
        *sms = dev->num_sms;
    });
}

rocp_status rocp_timer_record(rocp_dev* dev, int slot) {
    return guarded(dev, [&] {
        if (slot < 0 || slot >= 8) throw_domain("timer slot out of range");
        if (!dev->timer[slot]) CK(cudaEventCreate(&dev->timer[slot]));
        CK(cudaEventRecord(dev->timer[slot], dev->stream));
    });
}

rocp_status rocp_timer_elapsed_ms(rocp_dev* dev, int a, int b, float* ms) {
    return guarded(dev, [&] {
        if (a < 0 || a >= 8 || b < 0 || b >= 8 || !dev->timer[a] || !dev->timer[b])
            throw_domain("timer slot not recorded");
        CK(cudaEventSynchronize(dev->timer[b]));
        CK(cudaEventElapsedTime(ms, dev->timer[a], dev->timer[b]));
    });
}

void* rocp_cuda_stream(rocp_dev* dev) { return dev ? static_cast<void*>(dev->stream) : nullptr; }

void* rocp_host_alloc(size_t bytes) { return host_alloc_huge(bytes); }

void rocp_host_free(void* p, size_t bytes) { host_free_huge(p, bytes); }

rocp_status rocp_synchronize(rocp_dev* dev) {
    return guarded(dev, [&] { CK(cudaStreamSynchronize(dev->stream)); });
}

uint64_t rocp_kernel_launches(const rocp_dev* dev) { return dev ? dev->launches : 0; }

int rocp_nccl_id_size(void) { return int(sizeof(ncclUniqueId)); }

rocp_status rocp_nccl_get_unique_id(void* out) {
    const NcclApi& api = nccl_api();
    if (!api.ok || !out) return ROCP_E_NCCL;
    ncclUniqueId id;
    if (api.get_unique_id(&id) != ncclSuccess) return ROCP_E_NCCL;
    std::memcpy(out, &id, sizeof(id));
    return ROCP_OK;
}

// ---- tensors ---------------------------------------------------------------
rocp_status rocp_tensor_create(rocp_dev* dev, const int64_t* dims, int order, const double* host,
                               rocp_tensor** out) {
    return guarded(dev, [&] {
        std::vector<int64_t> d(dims, dims + order);
        check_tensor_dims(d);
        auto t = std::make_unique<rocp_tensor>();
        t->dims = d;
        t->numel = prod(d);
        t->owned = true;
        CK(cudaMalloc(&t->d, size_t(t->numel) * sizeof(double)));
        if (host)
            CK(cudaMemcpyAsync(t->d, host, size_t(t->numel) * sizeof(double), cudaMemcpyHostToDevice, dev->stream));
        else
            CK(cudaMemsetAsync(t->d, 0, size_t(t->numel) * sizeof(double), dev->stream));
        CK(cudaStreamSynchronize(dev->stream));
        *out = t.release();
    });
}

rocp_status rocp_tensor_slab(rocp_dev* dev, const rocp_tensor* t, int64_t t0, int64_t len,
                             rocp_tensor** out) {
    return guarded(dev, [&] {
        const int64_t T = t->dims.back();
        if (t0 < 0 || len < 1 || t0 + len > T) throw_domain("slab out of range");
        auto v = std::make_unique<rocp_tensor>();
        v->dims = t->dims;
        v->dims.back() = len;
        v->numel = prod(v->dims);
        const int64_t slice = t->numel / T;
        v->d = t->d + t0 * slice;
        v->owned = false;
        *out = v.release();
    });
}

rocp_status rocp_tensor_rows(rocp_dev* dev, const rocp_tensor* t, int64_t r0, int64_t r1, rocp_tensor** out) {
    return guarded(dev, [&] {
        const int64_t I1 = t->dims[0];
        if (r0 < 0 || r1 <= r0 || r1 > I1) throw_domain("row range out of bounds");
        auto v = std::make_unique<rocp_tensor>();
        v->dims = t->dims;
        v->dims[0] = r1 - r0;
        v->numel = prod(v->dims);
        CK(cudaMalloc(&v->d, size_t(v->numel) * sizeof(double)));
        v->owned = true;
        CK(cudaMemcpy2DAsync(v->d, size_t(r1 - r0) * 8, t->d + r0, size_t(I1) * 8, size_t(r1 - r0) * 8,
                             size_t(t->numel / I1), cudaMemcpyDeviceToDevice, dev->stream));
        CK(cudaStreamSynchronize(dev->stream));
        *out = v.release();
    });
}

void rocp_tensor_free(rocp_tensor* t) { delete t; }

rocp_status rocp_tensor_upload(rocp_dev* dev, rocp_tensor* t, const double* host) {
    return guarded(dev, [&] {
        CK(cudaMemcpyAsync(t->d, host, size_t(t->numel) * sizeof(double), cudaMemcpyHostToDevice, dev->stream));
        CK(cudaStreamSynchronize(dev->stream));
    });
}

rocp_status rocp_tensor_download(rocp_dev* dev, const rocp_tensor* t, double* host) {
    return guarded(dev, [&] {
        CK(cudaMemcpyAsync(host, t->d, size_t(t->numel) * sizeof(double), cudaMemcpyDeviceToHost, dev->stream));
        CK(cudaStreamSynchronize(dev->stream));
    });
}

double* rocp_tensor_device_ptr(rocp_tensor* t) { return t ? t->d : nullptr; }
int64_t rocp_tensor_numel(const rocp_tensor* t) { return t ? t->numel : 0; }

rocp_status rocp_generate_synthetic(rocp_dev* dev, rocp_tensor* t, const double* const* factors,
                                    int rank, int has_noise, double snr_db, uint64_t noise_seed) {
    return guarded(dev, [&] {
        check_rank(rank);
        const int N = int(t->dims.size());
        std::vector<DBuf<double>> U;
        SynJob j{};
        for (int n = 0; n < N; ++n) {
            U.emplace_back(size_t(t->dims[size_t(n)] * rank));
            upload_rowmajor(dev, factors[n], t->dims[size_t(n)], rank, U.back().p);
            j.U[n] = U.back().p;
            j.dims[n] = t->dims[size_t(n)];
        }
        j.t = t->d;
        j.numel = t->numel;
        j.I1 = t->dims[0];
        j.N = N;
        j.R = rank;
        j.seed = noise_seed;
        const int grid = dev->num_sms * 8;  // fixed: deterministic partial layout
        DBuf<double> ps(static_cast<size_t>(grid)), pn(static_cast<size_t>(grid));
        j.part_sig = ps.p;
        j.part_noise = has_noise ? pn.p : nullptr;
        k_synth_signal<<<grid, 256, 0, dev->stream>>>(j);
        after_launch(dev, "k_synth_signal");
        if (has_noise) {
            std::vector<double> hs(static_cast<size_t>(grid)), hn(static_cast<size_t>(grid));
            CK(cudaMemcpyAsync(hs.data(), ps.p, hs.size() * 8, cudaMemcpyDeviceToHost, dev->stream));
            CK(cudaMemcpyAsync(hn.data(), pn.p, hn.size() * 8, cudaMemcpyDeviceToHost, dev->stream));
            CK(cudaStreamSynchronize(dev->stream));
            double ss = 0.0, nn = 0.0;
            for (int b = 0; b < grid; ++b) { ss += hs[size_t(b)]; nn += hn[size_t(b)]; }
            // |noise|^2 = |signal|^2 * 10^(-snr/10), scaled after the draw (synthetic.cpp:26-27)
            const double scale = std::sqrt(ss) * std::pow(10.0, -snr_db / 20.0) / std::sqrt(nn);
            CK(cudaMemcpyAsync(dev->scalars.p + 15, &scale, 8, cudaMemcpyHostToDevice, dev->stream));
            k_synth_noise<<<grid, 256, 0, dev->stream>>>(t->d, t->numel, noise_seed, dev->scalars.p + 15);
            after_launch(dev, "k_synth_noise");
        }
        CK(cudaStreamSynchronize(dev->stream));
    });
}

// ---- primitives --------------------------------------------------------------
rocp_status rocp_draw_samples(rocp_dev* dev, const int64_t* dims, int order, int mode, int64_t s,
                              uint64_t seed, uint32_t batch, uint32_t iteration, int64_t* rows,
                              int64_t* decoded) {
    return guarded(dev, [&] {
        std::vector<int64_t> d(dims, dims + order);
        check_tensor_dims(d);
        if (mode < 1 || mode > order) throw_domain("mode out of range");
        if (s < 1) throw_domain("sample count must be positive");  // sampling.cpp:48-49
        DBuf<int64_t> drows(static_cast<size_t>(s)), dbase(static_cast<size_t>(s));
        DBuf<int32_t> didx(static_cast<size_t>(s) * (order - 1));
        upload_jobs(dev, dev->jobs, {make_draw(d, mode, s, seed, batch, iteration, nullptr, drows.p, didx.p, dbase.p)}, {});
        launch_draw(dev, dev->jobs);
        CK(cudaMemcpyAsync(rows, drows.p, size_t(s) * 8, cudaMemcpyDeviceToHost, dev->stream));
        std::vector<int32_t> hidx(size_t(s) * (order - 1));
        CK(cudaMemcpyAsync(hidx.data(), didx.p, hidx.size() * 4, cudaMemcpyDeviceToHost, dev->stream));
        CK(cudaStreamSynchronize(dev->stream));
        if (decoded)
            for (size_t e = 0; e < hidx.size(); ++e) decoded[e] = int64_t(hidx[e]) + 1;
    });
}

rocp_status rocp_decode_rows(rocp_dev* dev, const int64_t* dims, int order, int mode,
                             const int64_t* rows, int64_t s, int64_t* decoded) {
    return guarded(dev, [&] {
        std::vector<int64_t> d(dims, dims + order);
        check_tensor_dims(d);
        if (mode < 1 || mode > order) throw_domain("mode out of range");
        int64_t co = 1;
        for (int k = 0; k < order; ++k)
            if (k + 1 != mode) co *= d[size_t(k)];
        for (int64_t c = 0; c < s; ++c)
            if (rows[c] < 1 || rows[c] > co) throw_domain("column index out of range");  // tensor.cpp:98-99
        DBuf<int64_t> din(static_cast<size_t>(s)), dbase(static_cast<size_t>(s));
        DBuf<int32_t> didx(static_cast<size_t>(s) * (order - 1));
        CK(cudaMemcpyAsync(din.p, rows, size_t(s) * 8, cudaMemcpyHostToDevice, dev->stream));
        upload_jobs(dev, dev->jobs, {make_draw(d, mode, s, 0, 0, 0, din.p, nullptr, didx.p, dbase.p)}, {});
        launch_draw(dev, dev->jobs);
        std::vector<int32_t> hidx(size_t(s) * (order - 1));
        CK(cudaMemcpyAsync(hidx.data(), didx.p, hidx.size() * 4, cudaMemcpyDeviceToHost, dev->stream));
        CK(cudaStreamSynchronize(dev->stream));
        for (size_t e = 0; e < hidx.size(); ++e) decoded[e] = int64_t(hidx[e]) + 1;
    });
}

rocp_status rocp_sample_unfolding(rocp_dev* dev, const rocp_tensor* t, int mode,
                                  const int64_t* rows, int64_t s, double* out) {
    return guarded(dev, [&] {
        const std::vector<int64_t>& d = t->dims;
        const int order = int(d.size());
        if (mode < 1 || mode > order) throw_domain("mode out of range");
        if (s < 1) throw_domain("sample count must be positive");
        int64_t co = 1;
        for (int k = 0; k < order; ++k)
            if (k + 1 != mode) co *= d[size_t(k)];
        for (int64_t c = 0; c < s; ++c)
            if (rows[c] < 1 || rows[c] > co)
                throw_domain("sample_unfolding: index set drawn against different dims");
        const int64_t I = d[size_t(mode - 1)];
        DBuf<int64_t> din(static_cast<size_t>(s)), dbase(static_cast<size_t>(s));
        DBuf<int32_t> didx(static_cast<size_t>(s) * (order - 1));
        DBuf<double> dout(static_cast<size_t>(I * s));
        CK(cudaMemcpyAsync(din.p, rows, size_t(s) * 8, cudaMemcpyHostToDevice, dev->stream));
        upload_jobs(dev, dev->jobs, {make_draw(d, mode, s, 0, 0, 0, din.p, nullptr, didx.p, dbase.p)},
                    {make_gather(t->d, d, mode, s, dbase.p, dout.p)});
        launch_draw(dev, dev->jobs);
        launch_gather(dev, dev->jobs);
        CK(cudaMemcpyAsync(out, dout.p, size_t(I * s) * 8, cudaMemcpyDeviceToHost, dev->stream));
        CK(cudaStreamSynchronize(dev->stream));
    });
}

rocp_status rocp_sampled_khatri_rao(rocp_dev* dev, const int64_t* decoded, int64_t s, int n_other,
                                    const double* const* factors, const int64_t* factor_rows,
                                    int rank, double* z) {
    return guarded(dev, [&] {
        check_rank(rank);
        if (n_other < 1 || n_other >= kMaxOrder) throw_domain("sampled_khatri_rao: factor count mismatch");
        for (int64_t c = 0; c < s; ++c)
            for (int k = 0; k < n_other; ++k) {
                const int64_t i = decoded[c * n_other + k];
                const int l = n_other - 1 - k;
                if (i < 1 || i > factor_rows[l])
                    throw_domain("sampled_khatri_rao: decoded index exceeds factor rows");  // sampling.cpp:99-100
            }
        std::vector<int32_t> hidx(size_t(s) * n_other);
        for (size_t e = 0; e < hidx.size(); ++e) hidx[e] = int32_t(decoded[e] - 1);
        DBuf<int32_t> didx(hidx.size());
        CK(cudaMemcpyAsync(didx.p, hidx.data(), hidx.size() * 4, cudaMemcpyHostToDevice, dev->stream));
        std::vector<DBuf<double>> F;
        SkrJob j{};
        for (int l = 0; l < n_other; ++l) {
            F.emplace_back(size_t(factor_rows[l] * rank));
            upload_rowmajor(dev, factors[l], factor_rows[l], rank, F.back().p);
            j.f[l] = F.back().p;
        }
        DBuf<double> dz(static_cast<size_t>(s * rank));
        j.idx = didx.p;
        j.n_other = n_other;
        j.s = int32_t(s);
        j.R = rank;
        j.z = dz.p;
        launch_skr(dev, j);
        download_colmajor(dev, dz.p, s, rank, z);
    });
}

rocp_status rocp_gram(rocp_dev* dev, const double* z, int64_t s, int rank, double* g) {
    return guarded(dev, [&] {
        check_rank(rank);
        DBuf<double> dz(static_cast<size_t>(s * rank)), dg(static_cast<size_t>(rank * rank));
        upload_rowmajor(dev, z, s, rank, dz.p);
        launch_gram(dev, dz.p, s, rank, nullptr, dg.p);
        CK(cudaMemcpyAsync(g, dg.p, size_t(rank * rank) * 8, cudaMemcpyDeviceToHost, dev->stream));
        CK(cudaStreamSynchronize(dev->stream));
    });
}

rocp_status rocp_contract(rocp_dev* dev, const double* x, int64_t rows, int64_t s, const double* z,
                          int rank, double* out) {
    return guarded(dev, [&] {
        check_rank(rank);
        DBuf<double> dx(static_cast<size_t>(rows * s)), dz(static_cast<size_t>(s * rank)), dout(static_cast<size_t>(rows * rank));
        CK(cudaMemcpyAsync(dx.p, x, size_t(rows * s) * 8, cudaMemcpyHostToDevice, dev->stream));
        upload_rowmajor(dev, z, s, rank, dz.p);
        reserve_contract(dev, rows, s, rank);
        launch_contract(dev, dx.p, rows, s, dz.p, rank, nullptr, dout.p);
        download_colmajor(dev, dout.p, rows, rank, out);
    });
}

rocp_status rocp_solve_gram(rocp_dev* dev, const double* gram, const double* rhs, int64_t rows,
                            int rank, double* out, int* regularized) {
    return guarded(dev, [&] {
        check_rank(rank);
        DBuf<double> dg(static_cast<size_t>(rank * rank)), drhs(static_cast<size_t>(std::max<int64_t>(rows, 1) * rank)),
            dout(size_t(std::max<int64_t>(rows, 1) * rank));
        CK(cudaMemcpyAsync(dg.p, gram, size_t(rank * rank) * 8, cudaMemcpyHostToDevice, dev->stream));
        if (rows > 0) upload_rowmajor(dev, rhs, rows, rank, drhs.p);
        CK(cudaMemsetAsync(dev->flags.p, 0, 2 * sizeof(int), dev->stream));
        launch_solve(dev, dg.p, rank, drhs.p, rows, dout.p, dev->flags.p, 1);
        int hf[2];
        CK(cudaMemcpyAsync(hf, dev->flags.p, sizeof(hf), cudaMemcpyDeviceToHost, dev->stream));
        if (rows > 0) download_colmajor(dev, dout.p, rows, rank, out);
        CK(cudaStreamSynchronize(dev->stream));
        if (regularized) *regularized = hf[0] & 1;
    });
}

rocp_status rocp_solve_sampled_ls(rocp_dev* dev, const double* z, const double* x, int64_t s,
                                  int64_t rows, int rank, double* out, int* regularized,
                                  int* underdetermined) {
    return guarded(dev, [&] {
        check_rank(rank);
        if (underdetermined) *underdetermined = (s < rank) ? 1 : 0;  // solve.cpp:40
        DBuf<double> dz(static_cast<size_t>(s * rank)), dx(static_cast<size_t>(rows * s)), dg(static_cast<size_t>(rank * rank)),
            drhs(size_t(rows * rank)), dout(size_t(rows * rank));
        upload_rowmajor(dev, z, s, rank, dz.p);
        CK(cudaMemcpyAsync(dx.p, x, size_t(rows * s) * 8, cudaMemcpyHostToDevice, dev->stream));
        launch_gram(dev, dz.p, s, rank, nullptr, dg.p);
        reserve_contract(dev, rows, s, rank);
        launch_contract(dev, dx.p, rows, s, dz.p, rank, nullptr, drhs.p);
        CK(cudaMemsetAsync(dev->flags.p, 0, 2 * sizeof(int), dev->stream));
        launch_solve(dev, dg.p, rank, drhs.p, rows, dout.p, dev->flags.p, 1);
        int hf[2];
        CK(cudaMemcpyAsync(hf, dev->flags.p, sizeof(hf), cudaMemcpyDeviceToHost, dev->stream));
        download_colmajor(dev, dout.p, rows, rank, out);
        if (regularized) *regularized = hf[0] & 1;
    });
}

rocp_status rocp_model_fitness(rocp_dev* dev, const rocp_tensor* t, const double* const* factors,
                               int rank, double* fit) {
    return guarded(dev, [&] {
        check_rank(rank);
        const int N = int(t->dims.size());
        std::vector<DBuf<double>> U;
        std::vector<const double*> ptrs;
        for (int n = 0; n < N; ++n) {
            U.emplace_back(size_t(t->dims[size_t(n)] * rank));
            upload_rowmajor(dev, factors[n], t->dims[size_t(n)], rank, U.back().p);
            ptrs.push_back(U.back().p);
        }
        launch_fitness(dev, t, nullptr, rank, 0);
        launch_fitness(dev, t, &ptrs, rank, 1);
        double h[2];
        CK(cudaMemcpyAsync(h, dev->scalars.p, sizeof(h), cudaMemcpyDeviceToHost, dev->stream));
        CK(cudaStreamSynchronize(dev->stream));
        if (h[0] == 0.0) throw_domain("fitness undefined for zero-norm reference tensor");  // kruskal.cpp:75-76
        *fit = 1.0 - std::sqrt(h[1]) / std::sqrt(h[0]);                                 // kruskal.cpp:84
    });
}

// ---- cprand (cprand.cpp:12-69) ------------------------------------------------
rocp_status rocp_cprand(rocp_dev* dev, const rocp_tensor* t, int rank, int64_t samples, double tol,
                        int max_iters, uint64_t seed, double* const* factors,
                        double* const* best_kr, double* best_fitness, int* iterations,
                        int* regularized, int* err_sweep, double* fit_trace) {
    return guarded(
        dev,
        [&] {
            if (rank < 1) throw_domain("cprand_decompose: rank must be positive");  // cprand.cpp:14-15
            check_rank(rank);
            if (max_iters < 1) throw_domain("cprand_decompose: need at least one sweep");  // :16-17
            const std::vector<int64_t>& d = t->dims;
            const int N = int(d.size());
            launch_fitness(dev, t, nullptr, rank, 0);
            double nsq = 0.0;
            CK(cudaMemcpyAsync(&nsq, dev->scalars.p, 8, cudaMemcpyDeviceToHost, dev->stream));
            CK(cudaStreamSynchronize(dev->stream));
            if (nsq == 0.0) throw_domain("cprand_decompose: zero tensor");  // :18-19
            const int64_t s = samples > 0 ? samples : auto_sample_count(rank);  // :23
            const std::vector<int64_t> strides = strides_of(d);

            std::vector<DBuf<double>> U, best;
            std::vector<const double*> uptr;
            std::vector<DBuf<int32_t>> idx;
            std::vector<DBuf<int64_t>> base;
            std::vector<DBuf<double>> X, Z, G, RHS;
            for (int n = 0; n < N; ++n) {
                const int64_t In = d[size_t(n)];
                U.emplace_back(size_t(In * rank));
                upload_rowmajor(dev, factors[n], In, rank, U.back().p);  // model = random_model(...) (:25)
                best.emplace_back(size_t(In * rank));
                uptr.push_back(U.back().p);
                idx.emplace_back(size_t(s) * (N - 1));
                base.emplace_back(size_t(s));
                X.emplace_back(size_t(In * s));
                Z.emplace_back(size_t(s * rank));
                G.emplace_back(size_t(rank * rank));
                RHS.emplace_back(size_t(In * rank));
            }
            for (int n = 0; n < N; ++n) reserve_contract(dev, d[size_t(n)], s, rank);
            double best_fit = -std::numeric_limits<double>::infinity();
            double prev = best_fit;
            bool reg_any = false;
            int sweep = 0;
            CK(cudaMemsetAsync(dev->flags.p, 0, 2 * sizeof(int), dev->stream));
            while (sweep < max_iters) {  // :32
                ++sweep;
                // All N draws and gathers of the sweep up front: indices never depend on factors.
                std::vector<DrawJob> dj;
                std::vector<GatherJob> gj;
                for (int n = 1; n <= N; ++n) {
                    dj.push_back(make_draw(d, n, s, seed, 0u, uint32_t(sweep), nullptr, nullptr,
                                           idx[size_t(n - 1)].p, base[size_t(n - 1)].p));
                    gj.push_back(make_gather(t->d, d, n, s, base[size_t(n - 1)].p, X[size_t(n - 1)].p));
                }
                upload_jobs(dev, dev->jobs, dj, gj);
                launch_draw(dev, dev->jobs);
                launch_gather(dev, dev->jobs);
                for (int n = 1; n <= N; ++n) {  // :35-45
                    SkrJob sj{};
                    sj.idx = idx[size_t(n - 1)].p;
                    sj.n_other = N - 1;
                    sj.s = int32_t(s);
                    sj.R = rank;
                    int l = 0;
                    for (int k = N; k >= 1; --k)
                        if (k != n) sj.f[l++] = U[size_t(k - 1)].p;  // factors_excluding (kruskal.cpp:44-53)
                    sj.z = Z[size_t(n - 1)].p;
                    launch_skr(dev, sj);
                    launch_gram(dev, sj.z, s, rank, nullptr, G[size_t(n - 1)].p);
                    launch_contract(dev, X[size_t(n - 1)].p, d[size_t(n - 1)], s, sj.z, rank, nullptr,
                                    RHS[size_t(n - 1)].p);
                    launch_solve(dev, G[size_t(n - 1)].p, rank, RHS[size_t(n - 1)].p, d[size_t(n - 1)],
                                 U[size_t(n - 1)].p, dev->flags.p, sweep);
                }
                launch_fitness(dev, t, &uptr, rank, 1);  // :47
                double rsq = 0.0;
                int hf[2];
                CK(cudaMemcpyAsync(&rsq, dev->scalars.p + 1, 8, cudaMemcpyDeviceToHost, dev->stream));
                CK(cudaMemcpyAsync(hf, dev->flags.p, sizeof(hf), cudaMemcpyDeviceToHost, dev->stream));
                CK(cudaStreamSynchronize(dev->stream));
                reg_any = reg_any || (hf[0] & 1);
                if (hf[1] != 0) {  // :42-43
                    RocpError e{ROCP_E_NUMERICAL,
                                "cprand_decompose: non-finite factor update (sweep " + std::to_string(hf[1]) + ")"};
                    e.sweep = hf[1];
                    throw e;
                }
                const double fit = 1.0 - std::sqrt(rsq) / std::sqrt(nsq);
                if (fit_trace) fit_trace[sweep - 1] = fit;
                if (!std::isfinite(fit)) {  // :48-49
                    RocpError e{ROCP_E_NUMERICAL,
                                "cprand_decompose: non-finite fitness (sweep " + std::to_string(sweep) + ")"};
                    e.sweep = sweep;
                    throw e;
                }
                if (fit > best_fit) {  // :50-53
                    best_fit = fit;
                    for (int n = 0; n < N; ++n)
                        CK(cudaMemcpyAsync(best[size_t(n)].p, U[size_t(n)].p, U[size_t(n)].n * 8,
                                           cudaMemcpyDeviceToDevice, dev->stream));
                }
                if (std::fabs(fit - prev) < tol) break;  // :54
                prev = fit;
            }
            // Z_best rebuild, one fresh draw per non-temporal mode (:61-67),
            // keyed (batch 0, iteration 0).
            rocp_dev::Init init;
            init.dims = d;
            init.rank = rank;
            init.s = s;
            init.regularized = reg_any;
            std::vector<DrawJob> dj;
            for (int n = 1; n < N; ++n)
                dj.push_back(make_draw(d, n, s, seed, 0u, 0u, nullptr, nullptr, idx[size_t(n - 1)].p,
                                       base[size_t(n - 1)].p));
            upload_jobs(dev, dev->jobs, dj, {});
            launch_draw(dev, dev->jobs);
            for (int n = 1; n < N; ++n) {
                SkrJob sj{};
                sj.idx = idx[size_t(n - 1)].p;
                sj.n_other = N - 1;
                sj.s = int32_t(s);
                sj.R = rank;
                int l = 0;
                for (int k = N; k >= 1; --k)
                    if (k != n) sj.f[l++] = best[size_t(k - 1)].p;
                init.best_kr.emplace_back(size_t(s * rank));
                sj.z = init.best_kr.back().p;
                launch_skr(dev, sj);
                if (best_kr) download_colmajor(dev, sj.z, s, rank, best_kr[n - 1]);
            }
            for (int n = 0; n < N; ++n) download_colmajor(dev, best[size_t(n)].p, d[size_t(n)], rank, factors[n]);
            init.factors = std::move(best);
            init.valid = true;
            dev->init = std::move(init);
            *best_fitness = best_fit;
            *iterations = sweep;
            if (regularized) *regularized = reg_any ? 1 : 0;
        },
        err_sweep);
}

// ---- stream ------------------------------------------------------------------
namespace {

rocp_stream* new_stream(rocp_dev* dev, int order, const int64_t* head_dims, int rank, int64_t s,
                        int64_t t_init, int64_t t_capacity) {
    if (order < 2 || order > kMaxOrder) throw_domain("stream order must be in [2, 8]");
    check_rank(rank);
    if (s < 1) throw_domain("init_state: sample count must be positive");
    auto st = std::make_unique<rocp_stream>();
    st->dev = dev;
    st->N = order;
    st->R = rank;
    st->s = s;
    st->head.assign(head_dims, head_dims + order - 1);
    st->t_len = t_init;
    st->t_cap = std::max<int64_t>(t_capacity, t_init);
    st->temporal.alloc(size_t(std::max<int64_t>(st->t_cap, 1) * rank));
    for (int n = 1; n < order; ++n) {
        const int64_t In = st->head[size_t(n - 1)];
        st->U.emplace_back(size_t(In * rank));
        st->P.emplace_back(size_t(In * rank));
        st->Q.emplace_back(size_t(rank * rank));
    }
    for (int stage = 0; stage < order; ++stage) st->Z.emplace_back(size_t(s * rank));
    st->G_t.alloc(size_t(rank * rank));
    st->resid.alloc(size_t(2 * order));
    st->flags.alloc(4);
    st->seed_dev.alloc(1);
    st->batch_dev.alloc(1);
    st->gpart.alloc(size_t(((s + kSuperSamples - 1) / kSuperSamples) * rank * rank));
    st->chpart.alloc(size_t(((s + kChunk - 1) / kChunk) * ((rank * rank + 1) & ~1)));
    st->zmodes.alloc(size_t(order * s * (((rank + kCRB - 1) / kCRB) * kCRB + 4)));
    st->LD.alloc(size_t(rank * rank + rank + 2));
    st->rpart.alloc(size_t(3 * s));
    st->mode_flag.alloc(4);
    CK(cudaMemsetAsync(st->flags.p, 0, 4 * sizeof(int), dev->stream));
    // Reduction scratch sized once: consume (and its CUDA graph) never allocates.
    dev->scratch_a.ensure(size_t((s + kChunk - 1) / kChunk + (s + kSuperSamples - 1) / kSuperSamples) * rank * rank);
    dev->scratch_b.ensure(size_t(3 * s));
    CK(cudaMemsetAsync(st->resid.p, 0, size_t(2 * order) * 8, dev->stream));
    ensure_window(st.get(), 1, 1);
    return st.release();
}

// init_state (rocp.cpp:45-69): Q = Z^T Z, P = U Q (or U with literal_init).
void init_pq(rocp_stream* st, const std::vector<const double*>& z_dev, bool literal) {
    rocp_dev* dev = st->dev;
    for (int n = 1; n < st->N; ++n) {
        launch_gram(dev, z_dev[size_t(n - 1)], st->s, st->R, nullptr, st->Q[size_t(n - 1)].p);
        const int64_t In = st->head[size_t(n - 1)];
        if (literal) {
            CK(cudaMemcpyAsync(st->P[size_t(n - 1)].p, st->U[size_t(n - 1)].p, size_t(In * st->R) * 8,
                               cudaMemcpyDeviceToDevice, dev->stream));
        } else {
            k_mul_uq<<<grid_for(In * st->R, 256, dev->num_sms * 4), 256, 0, dev->stream>>>(
                st->U[size_t(n - 1)].p, int32_t(In), st->R, st->Q[size_t(n - 1)].p, st->P[size_t(n - 1)].p);
            after_launch(dev, "k_mul_uq");
        }
    }
    CK(cudaStreamSynchronize(dev->stream));
}

#include "io_host.inc"

}  // namespace

rocp_status rocp_stream_create(rocp_dev* dev, int order, const int64_t* head_dims, int rank,
                               int64_t s, int literal_init, const double* const* factors,
                               int64_t t_init, const double* const* best_kr, int regularized,
                               int64_t t_capacity, rocp_stream** out) {
    return guarded(dev, [&] {
        std::unique_ptr<rocp_stream> st(new_stream(dev, order, head_dims, rank, s, t_init, t_capacity));
        st->regularized = regularized != 0;
        for (int n = 1; n < order; ++n)
            upload_rowmajor(dev, factors[n - 1], st->head[size_t(n - 1)], rank, st->U[size_t(n - 1)].p);
        if (t_init > 0) upload_rowmajor(dev, factors[order - 1], t_init, rank, st->temporal.p);
        std::vector<DBuf<double>> zb;
        std::vector<const double*> zp;
        for (int n = 1; n < order; ++n) {
            zb.emplace_back(size_t(s * rank));
            upload_rowmajor(dev, best_kr[n - 1], s, rank, zb.back().p);
            zp.push_back(zb.back().p);
        }
        init_pq(st.get(), zp, literal_init != 0);
        *out = st.release();
    });
}

rocp_status rocp_stream_create_from_init(rocp_dev* dev, int literal_init, int64_t t_capacity,
                                         rocp_stream** out) {
    return guarded(dev, [&] {
        if (!dev->init.valid) throw RocpError{ROCP_E_STATE, "no device-resident cprand result"};
        const auto& in = dev->init;
        const int N = int(in.dims.size());
        std::unique_ptr<rocp_stream> st(new_stream(dev, N, in.dims.data(), in.rank, in.s, in.dims.back(), t_capacity));
        st->regularized = in.regularized;
        for (int n = 1; n < N; ++n)
            CK(cudaMemcpyAsync(st->U[size_t(n - 1)].p, in.factors[size_t(n - 1)].p, in.factors[size_t(n - 1)].n * 8,
                               cudaMemcpyDeviceToDevice, dev->stream));
        CK(cudaMemcpyAsync(st->temporal.p, in.factors[size_t(N - 1)].p, in.factors[size_t(N - 1)].n * 8,
                           cudaMemcpyDeviceToDevice, dev->stream));
        std::vector<const double*> zp;
        for (auto& z : in.best_kr) zp.push_back(z.p);
        init_pq(st.get(), zp, literal_init != 0);
        *out = st.release();
    });
}

void rocp_stream_free(rocp_stream* st) {
    if (!st) return;
    cudaStreamSynchronize(st->dev->stream);
    delete st;
}

rocp_status rocp_stream_consume(rocp_stream* st, const rocp_tensor* x_new, uint64_t seed,
                                uint32_t batch_id) {
    return guarded(st->dev, [&] {
        check_head_dims(st, x_new);  // rocp.cpp:145
        if (st->sharded)
            sharded_consume_range(st, x_new->d, x_new->numel / x_new->dims.back(), x_new->dims.back(), 1, seed,
                                  batch_id);
        else
            consume_one(st, x_new->d, x_new->dims.back(), seed, batch_id);
    });
}

rocp_status rocp_tensor_write_file(rocp_dev* dev, const rocp_tensor* t, const char* path) {
    return guarded(dev, [&] {
        File out(path, "wb");
        write_tensor_rec(dev, t, out);
    });
}

rocp_status rocp_tensor_read_file(rocp_dev* dev, const char* path, rocp_tensor** out) {
    return guarded(dev, [&] {
        File in(path, "rb");
        *out = read_tensor_rec(dev, in).release();
    });
}

rocp_status rocp_stream_write_state(rocp_stream* st, const char* path) {
    return guarded(st->dev, [&] {
        if (st->sharded) throw_domain("state records hold the full U(1)/P(1); this stream is sharded");
        File out(path, "wb");
        write_state(st, out);
    });
}

rocp_status rocp_stream_read_state(rocp_stream* st, const char* path) {
    return guarded(st->dev, [&] {
        if (st->sharded) throw_domain("state records hold the full U(1)/P(1); this stream is sharded");
        File in(path, "rb");
        read_state(st, in);
    });
}

rocp_status rocp_stream_write_checkpoint(rocp_stream* st, const char* path) {
    return guarded(st->dev, [&] {
        if (st->sharded) throw_domain("checkpoints hold the full U(1)/P(1); this stream is sharded");
        File out(path, "wb");
        write_checkpoint(st, out);
    });
}

rocp_status rocp_stream_consume_file(rocp_stream* st, const char* path, int64_t t0, int64_t batch, int64_t nb,
                                     uint64_t seed, uint32_t first_batch_id, int threads) {
    return guarded(st->dev, [&] {
        if (st->sharded) throw_domain("file-backed consume is single-GPU (stream is sharded)");
        if (st->resid_level >= 2) throw_domain("consume_file: residual level 2 needs device slabs");
        consume_file(st, path, t0, batch, nb, seed, first_batch_id, threads > 0 ? threads : st->host_threads);
    });
}

rocp_status rocp_stream_create_from_checkpoint(rocp_dev* dev, const char* path, int64_t t_capacity,
                                               rocp_stream** out) {
    return guarded(dev, [&] {
        File in(path, "rb");
        *out = read_checkpoint(dev, in, t_capacity);
    });
}

rocp_status rocp_stream_shard(rocp_stream* st, int virtual_shards) {
    return guarded(st->dev, [&] { shard_stream(st, virtual_shards); });
}

rocp_status rocp_stream_shard_info(rocp_stream* st, int* virtual_shards, int64_t* row0, int64_t* row1) {
    return guarded(st->dev, [&] {
        *virtual_shards = st->sharded ? st->V : 0;
        *row0 = st->sharded ? st->r0 : 0;
        *row1 = st->sharded ? st->r1 : st->head[0];
    });
}

rocp_status rocp_stream_consume_host(rocp_stream* st, const double* x_new, int64_t batch,
                                     uint64_t seed, uint32_t batch_id) {
    return guarded(st->dev, [&] {
        if (batch < 1) throw_domain("batch must hold at least one slice");
        if (st->sharded) throw_domain("host-slab consume is single-GPU (stream is sharded)");
        rocp_dev* dev = st->dev;
        const int64_t numel = prod(st->head) * batch;
        if (st->resid_level >= 2 && st->staging.n < size_t(numel)) {
            CK(cudaStreamSynchronize(dev->stream));
            st->staging.alloc(size_t(numel));
        }
        (void)numel;
        if (st->resid_level >= 2) {  // every-stage residuals use the per-stage kernels: full slab copy
            CK(cudaMemcpyAsync(st->staging.p, x_new, size_t(numel) * 8, cudaMemcpyHostToDevice, dev->stream));
            consume_one(st, st->staging.p, batch, seed, batch_id);
        } else {
            consume_range_host(st, x_new, batch, 1, seed, batch_id, st->host_threads, 1);
        }
    });
}

rocp_status rocp_stream_consume_range(rocp_stream* st, const rocp_tensor* x, int64_t t0,
                                      int64_t batch, int64_t nb, uint64_t seed,
                                      uint32_t first_batch_id) {
    return guarded(st->dev, [&] {
        check_head_dims(st, x);
        if (batch < 1 || nb < 1 || t0 < 0 || t0 + batch * nb > x->dims.back())
            throw_domain("consume_range: slab range out of bounds");
        check_capacity(st, batch * nb);
        rocp_dev* dev = st->dev;
        const int64_t slice = x->numel / x->dims.back();
        if (st->sharded) {
            sharded_consume_range(st, x->d + t0 * slice, slice, batch, nb, seed, first_batch_id);
            return;
        }
        st->win_gsms = st->resid_level <= 1 ? gather_sms(st, batch) : 0;
        const bool overlap = st->win_gsms > 0;
        prepare_window(st, x->d, t0, slice, batch, nb, nullptr, nullptr, -1, false, nullptr, !overlap);
        enqueue_draw_gather(st, seed, first_batch_id, overlap);
        if (st->resid_level <= 1) {
            launch_chain(st, nb, batch, 0, overlap);
        } else {
            auto key = std::make_tuple(nb, batch, st->t_len);
            auto it = st->graphs.find(key);
            if (it == st->graphs.end()) {
                const uint64_t l0 = dev->launches;
                cudaGraph_t graph;
                CK(cudaStreamBeginCapture(dev->stream, cudaStreamCaptureModeThreadLocal));
                try {
                    enqueue_chain(st, nb, batch);
                } catch (...) {
                    cudaStreamEndCapture(dev->stream, &graph);
                    throw;
                }
                CK(cudaStreamEndCapture(dev->stream, &graph));
                cudaGraphExec_t exec;
                CK(cudaGraphInstantiate(&exec, graph, 0));
                cudaGraphDestroy(graph);
                const uint64_t nodes = dev->launches - l0;
                dev->launches = l0;
                it = st->graphs.emplace(key, std::make_pair(exec, nodes)).first;
            }
            CK(cudaGraphLaunch(it->second.first, dev->stream));
            dev->launches += it->second.second;
        }
        st->t_len += batch * nb;
    });
}

rocp_status rocp_stream_consume_range_host(rocp_stream* st, const double* x, int64_t batch, int64_t nb,
                                           uint64_t seed, uint32_t first_batch_id, int threads) {
    return guarded(st->dev, [&] {
        if (batch < 1 || nb < 1) throw_domain("consume_range_host: empty range");
        if (st->sharded) throw_domain("host-slab consume is single-GPU (stream is sharded)");
        if (st->resid_level >= 2) throw_domain("consume_range_host: residual level 2 needs device slabs");
        consume_range_host(st, x, batch, nb, seed, first_batch_id, threads > 0 ? threads : st->host_threads, 0);
    });
}

rocp_status rocp_stream_update_last_mode_with(rocp_stream* st, const rocp_tensor* x_new,
                                              const int64_t* rows, int64_t s, double* u_new,
                                              double* z_s, int* regularized) {
    return guarded(st->dev, [&] {
        if (st->sharded) throw_domain("replay seams are single-GPU (stream is sharded)");
        check_head_dims(st, x_new);
        if (s != st->s) throw_domain("index set size must equal the stream sample count");
        rocp_dev* dev = st->dev;
        const int64_t B = x_new->dims.back();
        const int64_t co = prod(st->head);
        for (int64_t c = 0; c < s; ++c)
            if (rows[c] < 1 || rows[c] > co) throw_domain("column index out of range");
        DBuf<int64_t> din(static_cast<size_t>(s));
        CK(cudaMemcpyAsync(din.p, rows, size_t(s) * 8, cudaMemcpyHostToDevice, dev->stream));
        prepare_window(st, x_new->d, 0, prod(st->head), B, 1, din.p, nullptr, 0);
        enqueue_draw_gather(st, 0, 0);
        DBuf<double> du(static_cast<size_t>(B * st->R));
        int saved = 0;
        CK(cudaMemcpyAsync(&saved, st->flags.p, sizeof(int), cudaMemcpyDeviceToHost, dev->stream));
        CK(cudaStreamSynchronize(dev->stream));
        CK(cudaMemsetAsync(st->flags.p, 0, sizeof(int), dev->stream));
        stage_temporal(st, 0, B, du.p);
        int hf = 0;
        CK(cudaMemcpyAsync(&hf, st->flags.p, sizeof(int), cudaMemcpyDeviceToHost, dev->stream));
        CK(cudaStreamSynchronize(dev->stream));
        // the replay seam leaves the stream's own flag untouched (rocp.cpp:71-84 is pure)
        CK(cudaMemcpyAsync(st->flags.p, &saved, sizeof(int), cudaMemcpyHostToDevice, dev->stream));
        download_colmajor(dev, du.p, B, st->R, u_new);
        if (z_s) download_colmajor(dev, st->Z[0].p, s, st->R, z_s);
        if (regularized) *regularized = hf & 1;
        st->win.key_x = nullptr;  // din is released: the job list must not be reused
    });
}

rocp_status rocp_stream_append_temporal(rocp_stream* st, const double* u_new, int64_t batch) {
    return guarded(st->dev, [&] {
        if (batch < 0) throw_domain("append_temporal: negative batch");
        check_capacity(st, batch);
        std::vector<double> rm = colmajor_to_rowmajor(u_new, batch, st->R);
        CK(cudaMemcpyAsync(st->temporal.p + st->t_len * st->R, rm.data(), rm.size() * 8, cudaMemcpyHostToDevice,
                           st->dev->stream));
        CK(cudaStreamSynchronize(st->dev->stream));
    });
}

rocp_status rocp_stream_update_mode_with(rocp_stream* st, const rocp_tensor* x_new,
                                         const double* u_new, int mode, const int64_t* rows,
                                         int64_t s, double* z_new, double* x_s, int* regularized) {
    return guarded(st->dev, [&] {
        if (st->sharded) throw_domain("replay seams are single-GPU (stream is sharded)");
        check_head_dims(st, x_new);
        if (mode < 1 || mode >= st->N)
            throw_domain("update_mode_with: index set must be over a non-temporal mode");  // rocp.cpp:100-101
        if (s != st->s) throw_domain("index set size must equal the stream sample count");
        rocp_dev* dev = st->dev;
        const int64_t B = x_new->dims.back();
        const std::vector<int64_t> d = slab_dims(st, B);
        int64_t co = 1;
        for (int k = 0; k < st->N; ++k)
            if (k + 1 != mode) co *= d[size_t(k)];
        for (int64_t c = 0; c < s; ++c)
            if (rows[c] < 1 || rows[c] > co) throw_domain("column index out of range");
        DBuf<int64_t> din(static_cast<size_t>(s));
        CK(cudaMemcpyAsync(din.p, rows, size_t(s) * 8, cudaMemcpyHostToDevice, dev->stream));
        DBuf<double> du(static_cast<size_t>(B * st->R));
        upload_rowmajor(dev, u_new, B, st->R, du.p);
        prepare_window(st, x_new->d, 0, prod(st->head), B, 1, nullptr, din.p, mode);
        enqueue_draw_gather(st, 0, 0);
        CK(cudaMemsetAsync(st->flags.p + 2, 0, sizeof(int), dev->stream));
        stage_mode(st, 0, mode, du.p);
        int hf[4];
        CK(cudaMemcpyAsync(hf, st->flags.p, sizeof(hf), cudaMemcpyDeviceToHost, dev->stream));
        if (z_new) download_colmajor(dev, st->Z[size_t(mode)].p, s, st->R, z_new);
        std::vector<double> xt;
        const int64_t In = st->head[size_t(mode - 1)];
        if (x_s) {
            xt.resize(size_t(xs_size(In, s)));
            CK(cudaMemcpyAsync(xt.data(), win_x(st, 0, mode), xt.size() * 8, cudaMemcpyDeviceToHost, dev->stream));
        }
        CK(cudaStreamSynchronize(dev->stream));
        if (x_s)
            for (int64_t c = 0; c < s; ++c)
                for (int64_t i = 0; i < In; ++i) x_s[i + c * In] = xt[size_t(xs_offset(i, c, s))];
        if (regularized) *regularized = hf[2] & 1;
        st->win.key_x = nullptr;
    });
}

rocp_status rocp_stream_finish_batch(rocp_stream* st, int64_t batch) {
    return guarded(st->dev, [&] {
        if (batch < 0) throw_domain("finish_batch: negative batch");
        check_capacity(st, batch);
        st->t_len += batch;
    });
}

rocp_status rocp_stream_mark_regularized(rocp_stream* st) {
    return guarded(st->dev, [&] { st->regularized = true; });
}

rocp_status rocp_stream_get(rocp_stream* st, int what, int mode, double* out) {
    return guarded(st->dev, [&] {
        rocp_dev* dev = st->dev;
        if (what == 3) {
            download_colmajor(dev, st->temporal.p, st->t_len, st->R, out);
            return;
        }
        if (mode < 1 || mode >= st->N) throw_domain("mode out of range");
        const int64_t In = st->head[size_t(mode - 1)];
        if (what == 0) download_colmajor(dev, st->U[size_t(mode - 1)].p, In, st->R, out);
        else if (what == 1) download_colmajor(dev, st->P[size_t(mode - 1)].p, In, st->R, out);
        else if (what == 2) download_colmajor(dev, st->Q[size_t(mode - 1)].p, st->R, st->R, out);
        else throw_domain("bad selector");
    });
}

rocp_status rocp_stream_set(rocp_stream* st, int what, int mode, const double* in) {
    return guarded(st->dev, [&] {
        rocp_dev* dev = st->dev;
        if (mode < 1 || mode >= st->N) throw_domain("mode out of range");
        const int64_t In = st->head[size_t(mode - 1)];
        if (what == 0) upload_rowmajor(dev, in, In, st->R, st->U[size_t(mode - 1)].p);
        else if (what == 1) upload_rowmajor(dev, in, In, st->R, st->P[size_t(mode - 1)].p);
        else if (what == 2) upload_rowmajor(dev, in, st->R, st->R, st->Q[size_t(mode - 1)].p);
        else throw_domain("bad selector");
    });
}

rocp_status rocp_stream_checkpoint(rocp_stream* st) {
    return guarded(st->dev, [&] {
        rocp_dev* dev = st->dev;
        if (st->ckU.empty()) {
            for (int n = 1; n < st->N; ++n) {
                st->ckU.emplace_back(st->U[size_t(n - 1)].n);
                st->ckP.emplace_back(st->P[size_t(n - 1)].n);
                st->ckQ.emplace_back(st->Q[size_t(n - 1)].n);
            }
        }
        for (int n = 0; n < st->N - 1; ++n) {
            CK(cudaMemcpyAsync(st->ckU[size_t(n)].p, st->U[size_t(n)].p, st->U[size_t(n)].n * 8, cudaMemcpyDeviceToDevice, dev->stream));
            CK(cudaMemcpyAsync(st->ckP[size_t(n)].p, st->P[size_t(n)].p, st->P[size_t(n)].n * 8, cudaMemcpyDeviceToDevice, dev->stream));
            CK(cudaMemcpyAsync(st->ckQ[size_t(n)].p, st->Q[size_t(n)].p, st->Q[size_t(n)].n * 8, cudaMemcpyDeviceToDevice, dev->stream));
        }
        int hf[4];
        CK(cudaMemcpyAsync(hf, st->flags.p, sizeof(hf), cudaMemcpyDeviceToHost, dev->stream));
        CK(cudaStreamSynchronize(dev->stream));
        st->ck_t_len = st->t_len;
        st->ck_reg = st->regularized || (hf[0] & 1);
    });
}

rocp_status rocp_stream_restore(rocp_stream* st) {
    return guarded(st->dev, [&] {
        if (st->ck_t_len < 0) throw RocpError{ROCP_E_STATE, "no checkpoint"};
        rocp_dev* dev = st->dev;
        for (int n = 0; n < st->N - 1; ++n) {
            CK(cudaMemcpyAsync(st->U[size_t(n)].p, st->ckU[size_t(n)].p, st->U[size_t(n)].n * 8, cudaMemcpyDeviceToDevice, dev->stream));
            CK(cudaMemcpyAsync(st->P[size_t(n)].p, st->ckP[size_t(n)].p, st->P[size_t(n)].n * 8, cudaMemcpyDeviceToDevice, dev->stream));
            CK(cudaMemcpyAsync(st->Q[size_t(n)].p, st->ckQ[size_t(n)].p, st->Q[size_t(n)].n * 8, cudaMemcpyDeviceToDevice, dev->stream));
        }
        // asynchronous: flags reset by a kernel, no host synchronisation
        k_set_i32<<<1, 32, 0, dev->stream>>>(st->flags.p, 4, 0);
        after_launch(dev, "k_set_i32");
        if (st->ck_reg) {
            k_set_i32<<<1, 32, 0, dev->stream>>>(st->flags.p, 1, 1);
            after_launch(dev, "k_set_i32");
        }
        st->t_len = st->ck_t_len;  // temporal rows beyond t_len are rewritten by the next consume
    });
}

int64_t rocp_stream_t_len(const rocp_stream* st) { return st ? st->t_len : -1; }

rocp_status rocp_stream_set_residual_tracking(rocp_stream* st, int enable) {
    return guarded(st->dev, [&] {
        if (enable < 0 || enable > 2) throw_domain("residual level must be 0, 1 or 2");
        if (st->resid_level != enable) clear_graphs(st);
        st->resid_level = enable;
    });
}

rocp_status rocp_stream_chain_times(rocp_stream* st, float* ms, int max, int* count) {
    return guarded(st->dev, [&] {
        CK(cudaStreamSynchronize(st->dev->stream));
        const int n = int(std::min<size_t>(st->chain_events_used, size_t(std::max(max, 0))));
        for (int k = 0; k < n; ++k)
            CK(cudaEventElapsedTime(ms + k, st->chain_events[size_t(k)].first, st->chain_events[size_t(k)].second));
        *count = int(st->chain_events_used);
        st->chain_events_used = 0;
    });
}

rocp_status rocp_stream_time_gather(rocp_stream* st, int enable) {
    return guarded(st->dev, [&] {
        st->time_gather = enable != 0;
        st->gather_events_used = 0;
        st->chain_events_used = 0;
    });
}

rocp_status rocp_stream_gather_window(rocp_stream* st, const rocp_tensor* x, int64_t t0, int64_t batch, int64_t nb,
                                      uint64_t seed, uint32_t first_batch_id, int sms, float* ms) {
    return guarded(st->dev, [&] {
        check_head_dims(st, x);
        if (st->sharded) throw_domain("gather_window: single-GPU streams only");
        if (batch < 1 || nb < 1 || t0 < 0 || t0 + batch * nb > x->dims.back())
            throw_domain("gather_window: slab range out of bounds");
        rocp_dev* dev = st->dev;
        if (sms <= 0 || sms > dev->num_sms) sms = dev->num_sms;
        gather_sms(st, batch);  // gather stream + kernel attributes
        prepare_window(st, x->d, t0, x->numel / x->dims.back(), batch, nb, nullptr, nullptr, -1);
        const JobList& L = st->win.jobs;
        k_set_u64<<<1, 1, 0, dev->stream>>>(st->seed_dev.p, seed);
        after_launch(dev, "k_set_u64");
        k_set_u32<<<1, 1, 0, dev->stream>>>(st->batch_dev.p, first_batch_id);
        after_launch(dev, "k_set_u32");
        CK(cudaMemsetAsync(L.done.p, 0, size_t(L.ngather) * sizeof(unsigned), dev->stream));
        launch_draw(dev, L);
        if (L.nsort > 0) {
            k_sort_by_base<<<L.nsort, 1024, 0, dev->stream>>>(L.sort.p);
            after_launch(dev, "k_sort_by_base");
        }
        struct Ev {  // destroyed on every exit path
            cudaEvent_t e = nullptr;
            ~Ev() {
                if (e) cudaEventDestroy(e);
            }
        } a, b;
        CK(cudaEventCreate(&a.e));
        CK(cudaEventCreate(&b.e));
        CK(cudaEventRecord(a.e, dev->stream));
        k_gather_warps<<<sms, kGWThreads, kGWSmem, dev->stream>>>(st->win.gtp, L.gather.p, L.ngather, L.ustart.p,
                                                                  L.done.p);
        after_launch(dev, "k_gather_warps");
        CK(cudaEventRecord(b.e, dev->stream));
        CK(cudaEventSynchronize(b.e));
        CK(cudaEventElapsedTime(ms, a.e, b.e));
    });
}

rocp_status rocp_stream_last_gather_sms(const rocp_stream* st, int* sms) {
    if (!st || !sms) return ROCP_E_DOMAIN;
    *sms = st->win_gsms;
    return ROCP_OK;
}

rocp_status rocp_stream_gather_times(rocp_stream* st, float* ms, int max, int* count) {
    return guarded(st->dev, [&] {
        CK(cudaStreamSynchronize(st->dev->stream));
        const int n = int(std::min<size_t>(st->gather_events_used, size_t(std::max(max, 0))));
        for (int k = 0; k < n; ++k)
            CK(cudaEventElapsedTime(ms + k, st->gather_events[size_t(k)].first, st->gather_events[size_t(k)].second));
        *count = int(st->gather_events_used);
        st->gather_events_used = 0;
    });
}

rocp_status rocp_stream_chain_trace(rocp_stream* st, int enable, uint64_t* out, int64_t max, int64_t* count) {
    return guarded(st->dev, [&] {
        st->trace_on = enable != 0;
        if (out && max > 0 && st->trace_n > 0) {
            CK(cudaStreamSynchronize(st->dev->stream));
            const int64_t n = std::min(max, st->trace_n);
            CK(cudaMemcpy(out, st->trace.p, size_t(n) * 8, cudaMemcpyDeviceToHost));
        }
        if (count) *count = st->trace_n;
    });
}

rocp_status rocp_stream_window_bytes(rocp_stream* st, int64_t* useful, int64_t* elements) {
    return guarded(st->dev, [&] {
        *elements = st->win.jobs.gather_elems;
        *useful = st->win.jobs.gather_elems * int64_t(sizeof(double));
    });
}

int rocp_stream_regularized(rocp_stream* st) {
    // The reference's consume raises the stream flag from the temporal solve
    // only (rocp.cpp:150); flags[0] accumulates device-side.
    int hf[2] = {0, 0};
    cudaMemcpyAsync(hf, st->flags.p, sizeof(hf), cudaMemcpyDeviceToHost, st->dev->stream);
    cudaStreamSynchronize(st->dev->stream);
    return (st->regularized || (hf[0] & 1)) ? 1 : 0;
}

rocp_status rocp_stream_last_residuals(rocp_stream* st, double* out) {
    return guarded(st->dev, [&] {
        std::vector<double> h(size_t(2 * st->N));
        CK(cudaMemcpyAsync(h.data(), st->resid.p, h.size() * 8, cudaMemcpyDeviceToHost, st->dev->stream));
        CK(cudaStreamSynchronize(st->dev->stream));
        for (int k = 0; k < st->N; ++k) {
            const double num = h[size_t(2 * k)], den = h[size_t(2 * k + 1)];
            out[k] = den > 0.0 ? std::sqrt(num) / std::sqrt(den) : 0.0;
        }
    });
}

}  // extern "C"
