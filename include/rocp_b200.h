/*
 * rocp_b200.h -- C ABI of the B200-native ROCP hot path (librocp_b200.so).
 *
 * This is the drop-in boundary: plain pointers and sizes, no C++ or torch
 * types.  Every entry point names the reference interface it replaces
 * (reference = /root/reference/proj).  The C++ host API that mirrors the
 * reference headers one-for-one (include/rocp/ *.hpp) is built on top of it,
 * and so are the Python tests and bench.py (ctypes).  INTEGRATION.md shows the
 * bindings a maintainer adds on the reference side.
 *
 * Layouts (identical to the reference unless stated):
 *   tensor   float64, first index fastest (tensor.hpp:14-16), dims int64.
 *   matrices column-major float64 (Eigen::MatrixXd default, tensor.hpp:10).
 *   indices  1-based int64: rows[s], decoded[s*(N-1)] row-major in increasing
 *            mode order (SampleIndexSet, sampling.hpp:14-26).
 * Device-internal layouts (factor rows contiguous) are
 * converted at this boundary.
 *
 * Errors: every call returns rocp_status; rocp_last_error(dev) gives the
 * message.  ROCP_E_DOMAIN <-> std::domain_error, ROCP_E_NUMERICAL <->
 * rocp::NumericalError (sweep in *err_sweep), matching errors.hpp:10-20.
 * Threading: one handle per GPU, one caller thread per handle (the reference's
 * single-owner contract).
 * Randomness: sample indices come from the counter RNG of DESIGN.md 3.1,
 * keyed by (seed, batch, iteration, mode); the host oracle reproduces them
 * bit-for-bit.
 */
#ifndef ROCP_B200_H
#define ROCP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    ROCP_OK = 0,
    ROCP_E_DOMAIN = 1,    /* std::domain_error in the reference */
    ROCP_E_NUMERICAL = 2, /* rocp::NumericalError (errors.hpp:10) */
    ROCP_E_CUDA = 3,
    ROCP_E_NCCL = 4,
    ROCP_E_OOM = 5,
    ROCP_E_STATE = 6,
    ROCP_E_IO = 7 /* file records (std::runtime_error in tensor_io.cpp / rocp.cpp) */
} rocp_status;

typedef struct rocp_dev rocp_dev;       /* one per GPU: stream, scratch, comm */
typedef struct rocp_tensor rocp_tensor; /* device-resident DenseTensor */
typedef struct rocp_stream rocp_stream; /* device-resident RocpStream state */

/* ---- handle ------------------------------------------------------------- */
/* world/rank/nccl_id: mode-1 sharding across GPUs;
 * world = 1 and nccl_id = NULL for one GPU. */
rocp_status rocp_create(int device, int world, int rank, const void* nccl_id, rocp_dev** out);
void rocp_destroy(rocp_dev* dev);
const char* rocp_last_error(const rocp_dev* dev);
rocp_status rocp_synchronize(rocp_dev* dev);
/* Number of kernels this library launched on dev since creation. */
uint64_t rocp_kernel_launches(const rocp_dev* dev);
/* CUDA-event timers on the handle's stream (8 slots): record, then the
 * elapsed milliseconds between two recorded slots (waits for the second). */
rocp_status rocp_timer_record(rocp_dev* dev, int slot);
rocp_status rocp_timer_elapsed_ms(rocp_dev* dev, int a, int b, float* ms);
/* SMs reserved for the overlapped window gather of stream windows (DESIGN.md
 * 5.3): the gather runs on `sms` SMs beside the persistent chain kernel, which
 * takes the rest; 0 gathers each window on every SM before the chain; < 0
 * (default, unless ROCP_GATHER_SMS is set) lets a per-stream model choose.
 * Results are bitwise identical for every setting.  No reference counterpart
 * (a B200 scheduling knob). */
rocp_status rocp_set_gather_sms(rocp_dev* dev, int sms);
/* Blocks of this handle's persistent chain kernel (0 = one per SM, the default;
 * otherwise 16 .. SM count).  For several independent streams on one GPU, one
 * handle each -- the reference's trial-level parallelism (bench.cpp:190-213,
 * ROCP_THREADS): with K handles at SMs/K blocks each, the K cooperative chains are
 * co-resident and the GPU's otherwise idle SMs serve the other streams.  Results
 * are bitwise identical for every setting.  No reference counterpart. */
rocp_status rocp_set_chain_sms(rocp_dev* dev, int sms);
/* The device's SM count (to size rocp_set_chain_sms shares). */
rocp_status rocp_sm_count(rocp_dev* dev, int* sms);
/* Measurement aid (no reference counterpart): event-timed kernel of `reads`
 * independent 8-byte loads at hashed offsets of t on every SM -- the device's
 * isolated random-read ceiling that bounds the strided sampled-fibre gather
 * (DESIGN.md section 5).  *ms = the timed launch (after one warm-up launch). */
rocp_status rocp_probe_random_reads(rocp_dev* dev, const rocp_tensor* t, int64_t reads, uint64_t seed, float* ms);
/* solve_gram regularisation decisions taken on this device since the last reset
 * (DESIGN.md 3.4): counts[0] no regularisation, [1] regularised, [2] settled by
 * exact (Jacobi) eigenvalues, [3] needed the tier-2 tr(G^-1) certificate.
 * Diagnostic (no reference counterpart). */
rocp_status rocp_decision_stats(rocp_dev* dev, uint64_t* counts, int reset);
/* The handle's cudaStream_t (for callers that interoperate). */
void* rocp_cuda_stream(rocp_dev* dev);
/* Page-locked, CUDA-registered host buffer backed by 2 MB (transparent huge)
 * pages, for host-slab streams (rocp_stream_consume_range_host).  NULL on
 * failure.  Free with the same size. */
void* rocp_host_alloc(size_t bytes);
void rocp_host_free(void* p, size_t bytes);
/* Size of the NCCL unique id blob (for the host bootstrap), 0 if no NCCL. */
int rocp_nccl_id_size(void);
rocp_status rocp_nccl_get_unique_id(void* out);

/* ---- tensors (DenseTensor, tensor.hpp:17-49) ------------------------------ */
/* host may be NULL (zero-filled). */
rocp_status rocp_tensor_create(rocp_dev* dev, const int64_t* dims, int order, const double* host,
                               rocp_tensor** out);
/* Contiguous slab [t0, t0+len) of the last mode, no copy (split_stream,
 * synthetic.cpp:33-57). */
rocp_status rocp_tensor_slab(rocp_dev* dev, const rocp_tensor* t, int64_t t0, int64_t len,
                             rocp_tensor** out);
/* Rows [r0, r1) of mode 1 as a new owned tensor (the local block of a
 * mode-1 sharded stream). */
rocp_status rocp_tensor_rows(rocp_dev* dev, const rocp_tensor* t, int64_t r0, int64_t r1, rocp_tensor** out);
/* The reference's binary tensor record ("ROCP", u8 version 1, u32le order,
 * u64le dims, little-endian binary64 values first index fastest;
 * write_tensor_file / read_tensor_file, tensor_io.cpp:49-89), streamed through
 * a pinned staging buffer.  ROCP_E_IO on open/format/truncation errors. */
rocp_status rocp_tensor_write_file(rocp_dev* dev, const rocp_tensor* t, const char* path);
rocp_status rocp_tensor_read_file(rocp_dev* dev, const char* path, rocp_tensor** out);
void rocp_tensor_free(rocp_tensor* t);
rocp_status rocp_tensor_upload(rocp_dev* dev, rocp_tensor* t, const double* host);
rocp_status rocp_tensor_download(rocp_dev* dev, const rocp_tensor* t, double* host);
double* rocp_tensor_device_ptr(rocp_tensor* t);
int64_t rocp_tensor_numel(const rocp_tensor* t);
/* Synthetic data (gen_synthetic, synthetic.cpp:8-31): t = [[factors]] plus
 * Gaussian noise scaled so 10 log10(|signal|^2/|noise|^2) = snr_db exactly
 * (no noise when has_noise == 0).  factors: N host column-major arrays. */
rocp_status rocp_generate_synthetic(rocp_dev* dev, rocp_tensor* t, const double* const* factors,
                                    int rank, int has_noise, double snr_db, uint64_t noise_seed);

/* ---- primitives (sampling.hpp:35-48, solve.hpp:20-24, kruskal.hpp:39) ----- */
/* draw_samples (sampling.cpp:47-55) with the counter RNG. decoded may be NULL. */
rocp_status rocp_draw_samples(rocp_dev* dev, const int64_t* dims, int order, int mode, int64_t s,
                              uint64_t seed, uint32_t batch, uint32_t iteration, int64_t* rows,
                              int64_t* decoded);
/* SampleIndexSet::from_rows decode (sampling.cpp:24-31). */
rocp_status rocp_decode_rows(rocp_dev* dev, const int64_t* dims, int order, int mode,
                             const int64_t* rows, int64_t s, int64_t* decoded);
/* sample_unfolding (sampling.cpp:57-79): out is I_mode x s column-major. */
rocp_status rocp_sample_unfolding(rocp_dev* dev, const rocp_tensor* t, int mode,
                                  const int64_t* rows, int64_t s, double* out);
/* sampled_khatri_rao (sampling.cpp:81-105): factors in factors_excluding
 * order (kruskal.cpp:44-53), each factor_rows[l] x rank column-major. */
rocp_status rocp_sampled_khatri_rao(rocp_dev* dev, const int64_t* decoded, int64_t s, int n_other,
                                    const double* const* factors, const int64_t* factor_rows,
                                    int rank, double* z);
/* Gram Z^T Z (solve.cpp:41) and contraction X_s Z (solve.cpp:42). */
rocp_status rocp_gram(rocp_dev* dev, const double* z, int64_t s, int rank, double* g);
rocp_status rocp_contract(rocp_dev* dev, const double* x, int64_t rows, int64_t s, const double* z,
                          int rank, double* out);
/* solve_gram (solve.cpp:9-35). */
rocp_status rocp_solve_gram(rocp_dev* dev, const double* gram, const double* rhs, int64_t rows,
                            int rank, double* out, int* regularized);
/* solve_sampled_ls (solve.cpp:37-44). */
rocp_status rocp_solve_sampled_ls(rocp_dev* dev, const double* z, const double* x, int64_t s,
                                  int64_t rows, int rank, double* out, int* regularized,
                                  int* underdetermined);
/* model_fitness (kruskal.cpp:87-89) without materialising x_hat. */
rocp_status rocp_model_fitness(rocp_dev* dev, const rocp_tensor* t, const double* const* factors,
                               int rank, double* fit);

/* ---- randomized CP-ALS (cprand_decompose, cprand.cpp:12-69) --------------- */
/* factors: N host column-major arrays, in = initial model (random_model),
 * out = best iterate.  best_kr: N-1 host s x rank outputs (InitResult::
 * best_sampled_kr).  fit_trace (optional, max_iters) gets the per-sweep fit. */
rocp_status rocp_cprand(rocp_dev* dev, const rocp_tensor* t, int rank, int64_t samples, double tol,
                        int max_iters, uint64_t seed, double* const* factors,
                        double* const* best_kr, double* best_fitness, int* iterations,
                        int* regularized, int* err_sweep, double* fit_trace);

/* ---- online stream (RocpStream, rocp.hpp:85-107; init_state rocp.cpp:45-69)  */
/* factors: N host column-major arrays (last = temporal factor, t_init rows);
 * best_kr: N-1 host s x rank arrays.  t_capacity preallocates the temporal
 * factor on device (>= total stream length). */
rocp_status rocp_stream_create(rocp_dev* dev, int order, const int64_t* head_dims, int rank,
                               int64_t s, int literal_init, const double* const* factors,
                               int64_t t_init, const double* const* best_kr, int regularized,
                               int64_t t_capacity, rocp_stream** out);
/* Same, from the device-resident result of the last rocp_cprand on dev (no
 * host round trip). */
rocp_status rocp_stream_create_from_init(rocp_dev* dev, int literal_init, int64_t t_capacity,
                                         rocp_stream** out);
void rocp_stream_free(rocp_stream* st);
/* RocpStream::consume (rocp.cpp:144-160) on a device slab; asynchronous.
 * Draws keyed by (seed, batch_id, iteration 0). */
rocp_status rocp_stream_consume(rocp_stream* st, const rocp_tensor* x_new, uint64_t seed,
                                uint32_t batch_id);
/* Mode-1 sharding (north star: tensors sharded along mode 1, partial
 * contractions / Grams of the non-owned modes combined by an NCCL collective,
 * owned-mode rows local).  Converts a freshly created
 * stream (identical on every rank) into rank dev->rank of dev->world: U(1),
 * P(1) keep rows [r0, r1) of the virtual shards [v0, v1) out of
 * `virtual_shards` fixed row ranges (the world size must divide it).  Every
 * later consume / consume_range takes the rank's LOCAL tensor (rocp_tensor_rows)
 * and reproduces oracle/orc_stream_consume_sharded bit for bit for any world
 * size; rocp_stream_get(mode 1) returns the local rows.  Host-slab consumes and
 * the replay seams stay single-GPU (E_DOMAIN on a sharded stream). */
rocp_status rocp_stream_shard(rocp_stream* st, int virtual_shards);
/* Emulated ranks (a test/measurement harness for the sharded path when fewer GPUs
 * than ranks exist): a handle that is rank `rank` of `world`
 * on `device` without NCCL.  Streams on such handles, sharded as usual, run together
 * through rocp_emulated_group_consume_range: every member's action is issued in
 * turn, the members' exchange tables point at each other's areas in device memory
 * (the peer-memory protocol of the real multi-GPU path, minus IPC), and all members'
 * producers are joined (events) before any consumer, so no kernel waits on a peer
 * that is not yet launched.  Results equal a real world-size run bit for bit
 * (oracle orc_stream_consume_sharded). */
rocp_status rocp_create_emulated_rank(int device, int world, int rank, rocp_dev** out);
rocp_status rocp_emulated_group_consume_range(rocp_stream* const* ranks, int world, const rocp_tensor* const* x_local,
                                              int64_t t0, int64_t batch, int64_t nb, uint64_t seed,
                                              uint32_t first_batch_id);
/* ComplementaryState records.  write_state writes exactly the reference's
 * save_state record (rocp.cpp:180-184: P(1..N-1), Q(1..N-1) matrix records,
 * u64le t_len), readable by its load_state; read_state loads such a record
 * into a stream of the same shape (rocp.cpp:186-211 + assignment).  A
 * checkpoint adds what resuming needs (section 8f of SURVEY.md): U(1..N-1)
 * and temporal records before P and Q, and a tail u64le t_len, s, flags.
 * Sharded streams: E_DOMAIN (their U(1)/P(1) are partial). */
rocp_status rocp_stream_write_state(rocp_stream* st, const char* path);
rocp_status rocp_stream_read_state(rocp_stream* st, const char* path);
rocp_status rocp_stream_write_checkpoint(rocp_stream* st, const char* path);
rocp_status rocp_stream_create_from_checkpoint(rocp_dev* dev, const char* path, int64_t t_capacity,
                                               rocp_stream** out);
/* File-backed stream: slabs [t0, t0 + nb*batch) of the last mode of a tensor
 * record (read_tensor_file format) are read into pinned huge-page staging and
 * consumed exactly as rocp_stream_consume_range_host (same results bit for
 * bit).  The head extents must match the stream; threads 0 = all cores. */
rocp_status rocp_stream_consume_file(rocp_stream* st, const char* path, int64_t t0, int64_t batch, int64_t nb,
                                     uint64_t seed, uint32_t first_batch_id, int threads);
rocp_status rocp_stream_shard_info(rocp_stream* st, int* virtual_shards, int64_t* row0, int64_t* row1);
/* Same for a host slab (head dims x batch, first index fastest): the
 * reference-facing call.  Only the sampled fibres cross PCIe (see
 * rocp_stream_consume_range_host). */
rocp_status rocp_stream_consume_host(rocp_stream* st, const double* x_new, int64_t batch,
                                     uint64_t seed, uint32_t batch_id);
/* Same for nb consecutive HOST slabs (head dims x nb*batch, first index
 * fastest): the device draws the window's indices, `threads` host threads
 * (0 = all) gather only the sampled fibres into pinned staging, and sub-window
 * copies overlap the device chain.  rocp_stream_consume_host uses this path
 * with nb = 1. */
rocp_status rocp_stream_consume_range_host(rocp_stream* st, const double* x, int64_t batch, int64_t nb,
                                           uint64_t seed, uint32_t first_batch_id, int threads);
/* Consume nb consecutive slabs of `batch` slices of a device tensor starting
 * at slice t0 (batch ids first_batch_id, first_batch_id+1, ...).  One call,
 * captured once into a CUDA graph per shape. */
rocp_status rocp_stream_consume_range(rocp_stream* st, const rocp_tensor* x, int64_t t0,
                                      int64_t batch, int64_t nb, uint64_t seed,
                                      uint32_t first_batch_id);
/* Replay seams (rocp.cpp:71-84 update_last_mode_with; 96-113
 * update_mode_with): explicit 1-based column indices over x_new's dims. */
rocp_status rocp_stream_update_last_mode_with(rocp_stream* st, const rocp_tensor* x_new,
                                              const int64_t* rows, int64_t s, double* u_new,
                                              double* z_s, int* regularized);
rocp_status rocp_stream_append_temporal(rocp_stream* st, const double* u_new, int64_t batch);
rocp_status rocp_stream_update_mode_with(rocp_stream* st, const rocp_tensor* x_new,
                                         const double* u_new, int mode, const int64_t* rows,
                                         int64_t s, double* z_new, double* x_s, int* regularized);
rocp_status rocp_stream_finish_batch(rocp_stream* st, int64_t batch);
/* Raises the stream's regularized flag (RocpStream::consume ORs the temporal
 * solve's flag into it, rocp.cpp:150; the replay seams leave it untouched). */
rocp_status rocp_stream_mark_regularized(rocp_stream* st);
/* what: 0 = U(mode) (I x R), 1 = P(mode), 2 = Q(mode) (R x R),
 *       3 = temporal factor (t_len x R, mode ignored).  Column-major. */
rocp_status rocp_stream_get(rocp_stream* st, int what, int mode, double* out);
rocp_status rocp_stream_set(rocp_stream* st, int what, int mode, const double* in);
int64_t rocp_stream_t_len(const rocp_stream* st);
int rocp_stream_regularized(rocp_stream* st);
/* Device-side checkpoint / restore of the whole stream state (factors, P, Q,
 * t_len, flag): the exact-resume primitive of SURVEY.md 8f row 3 (the
 * reference's save_state/load_state, rocp.cpp:180-211, keeps only P, Q, t_len;
 * with the counter RNG, (seed, next batch id) is the only other state). */
rocp_status rocp_stream_checkpoint(rocp_stream* st);
rocp_status rocp_stream_restore(rocp_stream* st);
/* Sampled residual per batch: 0 off, 1 temporal solve only (default), 2 every
 * stage. */
rocp_status rocp_stream_set_residual_tracking(rocp_stream* st, int level);
/* CUDA events around every window gather launch (the HBM-bound kernel) and
 * every persistent chain launch: enable, then read the per-launch
 * milliseconds (each call resets its list). */
rocp_status rocp_stream_time_gather(rocp_stream* st, int enable);
rocp_status rocp_stream_gather_times(rocp_stream* st, float* ms, int max, int* count);
rocp_status rocp_stream_chain_times(rocp_stream* st, float* ms, int max, int* count);
/* Profiling aid: draw + sort + the window gather of consume_range's window
 * (t0, batch, nb, seed, first_batch_id) ALONE, as k_gather_warps on `sms` SMs
 * (<= 0: every SM), event-timed into *ms.  Fills the window scratch only; the
 * stream's model is untouched.  Used by bench.py for the gather kernel's
 * whole-device roofline (in a step it runs overlapped on a few SMs). */
/* SMs the last stream window's gather was overlapped on (0: gathered on every
 * SM before the chain). */
rocp_status rocp_stream_last_gather_sms(const rocp_stream* st, int* sms);
rocp_status rocp_stream_gather_window(rocp_stream* st, const rocp_tensor* x, int64_t t0, int64_t batch, int64_t nb,
                                      uint64_t seed, uint32_t first_batch_id, int sms, float* ms);
/* Profiling aid: globaltimer stamps of the persistent chain kernel, 24 per
 * (batch, stage) of the last window (phase boundaries, Gram finisher steps,
 * row solves; tools_trace.py decodes them).  enable toggles recording; out
 * may be NULL. */
rocp_status rocp_stream_chain_trace(rocp_stream* st, int enable, uint64_t* out, int64_t max,
                                    int64_t* count);
/* Elements (and useful bytes) the current window's gather moves per launch. */
rocp_status rocp_stream_window_bytes(rocp_stream* st, int64_t* useful, int64_t* elements);
/* Sampled residual of the last consume (north-star item 5): per stage
 * (temporal, then modes 1..N-1) |X_s - U Z_s^T|_F / |X_s|_F.  out[N]. */
rocp_status rocp_stream_last_residuals(rocp_stream* st, double* out);

#ifdef __cplusplus
}
#endif
#endif /* ROCP_B200_H */
