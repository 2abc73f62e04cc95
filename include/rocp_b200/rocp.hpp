// rocp.hpp -- C++ host API of the B200 ROCP hot path.
//
// Drop-in mirror of the reference's public C++ interface for the sampled-update
// path (reference = /root/reference/proj/include/rocp/*.hpp): same names,
// argument meaning, layouts and exception types, implemented over the C ABI of
// include/rocp_b200.h (librocp_b200.so).  Differences, all documented in
// DESIGN.md section 3:
//   * Matrix is a minimal column-major dense matrix (layout of Eigen::MatrixXd,
//     tensor.hpp:10) instead of Eigen.
//   * Sample indices come from the counter RNG: overloads taking Rng& draw ONE
//     64-bit seed from it per call; explicit-key overloads take (seed, batch,
//     iteration).
//   * CprandTrace / UpdateTrace are filled (cprand.cpp:34,44; rocp.cpp:125-129).
//     A traced RocpStream::consume runs the per-stage replay path
//     (update_last_mode_with / update_mode_with on the device), which is
//     bitwise equal to the untraced persistent-chain path.
//   * The free functions (init_state, update_last_mode[_with], update_mode_with,
//     update_other_modes) take host matrices by value/reference as the
//     reference does; each device primitive round-trips its operands.  They are
//     the replay/reference-compatibility surface; RocpStream is the fast path.
#pragma once

#include <cstdint>
#include <iosfwd>
#include <random>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

struct rocp_dev;
struct rocp_stream;

namespace rocp {

using Index = std::int64_t;
using Dims = std::vector<Index>;
using Rng = std::mt19937_64;  // kruskal.hpp:10

// ---- errors (errors.hpp:10-20) -------------------------------------------------
class NumericalError : public std::runtime_error {
public:
    NumericalError(const std::string& what, int sweep)
        : std::runtime_error(what + " (sweep " + std::to_string(sweep) + ")"), sweep_(sweep) {}
    int sweep() const { return sweep_; }

private:
    int sweep_;
};

// ---- column-major matrix ---------------------------------------------------------
class Matrix {
public:
    Matrix() = default;
    Matrix(Index rows, Index cols) : r_(rows), c_(cols), v_(static_cast<size_t>(rows * cols), 0.0) {}
    static Matrix Zero(Index rows, Index cols) { return Matrix(rows, cols); }
    static Matrix Ones(Index rows, Index cols) {
        Matrix m(rows, cols);
        for (double& x : m.v_) x = 1.0;
        return m;
    }
    static Matrix Identity(Index n, Index m) {
        Matrix out(n, m);
        for (Index i = 0; i < std::min(n, m); ++i) out(i, i) = 1.0;
        return out;
    }
    Index rows() const { return r_; }
    Index cols() const { return c_; }
    Index size() const { return r_ * c_; }
    double* data() { return v_.data(); }
    const double* data() const { return v_.data(); }
    double& operator()(Index i, Index j) { return v_[static_cast<size_t>(i + j * r_)]; }
    double operator()(Index i, Index j) const { return v_[static_cast<size_t>(i + j * r_)]; }
    bool operator==(const Matrix& o) const { return r_ == o.r_ && c_ == o.c_ && v_ == o.v_; }
    bool allFinite() const;

private:
    Index r_ = 0, c_ = 0;
    std::vector<double> v_;
};

// ---- dense tensor (tensor.hpp:17-49): host values + lazily uploaded copy ----------
class DenseTensor {
public:
    DenseTensor() = default;
    explicit DenseTensor(Dims dims);
    DenseTensor(Dims dims, std::vector<double> data);
    const Dims& dims() const { return dims_; }
    int order() const { return static_cast<int>(dims_.size()); }
    Index size() const { return static_cast<Index>(data_.size()); }
    double* data() { return data_.data(); }
    const double* data() const { return data_.data(); }
    std::vector<double>& values() { return data_; }
    const std::vector<double>& values() const { return data_; }
    double operator[](Index flat) const { return data_[static_cast<size_t>(flat)]; }
    double& operator[](Index flat) { return data_[static_cast<size_t>(flat)]; }

private:
    Dims dims_;
    std::vector<double> data_;
};

Index element_count(const Dims& dims);
Index codomain_size(const Dims& dims, int mode);
Index linear_index(std::span<const Index> multi_index, const Dims& dims, int mode);
std::vector<Index> decode_index(Index j, const Dims& dims, int mode);

// ---- model (kruskal.hpp:13-39) ---------------------------------------------------
struct KruskalModel {
    int rank = 0;
    std::vector<Matrix> factors;
    int order() const { return static_cast<int>(factors.size()); }
    Dims dims() const;
};

// Gaussian initial model, i.i.d. N(0,1) in (i outer, r inner) order with
// std::normal_distribution -- the reference's random_model (kruskal.cpp:29-42).
KruskalModel random_model(const Dims& dims, int rank, Rng& rng);
std::vector<Matrix> factors_excluding(const KruskalModel& m, int mode);
double model_fitness(const DenseTensor& x, const KruskalModel& m);

// ---- sampling (sampling.hpp:14-48) -----------------------------------------------
struct SampleIndexSet {
    int mode = 0;
    Dims dims;
    std::vector<Index> rows;     // 1-based column indices
    std::vector<Index> decoded;  // s x (N-1), row-major, 1-based
    Index count() const { return static_cast<Index>(rows.size()); }
    int n_other() const { return static_cast<int>(dims.size()) - 1; }
    Index decoded_at(Index c, int k) const { return decoded[static_cast<size_t>(c * n_other() + k)]; }
    static SampleIndexSet from_rows(const Dims& dims, int mode, std::vector<Index> rows);
    static SampleIndexSet all_columns(const Dims& dims, int mode);
};

struct CounterKey {
    std::uint64_t seed = 0;
    std::uint32_t batch = 0, iteration = 0;
};

Index auto_sample_count(int rank);
SampleIndexSet draw_samples(const Dims& dims, int mode, Index s, CounterKey key);
SampleIndexSet draw_samples(const Dims& dims, int mode, Index s, Rng& rng);
Matrix sample_unfolding(const DenseTensor& t, const SampleIndexSet& idx);
Matrix sampled_khatri_rao(const SampleIndexSet& idx, std::span<const Matrix> factors);

// ---- solve (solve.hpp:8-24) ---------------------------------------------------------
struct SolveInfo {
    bool regularized = false;
    bool underdetermined = false;
};
inline constexpr double kGramConditionLimit = 1e12;
Matrix solve_gram(const Matrix& gram, const Matrix& rhs, SolveInfo* info = nullptr);
Matrix solve_sampled_ls(const Matrix& z_s, const Matrix& x_s, SolveInfo* info = nullptr);

// ---- cprand (cprand.hpp:10-37) ----------------------------------------------------
struct CprandOptions {
    Index samples = 0;
    double tol = 1e-4;
    int max_iters = 100;
};
struct InitResult {
    KruskalModel model;
    std::vector<Matrix> best_sampled_kr;
    std::vector<Matrix> best_sampled_factors;
    double best_fitness = 0.0;
    int iterations = 0;
    bool regularized = false;
    std::uint64_t seed = 0;  // counter-RNG key the draws used
};
struct CprandTrace {
    std::vector<std::vector<SampleIndexSet>> sweeps;  // [sweep][mode-1] (cprand.hpp:28-31)
};
InitResult cprand_decompose(const DenseTensor& x, int rank, const CprandOptions& opts, Rng& rng,
                            CprandTrace* trace = nullptr);
// Explicit form: initial model and counter seed given.
InitResult cprand_decompose(const DenseTensor& x, const KruskalModel& initial, const CprandOptions& opts,
                            std::uint64_t seed, CprandTrace* trace = nullptr);

// ---- online stream (rocp.hpp:15-117) ---------------------------------------------
struct ComplementaryState {
    std::vector<Matrix> p;
    std::vector<Matrix> q;
    Index t_len = 0;
    Index sample_count = 0;
    Dims dims_head;
    std::size_t byte_size() const;
};
struct RocpConfig {
    bool literal_init = false;
};
struct UpdateTrace {
    std::vector<SampleIndexSet> mode_idx;  // n = 1..N-1 (rocp.hpp:56-61)
    std::vector<Matrix> mode_z;            // Z_s(n)^new, s x R
    std::vector<Matrix> mode_x;            // X_s(n)^new, I_n x s
};

// init_state (rocp.hpp:35, rocp.cpp:45-69): Q(n) = Z_best(n)^T Z_best(n),
// P(n) = U_best(n) Q(n) (or U_best(n) with literal_init), on the device.
ComplementaryState init_state(const InitResult& init, Index s, const RocpConfig& cfg = {});

// Temporal-mode solve for one batch (rocp.hpp:38-53, rocp.cpp:71-94).
struct LastModeUpdate {
    Matrix u_new;        // I_N,new x R
    SampleIndexSet idx;  // the draw used
    Matrix z_s;          // s x R
    bool regularized = false;
};
LastModeUpdate update_last_mode_with(const KruskalModel& model, const DenseTensor& x_new, SampleIndexSet idx);
// Counter-RNG draw keyed by `key` over x_new's temporal co-domain; the Rng&
// form draws one 64-bit seed from rng (key = {seed, 0, 0}).
LastModeUpdate update_last_mode(const KruskalModel& model, const DenseTensor& x_new, Index s, CounterKey key);
LastModeUpdate update_last_mode(const KruskalModel& model, const DenseTensor& x_new, Index s, Rng& rng);

// One non-temporal mode against an explicit index set (rocp.hpp:63-75,
// rocp.cpp:96-113): P += X_s Z_new, Q += Z_new^T Z_new, U = P Q^-1.
struct ModeUpdate {
    Matrix z_new;  // s x R
    Matrix x_s;    // I_n x s
    bool regularized = false;
};
ModeUpdate update_mode_with(ComplementaryState& state, KruskalModel& model, const DenseTensor& x_new,
                            const Matrix& u_new, const SampleIndexSet& idx);
// Modes 1..N-1, Gauss-Seidel (rocp.hpp:77-81, rocp.cpp:115-131).  The draws of
// mode n use `key` (the same key RocpStream::consume(x, seed, batch) uses for
// all N draws of a batch, so update_last_mode + update_other_modes with
// key = {seed, batch, 0} replays consume bit for bit); the Rng& form draws one
// seed from rng.
void update_other_modes(ComplementaryState& state, KruskalModel& model, const DenseTensor& x_new, const Matrix& u_new,
                        CounterKey key, UpdateTrace* trace = nullptr);
void update_other_modes(ComplementaryState& state, KruskalModel& model, const DenseTensor& x_new, const Matrix& u_new,
                        Rng& rng, UpdateTrace* trace = nullptr);

class RocpStream {
public:
    // t_capacity is an initial reservation only: the device temporal factor
    // grows geometrically as in rocp.cpp:152-155, so streams of any length run.
    RocpStream(InitResult init, Index s, RocpConfig cfg = {}, Index t_capacity = 0);
    ~RocpStream();
    RocpStream(const RocpStream&) = delete;
    RocpStream& operator=(const RocpStream&) = delete;

    void consume(const DenseTensor& x_new, Rng& rng, UpdateTrace* trace = nullptr);
    void consume(const DenseTensor& x_new, std::uint64_t seed, std::uint32_t batch_id,
                 UpdateTrace* trace = nullptr);
    KruskalModel model() const;
    ComplementaryState state() const;
    Index t_len() const;
    bool regularized() const;
    double last_residual() const;  // sampled residual of the last temporal solve

private:
    rocp_stream* h_ = nullptr;
    int order_ = 0, rank_ = 0;
    Dims head_;
    Index s_ = 0;
    std::uint32_t next_batch_ = 1;
};

KruskalModel rocp_run(const DenseTensor& x_init, std::span<const DenseTensor> batches, int rank,
                      const CprandOptions& init_opts, Rng& rng, const RocpConfig& cfg = {});

// ---- binary records (tensor_io.hpp:10-27, rocp.hpp:116-117) ------------------------
// Byte format of the reference: "ROCP", version 1, u32le order, u64le extents,
// little-endian binary64 values first index fastest (matrices: order-2,
// column-major).  std::runtime_error on open / format / truncation errors.
void write_tensor(const DenseTensor& t, std::ostream& out);
DenseTensor read_tensor(std::istream& in);
void write_tensor_file(const DenseTensor& t, const std::string& path);
DenseTensor read_tensor_file(const std::string& path);
void write_matrix(const Matrix& m, std::ostream& out);
Matrix read_matrix(std::istream& in);
void put_u64le(std::ostream& out, std::uint64_t v);
std::uint64_t get_u64le(std::istream& in);
// ComplementaryState: P records, Q records, u64le t_len
void save_state(const ComplementaryState& state, std::ostream& out);
ComplementaryState load_state(std::istream& in);

// Device selection for this thread's calls (default: device 0, created lazily).
void set_device(int device);
int current_device();  // the calling thread's device ordinal (set_device; default 0)
rocp_dev* device_handle();

}  // namespace rocp
