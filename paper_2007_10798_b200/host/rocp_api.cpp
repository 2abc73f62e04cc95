// rocp_api.cpp -- C++ host API (include/rocp_b200/rocp.hpp) over the C ABI.
// Every call goes to librocp_b200.so (sm_100a kernels); there is no CPU
// compute path here apart from argument validation, layout bookkeeping and the
// reference's own host-side random_model and binary record IO.

#include "../../include/rocp_b200/rocp.hpp"

#include "../../include/rocp_b200.h"

#include <bit>
#include <cstring>
#include <fstream>
#include <istream>
#include <ostream>

#include <cmath>
#include <memory>

namespace rocp {

namespace {

struct DevHolder {
    int device = 0;
    rocp_dev* h = nullptr;
    ~DevHolder() {
        if (h) rocp_destroy(h);
    }
};
thread_local DevHolder g_dev;

void raise(rocp_dev* d, rocp_status st, int sweep = 0) {
    const std::string msg = rocp_last_error(d);
    if (st == ROCP_E_DOMAIN) throw std::domain_error(msg);
    if (st == ROCP_E_NUMERICAL) throw NumericalError(msg, sweep);
    if (st == ROCP_E_IO) throw std::runtime_error(msg);  // tensor_io.cpp / rocp.cpp record errors
    throw std::runtime_error("rocp_b200 status " + std::to_string(int(st)) + ": " + msg);
}

void check(rocp_status st, int sweep = 0) {
    if (st != ROCP_OK) raise(device_handle(), st, sweep);
}

void check_head_dims(const Dims& head, const DenseTensor& x_new) {  // rocp.cpp:14-21
    const Dims& d = x_new.dims();
    if (d.size() != head.size() + 1) throw std::domain_error("batch order does not match stream order");
    for (size_t k = 0; k < head.size(); ++k)
        if (d[k] != head[k]) throw std::domain_error("batch head extents do not match stream");
}

void check_mode(const Dims& dims, int mode) {  // tensor.cpp:19-23
    if (mode < 1 || mode > static_cast<int>(dims.size()))
        throw std::domain_error("mode " + std::to_string(mode) + " out of range for order " +
                                std::to_string(dims.size()));
}

// RAII device tensor uploaded from a host DenseTensor.
struct DevTensor {
    rocp_tensor* t = nullptr;
    explicit DevTensor(const DenseTensor& x) {
        check(rocp_tensor_create(device_handle(), x.dims().data(), x.order(), x.data(), &t));
    }
    ~DevTensor() {
        if (t) rocp_tensor_free(t);
    }
};

std::vector<const double*> ptrs(const std::vector<Matrix>& ms) {
    std::vector<const double*> p;
    for (const Matrix& m : ms) p.push_back(m.data());
    return p;
}

}  // namespace

void set_device(int device) {
    if (g_dev.h && g_dev.device != device) {
        rocp_destroy(g_dev.h);
        g_dev.h = nullptr;
    }
    g_dev.device = device;
}

int current_device() { return g_dev.device; }

rocp_dev* device_handle() {
    if (!g_dev.h) {
        rocp_dev* d = nullptr;
        if (rocp_create(g_dev.device, 1, 0, nullptr, &d) != ROCP_OK)
            throw std::runtime_error("rocp_b200: cannot open CUDA device " + std::to_string(g_dev.device));
        g_dev.h = d;
    }
    return g_dev.h;
}

bool Matrix::allFinite() const {
    for (double x : v_)
        if (!std::isfinite(x)) return false;
    return true;
}

// ---- tensor -------------------------------------------------------------------------
Index element_count(const Dims& dims) {
    Index n = 1;
    for (Index d : dims) n *= d;
    return n;
}

DenseTensor::DenseTensor(Dims dims) : dims_(std::move(dims)) {
    if (dims_.size() < 2) throw std::domain_error("tensor order must be at least 2");
    for (Index d : dims_)
        if (d < 1) throw std::domain_error("tensor extents must be positive");
    data_.assign(static_cast<size_t>(element_count(dims_)), 0.0);
}

DenseTensor::DenseTensor(Dims dims, std::vector<double> data) : dims_(std::move(dims)), data_(std::move(data)) {
    if (dims_.size() < 2) throw std::domain_error("tensor order must be at least 2");
    for (Index d : dims_)
        if (d < 1) throw std::domain_error("tensor extents must be positive");
    if (static_cast<Index>(data_.size()) != element_count(dims_))
        throw std::domain_error("data length does not match product of extents");
}

Index codomain_size(const Dims& dims, int mode) {
    check_mode(dims, mode);
    return element_count(dims) / dims[static_cast<size_t>(mode - 1)];
}

Index linear_index(std::span<const Index> multi, const Dims& dims, int mode) {
    check_mode(dims, mode);
    if (multi.size() != dims.size() - 1)
        throw std::domain_error("multi-index must cover all modes except the unfolding mode");
    Index j = 0, stride = 1;
    size_t pos = 0;
    for (size_t k = 0; k < dims.size(); ++k) {
        if (static_cast<int>(k) + 1 == mode) continue;
        const Index i = multi[pos++];
        if (i < 1 || i > dims[k]) throw std::domain_error("multi-index out of range");
        j += (i - 1) * stride;
        stride *= dims[k];
    }
    return j + 1;
}

std::vector<Index> decode_index(Index j, const Dims& dims, int mode) {
    std::vector<Index> out(dims.size() - 1);
    check(rocp_decode_rows(device_handle(), dims.data(), static_cast<int>(dims.size()), mode, &j, 1, out.data()));
    return out;
}

// ---- model --------------------------------------------------------------------------
Dims KruskalModel::dims() const {
    Dims d;
    for (const Matrix& f : factors) d.push_back(f.rows());
    return d;
}

KruskalModel random_model(const Dims& dims, int rank, Rng& rng) {
    KruskalModel m;
    m.rank = rank;
    std::normal_distribution<double> gauss(0.0, 1.0);
    for (Index d : dims) {
        Matrix f(d, rank);
        for (Index i = 0; i < d; ++i)  // i outer, r inner, one distribution across factors
            for (int r = 0; r < rank; ++r) f(i, r) = gauss(rng);
        m.factors.push_back(std::move(f));
    }
    return m;
}

std::vector<Matrix> factors_excluding(const KruskalModel& m, int mode) {
    if (mode < 1 || mode > m.order()) throw std::domain_error("mode out of range");
    std::vector<Matrix> out;
    for (int k = m.order(); k >= 1; --k)
        if (k != mode) out.push_back(m.factors[static_cast<size_t>(k - 1)]);
    return out;
}

double model_fitness(const DenseTensor& x, const KruskalModel& m) {
    if (m.dims() != x.dims()) throw std::domain_error("dims order does not match model");
    DevTensor t(x);
    const auto p = ptrs(m.factors);
    double fit = 0.0;
    check(rocp_model_fitness(device_handle(), t.t, p.data(), m.rank, &fit));
    return fit;
}

// ---- sampling -----------------------------------------------------------------------
SampleIndexSet SampleIndexSet::from_rows(const Dims& dims, int mode, std::vector<Index> rows) {
    SampleIndexSet idx;
    idx.mode = mode;
    idx.dims = dims;
    idx.decoded.assign(rows.size() * (dims.size() - 1), 0);
    if (!rows.empty())
        check(rocp_decode_rows(device_handle(), dims.data(), static_cast<int>(dims.size()), mode, rows.data(),
                               static_cast<Index>(rows.size()), idx.decoded.data()));
    idx.rows = std::move(rows);
    return idx;
}

SampleIndexSet SampleIndexSet::all_columns(const Dims& dims, int mode) {
    const Index co = codomain_size(dims, mode);
    std::vector<Index> rows(static_cast<size_t>(co));
    for (Index j = 0; j < co; ++j) rows[static_cast<size_t>(j)] = j + 1;
    return from_rows(dims, mode, std::move(rows));
}

Index auto_sample_count(int rank) {  // sampling.cpp:40-45
    if (rank < 1) throw std::domain_error("rank must be positive");
    const double s = 10.0 * rank * std::log(static_cast<double>(rank));
    return std::max<Index>(rank, static_cast<Index>(std::ceil(s)));
}

SampleIndexSet draw_samples(const Dims& dims, int mode, Index s, CounterKey key) {
    SampleIndexSet idx;
    idx.mode = mode;
    idx.dims = dims;
    idx.rows.assign(static_cast<size_t>(std::max<Index>(s, 0)), 0);
    idx.decoded.assign(static_cast<size_t>(std::max<Index>(s, 0)) * (dims.size() - 1), 0);
    check(rocp_draw_samples(device_handle(), dims.data(), static_cast<int>(dims.size()), mode, s, key.seed,
                            key.batch, key.iteration, idx.rows.data(), idx.decoded.data()));
    return idx;
}

SampleIndexSet draw_samples(const Dims& dims, int mode, Index s, Rng& rng) {
    return draw_samples(dims, mode, s, CounterKey{rng(), 0, 0});
}

Matrix sample_unfolding(const DenseTensor& t, const SampleIndexSet& idx) {
    if (t.dims() != idx.dims) throw std::domain_error("sample_unfolding: index set drawn against different dims");
    Matrix out(t.dims()[static_cast<size_t>(idx.mode - 1)], idx.count());
    DevTensor d(t);
    check(rocp_sample_unfolding(device_handle(), d.t, idx.mode, idx.rows.data(), idx.count(), out.data()));
    return out;
}

Matrix sampled_khatri_rao(const SampleIndexSet& idx, std::span<const Matrix> factors) {
    if (static_cast<int>(factors.size()) != idx.n_other())
        throw std::domain_error("sampled_khatri_rao: factor count mismatch");
    const Index rank = factors.empty() ? 0 : factors[0].cols();
    for (const Matrix& f : factors)
        if (f.cols() != rank) throw std::domain_error("sampled_khatri_rao: factor column counts differ");
    std::vector<const double*> p;
    std::vector<Index> frows;
    for (const Matrix& f : factors) {
        p.push_back(f.data());
        frows.push_back(f.rows());
    }
    Matrix z(idx.count(), rank);
    check(rocp_sampled_khatri_rao(device_handle(), idx.decoded.data(), idx.count(), idx.n_other(), p.data(),
                                  frows.data(), static_cast<int>(rank), z.data()));
    return z;
}

// ---- solve --------------------------------------------------------------------------
Matrix solve_gram(const Matrix& gram, const Matrix& rhs, SolveInfo* info) {
    if (gram.rows() != gram.cols()) throw std::domain_error("solve_gram: gram matrix must be square");
    if (rhs.cols() != gram.rows()) throw std::domain_error("solve_gram: rhs column count must match gram size");
    Matrix out(rhs.rows(), rhs.cols());
    int reg = 0;
    check(rocp_solve_gram(device_handle(), gram.data(), rhs.data(), rhs.rows(), static_cast<int>(gram.rows()),
                          out.data(), &reg));
    if (info && reg) info->regularized = true;
    return out;
}

Matrix solve_sampled_ls(const Matrix& z_s, const Matrix& x_s, SolveInfo* info) {
    if (x_s.cols() != z_s.rows()) throw std::domain_error("solve_sampled_ls: sample counts of z_s and x_s differ");
    Matrix out(x_s.rows(), z_s.cols());
    int reg = 0, und = 0;
    check(rocp_solve_sampled_ls(device_handle(), z_s.data(), x_s.data(), z_s.rows(), x_s.rows(),
                                static_cast<int>(z_s.cols()), out.data(), &reg, &und));
    if (info) {
        if (reg) info->regularized = true;
        if (und) info->underdetermined = true;
    }
    return out;
}

// ---- cprand -------------------------------------------------------------------------
InitResult cprand_decompose(const DenseTensor& x, const KruskalModel& initial, const CprandOptions& opts,
                            std::uint64_t seed, CprandTrace* trace) {
    if (initial.rank < 1) throw std::domain_error("cprand_decompose: rank must be positive");
    const int N = x.order();
    const Index s = opts.samples > 0 ? opts.samples : auto_sample_count(initial.rank);
    InitResult res;
    res.model = initial;
    res.best_sampled_kr.assign(static_cast<size_t>(N - 1), Matrix(s, initial.rank));
    std::vector<double*> f, kr;
    for (Matrix& m : res.model.factors) f.push_back(m.data());
    for (Matrix& m : res.best_sampled_kr) kr.push_back(m.data());
    DevTensor t(x);
    int iters = 0, reg = 0, err_sweep = 0;
    const rocp_status st = rocp_cprand(device_handle(), t.t, initial.rank, opts.samples, opts.tol, opts.max_iters,
                                       seed, f.data(), kr.data(), &res.best_fitness, &iters, &reg, &err_sweep,
                                       nullptr);
    if (st != ROCP_OK) raise(device_handle(), st, err_sweep);
    res.iterations = iters;
    res.regularized = reg != 0;
    res.seed = seed;
    for (int n = 0; n + 1 < N; ++n) res.best_sampled_factors.push_back(res.model.factors[static_cast<size_t>(n)]);
    if (trace) {  // cprand.cpp:34,44: the index sets of every sweep, [sweep][mode-1]
        // The counter RNG makes them a pure function of (seed, sweep, mode): sweep k
        // draws with key (seed, batch 0, iteration k), so they are
        // regenerated on the device rather than copied out of the sweep loop.
        for (int sweep = 1; sweep <= iters; ++sweep) {
            trace->sweeps.emplace_back();
            for (int n = 1; n <= N; ++n)
                trace->sweeps.back().push_back(
                    draw_samples(x.dims(), n, s, CounterKey{seed, 0, static_cast<std::uint32_t>(sweep)}));
        }
    }
    return res;
}

InitResult cprand_decompose(const DenseTensor& x, int rank, const CprandOptions& opts, Rng& rng,
                            CprandTrace* trace) {
    if (rank < 1) throw std::domain_error("cprand_decompose: rank must be positive");
    if (opts.max_iters < 1) throw std::domain_error("cprand_decompose: need at least one sweep");
    const KruskalModel init = random_model(x.dims(), rank, rng);  // cprand.cpp:25
    return cprand_decompose(x, init, opts, rng(), trace);
}

// ---- stream -------------------------------------------------------------------------
std::size_t ComplementaryState::byte_size() const {
    std::size_t bytes = sizeof(*this) + dims_head.size() * sizeof(Index);
    for (const Matrix& m : p) bytes += static_cast<std::size_t>(m.size()) * sizeof(double);
    for (const Matrix& m : q) bytes += static_cast<std::size_t>(m.size()) * sizeof(double);
    return bytes;
}

RocpStream::RocpStream(InitResult init, Index s, RocpConfig cfg, Index t_capacity) {
    order_ = init.model.order();
    rank_ = init.model.rank;
    s_ = s;
    for (int n = 0; n + 1 < order_; ++n) head_.push_back(init.model.factors[static_cast<size_t>(n)].rows());
    if (static_cast<int>(init.best_sampled_kr.size()) != order_ - 1)
        throw std::domain_error("init_state: expected one sampled system per non-temporal mode");
    for (const Matrix& z : init.best_sampled_kr)
        if (z.rows() != s) throw std::domain_error("init_state: sampled Khatri-Rao row count differs from s");
    const Index t_init = init.model.factors.back().rows();
    const auto f = ptrs(init.model.factors);
    const auto kr = ptrs(init.best_sampled_kr);
    check(rocp_stream_create(device_handle(), order_, head_.data(), rank_, s, cfg.literal_init ? 1 : 0, f.data(),
                             t_init, kr.data(), init.regularized ? 1 : 0, std::max<Index>(t_capacity, 4 * t_init + 64),
                             &h_));
}

RocpStream::~RocpStream() {
    if (h_) rocp_stream_free(h_);
}

void RocpStream::consume(const DenseTensor& x_new, std::uint64_t seed, std::uint32_t batch_id, UpdateTrace* trace) {
    check_head_dims(head_, x_new);  // rocp.cpp:145
    if (!trace) {
        check(rocp_stream_consume_host(h_, x_new.data(), x_new.dims().back(), seed, batch_id));
        next_batch_ = batch_id + 1;
        return;
    }
    // Traced: the same batch through the per-stage replay seams (rocp.cpp:144-160 step by
    // step), which are bitwise equal to the persistent chain, recording each mode's
    // sampled system (rocp.cpp:125-129).
    const Index B = x_new.dims().back();
    const Dims& dims = x_new.dims();
    DevTensor t(x_new);
    const SampleIndexSet it = draw_samples(dims, order_, s_, CounterKey{seed, batch_id, 0});
    Matrix u_new(B, rank_);
    int reg = 0;
    check(rocp_stream_update_last_mode_with(h_, t.t, it.rows.data(), s_, u_new.data(), nullptr, &reg));
    if (reg) check(rocp_stream_mark_regularized(h_));  // rocp.cpp:150
    check(rocp_stream_append_temporal(h_, u_new.data(), B));
    for (int n = 1; n < order_; ++n) {
        SampleIndexSet idx = draw_samples(dims, n, s_, CounterKey{seed, batch_id, 0});
        Matrix z(s_, rank_), xs(dims[static_cast<size_t>(n - 1)], s_);
        int r2 = 0;
        check(rocp_stream_update_mode_with(h_, t.t, u_new.data(), n, idx.rows.data(), s_, z.data(), xs.data(), &r2));
        trace->mode_idx.push_back(std::move(idx));
        trace->mode_z.push_back(std::move(z));
        trace->mode_x.push_back(std::move(xs));
    }
    check(rocp_stream_finish_batch(h_, B));
    next_batch_ = batch_id + 1;
}

void RocpStream::consume(const DenseTensor& x_new, Rng& rng, UpdateTrace* trace) {
    consume(x_new, rng(), next_batch_, trace);
}

KruskalModel RocpStream::model() const {
    KruskalModel m;
    m.rank = rank_;
    for (int n = 1; n < order_; ++n) {
        Matrix u(head_[static_cast<size_t>(n - 1)], rank_);
        check(rocp_stream_get(h_, 0, n, u.data()));
        m.factors.push_back(std::move(u));
    }
    Matrix t(rocp_stream_t_len(h_), rank_);
    check(rocp_stream_get(h_, 3, 0, t.data()));
    m.factors.push_back(std::move(t));
    return m;
}

ComplementaryState RocpStream::state() const {
    ComplementaryState st;
    for (int n = 1; n < order_; ++n) {
        Matrix p(head_[static_cast<size_t>(n - 1)], rank_), q(rank_, rank_);
        check(rocp_stream_get(h_, 1, n, p.data()));
        check(rocp_stream_get(h_, 2, n, q.data()));
        st.p.push_back(std::move(p));
        st.q.push_back(std::move(q));
    }
    st.t_len = rocp_stream_t_len(h_);
    st.sample_count = s_;
    st.dims_head = head_;
    return st;
}

Index RocpStream::t_len() const { return rocp_stream_t_len(h_); }
bool RocpStream::regularized() const { return rocp_stream_regularized(h_) != 0; }

double RocpStream::last_residual() const {
    std::vector<double> r(static_cast<size_t>(order_));
    check(rocp_stream_last_residuals(h_, r.data()));
    return r[0];
}

// ---- free functions of the online update (rocp.hpp:35-81) ---------------------------
ComplementaryState init_state(const InitResult& init, Index s, const RocpConfig& cfg) {  // rocp.cpp:45-69
    const int N = init.model.order();
    if (static_cast<int>(init.best_sampled_kr.size()) != N - 1 ||
        static_cast<int>(init.best_sampled_factors.size()) != N - 1)
        throw std::domain_error("init_state: expected one sampled system per non-temporal mode");
    Dims head;
    for (int n = 0; n + 1 < N; ++n) {
        const Matrix& z = init.best_sampled_kr[static_cast<size_t>(n)];
        const Matrix& u = init.best_sampled_factors[static_cast<size_t>(n)];
        if (z.rows() != s) throw std::domain_error("init_state: sampled Khatri-Rao row count differs from s");
        if (z.cols() != u.cols()) throw std::domain_error("init_state: rank mismatch");
        head.push_back(u.rows());
    }
    const int R = init.model.rank;
    // Q = Z^T Z and P = U Q in the canonical order of the stream's own init
    // (k_gram / k_mul_uq), through a transient device stream.
    std::vector<const double*> f = ptrs(init.best_sampled_factors);
    f.push_back(init.model.factors.back().data());
    const auto kr = ptrs(init.best_sampled_kr);
    const Index t_init = init.model.factors.back().rows();
    rocp_stream* h = nullptr;
    check(rocp_stream_create(device_handle(), N, head.data(), R, s, cfg.literal_init ? 1 : 0, f.data(), t_init,
                             kr.data(), init.regularized ? 1 : 0, t_init, &h));
    std::unique_ptr<rocp_stream, void (*)(rocp_stream*)> guard(h, rocp_stream_free);
    ComplementaryState st;
    st.sample_count = s;
    st.t_len = t_init;
    st.dims_head = head;
    for (int n = 1; n < N; ++n) {
        Matrix p(head[static_cast<size_t>(n - 1)], R), q(R, R);
        check(rocp_stream_get(h, 1, n, p.data()));
        check(rocp_stream_get(h, 2, n, q.data()));
        st.p.push_back(std::move(p));
        st.q.push_back(std::move(q));
    }
    return st;
}

LastModeUpdate update_last_mode_with(const KruskalModel& model, const DenseTensor& x_new,
                                     SampleIndexSet idx) {  // rocp.cpp:71-84
    const int N = model.order();
    if (idx.mode != N) throw std::domain_error("update_last_mode: index set must be over the temporal mode");
    LastModeUpdate upd;
    upd.z_s = sampled_khatri_rao(idx, factors_excluding(model, N));
    const Matrix x_s = sample_unfolding(x_new, idx);
    SolveInfo info;
    upd.u_new = solve_sampled_ls(upd.z_s, x_s, &info);
    upd.regularized = info.regularized;
    upd.idx = std::move(idx);
    return upd;
}

LastModeUpdate update_last_mode(const KruskalModel& model, const DenseTensor& x_new, Index s, CounterKey key) {
    Dims head = model.dims();  // rocp.cpp:86-94
    head.pop_back();
    check_head_dims(head, x_new);
    return update_last_mode_with(model, x_new, draw_samples(x_new.dims(), model.order(), s, key));
}

LastModeUpdate update_last_mode(const KruskalModel& model, const DenseTensor& x_new, Index s, Rng& rng) {
    return update_last_mode(model, x_new, s, CounterKey{rng(), 0, 0});
}

ModeUpdate update_mode_with(ComplementaryState& state, KruskalModel& model, const DenseTensor& x_new,
                            const Matrix& u_new, const SampleIndexSet& idx) {  // rocp.cpp:96-113
    const int n = idx.mode;
    if (n < 1 || n >= model.order())
        throw std::domain_error("update_mode_with: index set must be over a non-temporal mode");
    if (static_cast<int>(state.p.size()) != model.order() - 1 || static_cast<int>(state.q.size()) != model.order() - 1)
        throw std::domain_error("update_mode_with: state does not match the model order");
    // slab_factors_excluding (rocp.cpp:25-34): u_new first, then modes N-1..1 without n
    std::vector<Matrix> fs;
    fs.push_back(u_new);
    for (int k = model.order() - 1; k >= 1; --k)
        if (k != n) fs.push_back(model.factors[static_cast<size_t>(k - 1)]);
    ModeUpdate upd;
    upd.z_new = sampled_khatri_rao(idx, fs);
    upd.x_s = sample_unfolding(x_new, idx);
    const int R = static_cast<int>(upd.z_new.cols());
    Matrix& p = state.p[static_cast<size_t>(n - 1)];
    Matrix& q = state.q[static_cast<size_t>(n - 1)];
    if (p.rows() != upd.x_s.rows() || p.cols() != R || q.rows() != R || q.cols() != R)
        throw std::domain_error("update_mode_with: state shapes do not match the sampled system");
    // P + (X_s Z) and Q + (Z^T Z), each increment in the canonical chunked order on
    // the device, then one IEEE add per entry -- the stream's accumulation
    Matrix inc(p.rows(), R), g(R, R);
    check(rocp_contract(device_handle(), upd.x_s.data(), upd.x_s.rows(), upd.x_s.cols(), upd.z_new.data(), R,
                        inc.data()));
    check(rocp_gram(device_handle(), upd.z_new.data(), upd.z_new.rows(), R, g.data()));
    for (Index e = 0; e < p.size(); ++e) p.data()[e] = p.data()[e] + inc.data()[e];
    for (Index e = 0; e < q.size(); ++e) q.data()[e] = q.data()[e] + g.data()[e];
    SolveInfo info;
    model.factors[static_cast<size_t>(n - 1)] = solve_gram(q, p, &info);
    upd.regularized = info.regularized;
    return upd;
}

void update_other_modes(ComplementaryState& state, KruskalModel& model, const DenseTensor& x_new, const Matrix& u_new,
                        CounterKey key, UpdateTrace* trace) {  // rocp.cpp:115-131
    check_head_dims(state.dims_head, x_new);
    if (u_new.rows() != x_new.dims().back())
        throw std::domain_error("update_other_modes: u_new rows must equal the batch size");
    for (int n = 1; n < model.order(); ++n) {
        SampleIndexSet idx = draw_samples(x_new.dims(), n, state.sample_count, key);
        ModeUpdate upd = update_mode_with(state, model, x_new, u_new, idx);
        if (trace) {
            trace->mode_idx.push_back(std::move(idx));
            trace->mode_z.push_back(std::move(upd.z_new));
            trace->mode_x.push_back(std::move(upd.x_s));
        }
    }
}

void update_other_modes(ComplementaryState& state, KruskalModel& model, const DenseTensor& x_new, const Matrix& u_new,
                        Rng& rng, UpdateTrace* trace) {
    update_other_modes(state, model, x_new, u_new, CounterKey{rng(), 0, 0}, trace);
}

KruskalModel rocp_run(const DenseTensor& x_init, std::span<const DenseTensor> batches, int rank,
                      const CprandOptions& init_opts, Rng& rng, const RocpConfig& cfg) {
    InitResult init = cprand_decompose(x_init, rank, init_opts, rng);  // rocp.cpp:170-178
    const Index s = init_opts.samples > 0 ? init_opts.samples : auto_sample_count(rank);
    Index total = x_init.dims().back();
    for (const DenseTensor& b : batches) total += b.dims().back();
    RocpStream stream(std::move(init), s, cfg, total);
    for (const DenseTensor& b : batches) stream.consume(b, rng);
    return stream.model();
}

// ---- binary records (tensor_io.cpp:12-101, rocp.cpp:180-211 semantics) ----------
namespace {

void put_le(std::ostream& out, std::uint64_t v, int bytes) {
    char b[8];
    for (int i = 0; i < bytes; ++i) b[i] = static_cast<char>((v >> (8 * i)) & 0xffu);
    out.write(b, bytes);
}

std::uint64_t get_le(std::istream& in, int bytes) {
    unsigned char b[8] = {};
    in.read(reinterpret_cast<char*>(b), bytes);
    if (!in) throw std::runtime_error("tensor record truncated");
    std::uint64_t v = 0;
    for (int i = bytes - 1; i >= 0; --i) v = (v << 8) | b[i];
    return v;
}

}  // namespace

void put_u64le(std::ostream& out, std::uint64_t v) { put_le(out, v, 8); }
std::uint64_t get_u64le(std::istream& in) { return get_le(in, 8); }

void write_tensor(const DenseTensor& t, std::ostream& out) {
    out.write("ROCP", 4);
    out.put(char(1));
    put_le(out, static_cast<std::uint64_t>(t.order()), 4);
    for (Index d : t.dims()) put_le(out, static_cast<std::uint64_t>(d), 8);
    for (Index i = 0; i < t.size(); ++i) put_le(out, std::bit_cast<std::uint64_t>(t[i]), 8);
    if (!out) throw std::runtime_error("tensor write failed");
}

DenseTensor read_tensor(std::istream& in) {
    char magic[4] = {};
    in.read(magic, 4);
    if (!in || std::memcmp(magic, "ROCP", 4) != 0) throw std::runtime_error("bad tensor magic");
    if (in.get() != 1) throw std::runtime_error("unsupported tensor format version");
    const std::uint64_t order = get_le(in, 4);
    if (order < 2 || order > 64) throw std::runtime_error("implausible tensor order");
    Dims dims(order);
    for (Index& d : dims) d = static_cast<Index>(get_le(in, 8));
    std::vector<double> v(static_cast<size_t>(element_count(dims)));
    for (double& x : v) x = std::bit_cast<double>(get_le(in, 8));
    return DenseTensor(std::move(dims), std::move(v));
}

void write_tensor_file(const DenseTensor& t, const std::string& path) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw std::runtime_error("cannot open " + path + " for writing");
    write_tensor(t, out);
}

DenseTensor read_tensor_file(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw std::runtime_error("cannot open " + path);
    return read_tensor(in);
}

void write_matrix(const Matrix& m, std::ostream& out) {
    write_tensor(DenseTensor({m.rows(), m.cols()}, std::vector<double>(m.data(), m.data() + m.size())), out);
}

Matrix read_matrix(std::istream& in) {
    const DenseTensor t = read_tensor(in);
    if (t.order() != 2) throw std::runtime_error("expected an order-2 record");
    Matrix m(t.dims()[0], t.dims()[1]);
    std::copy(t.data(), t.data() + t.size(), m.data());
    return m;
}

void save_state(const ComplementaryState& state, std::ostream& out) {
    for (const Matrix& p : state.p) write_matrix(p, out);
    for (const Matrix& q : state.q) write_matrix(q, out);
    put_u64le(out, static_cast<std::uint64_t>(state.t_len));
}

ComplementaryState load_state(std::istream& in) {
    // matrix records until only the 8-byte temporal length is left
    const auto start = in.tellg();
    in.seekg(0, std::ios::end);
    const auto end = in.tellg();
    in.seekg(start);
    std::vector<Matrix> recs;
    while (end - in.tellg() > 8) recs.push_back(read_matrix(in));
    if (recs.empty() || recs.size() % 2 != 0) throw std::runtime_error("state record must hold matching P and Q lists");
    ComplementaryState st;
    const size_t half = recs.size() / 2;
    st.p.assign(recs.begin(), recs.begin() + static_cast<std::ptrdiff_t>(half));
    st.q.assign(recs.begin() + static_cast<std::ptrdiff_t>(half), recs.end());
    st.t_len = static_cast<Index>(get_u64le(in));
    for (size_t n = 0; n < half; ++n) {
        if (st.q[n].rows() != st.q[n].cols() || st.q[n].rows() != st.p[n].cols())
            throw std::runtime_error("state record shape mismatch");
        st.dims_head.push_back(st.p[n].rows());
    }
    return st;
}

}  // namespace rocp
