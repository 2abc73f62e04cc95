// rocp_bench.cpp -- the benchmark-report surface of the reference
// (include/rocp/synthetic.hpp, include/rocp/bench.hpp: the CSV schema and the
// trial/seed conventions) implemented on the B200 stream.  Behavioural notes
// and deviations are listed in include/rocp_b200/bench.hpp.
//
// Structure (own design, not the reference's):
//   * SlabCutter   -- the init/batch boundaries of a stream split, computed once
//                     and materialised slab by slab;
//   * RunningStats -- Welford mean / sample standard deviation per column;
//   * TrialTimer   -- wall-clock bracket around a device-synchronised region;
//   * CsvLine      -- field joiner for the two report tables.

#include "../../include/rocp_b200/bench.hpp"

#include "../../include/rocp_b200.h"

#include <algorithm>
#include <array>
#include <atomic>
#include <chrono>
#include <cstdlib>
#include <exception>
#include <thread>
#include <cmath>
#include <map>
#include <ostream>
#include <sstream>
#include <stdexcept>
#include <utility>

namespace rocp {

namespace {

// ---- device plumbing ------------------------------------------------------------
void status_or_throw(rocp_status st) {
    switch (st) {
        case ROCP_OK: return;
        case ROCP_E_DOMAIN: throw std::domain_error(rocp_last_error(device_handle()));
        case ROCP_E_NUMERICAL: throw NumericalError(rocp_last_error(device_handle()), 0);
        default:
            throw std::runtime_error("rocp_b200 status " + std::to_string(int(st)) + ": " +
                                     rocp_last_error(device_handle()));
    }
}

// Wall time of a region that ends with the device drained, so an asynchronous
// launch is charged to the update that issued it.
class TrialTimer {
public:
    TrialTimer() : t0_(std::chrono::steady_clock::now()) {}
    double stop() const {
        status_or_throw(rocp_synchronize(device_handle()));
        return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0_).count();
    }

private:
    std::chrono::steady_clock::time_point t0_;
};

// Independent std::mt19937_64 per (seed, trial, purpose): the reference seeds its
// generators from the triple through std::seed_seq (bench.hpp seed semantics); purpose
// 0 is the data, purpose 1 + algorithm index the algorithm's draws.
Rng seeded_engine(std::uint64_t seed, int trial, int purpose) {
    std::seed_seq seq{seed, static_cast<std::uint64_t>(trial), static_cast<std::uint64_t>(purpose)};
    return Rng(seq);
}

// ---- stream split ------------------------------------------------------------------
// Boundaries along the last mode: [0, init) then runs of `batch` (the last one may be
// short).  Slabs are contiguous in the first-index-fastest layout.
class SlabCutter {
public:
    SlabCutter(const DenseTensor& x, double init_fraction, Index batch) : x_(x) {
        if (!(init_fraction > 0.0 && init_fraction < 1.0))
            throw std::domain_error("split_stream: init fraction must lie in (0,1)");
        if (batch < 1) throw std::domain_error("split_stream: batch size must be positive");
        const Index t = x.dims().back();
        const Index t_init = static_cast<Index>(std::floor(init_fraction * static_cast<double>(t)));
        if (t_init < 1) throw std::domain_error("split_stream: initial slice is empty");
        slice_ = x.size() / t;
        cuts_.push_back(0);
        cuts_.push_back(t_init);
        while (cuts_.back() < t) cuts_.push_back(std::min(t, cuts_.back() + batch));
    }
    size_t pieces() const { return cuts_.size() - 1; }
    DenseTensor piece(size_t k) const {
        Dims d = x_.dims();
        d.back() = cuts_[k + 1] - cuts_[k];
        const double* lo = x_.data() + cuts_[k] * slice_;
        return DenseTensor(std::move(d), std::vector<double>(lo, lo + d.back() * slice_));
    }

private:
    const DenseTensor& x_;
    Index slice_ = 0;
    std::vector<Index> cuts_;
};

// ---- statistics -----------------------------------------------------------------------
class RunningStats {
public:
    void add(double v) {
        ++n_;
        const double delta = v - mean_;
        mean_ += delta / static_cast<double>(n_);
        m2_ += delta * (v - mean_);
    }
    double mean() const { return mean_; }
    // sample standard deviation; a single observation has none (reported as 0)
    double stddev() const { return n_ > 1 ? std::sqrt(m2_ / static_cast<double>(n_ - 1)) : 0.0; }

private:
    long n_ = 0;
    double mean_ = 0.0, m2_ = 0.0;
};

// ---- CSV ------------------------------------------------------------------------------
class CsvLine {
public:
    explicit CsvLine(std::ostream& out) : out_(out) {}
    template <class T>
    CsvLine& operator<<(const T& field) {
        if (fields_++) out_ << ',';
        out_ << field;
        return *this;
    }
    ~CsvLine() { out_ << '\n'; }

private:
    std::ostream& out_;
    int fields_ = 0;
};

// Restores the caller's stream formatting after writing with 17 significant digits.
class FullPrecision {
public:
    explicit FullPrecision(std::ostream& out) : out_(out), flags_(out.flags()), prec_(out.precision(17)) {}
    ~FullPrecision() {
        out_.precision(prec_);
        out_.flags(flags_);
    }

private:
    std::ostream& out_;
    std::ios::fmtflags flags_;
    std::streamsize prec_;
};

constexpr std::array<std::pair<Algorithm, const char*>, 4> kAlgorithmNames{{
    {Algorithm::rocp, "rocp"},
    {Algorithm::online_full, "online_full"},
    {Algorithm::batch_hot, "batch_hot"},
    {Algorithm::batch_cold, "batch_cold"},
}};

// The B200 cell: randomized init + device stream, each update timed around the
// reference-facing host-slab consume.
TrialResult rocp_trial(const BenchConfig& cfg, int trial, const DenseTensor& full, const SlabCutter& cut) {
    TrialResult out;
    out.trial = trial;
    out.algorithm = Algorithm::rocp;
    Rng rng = seeded_engine(cfg.seed, trial, static_cast<int>(Algorithm::rocp) + 1);
    const Index s = cfg.samples > 0 ? cfg.samples : auto_sample_count(cfg.rank);
    const TrialTimer init_timer;
    InitResult init = cprand_decompose(cut.piece(0), cfg.rank, CprandOptions{cfg.samples, cfg.rocp_tol,
                                                                            cfg.rocp_max_iters}, rng);
    RocpStream stream(std::move(init), s, RocpConfig{}, full.dims().back());
    out.init_seconds = init_timer.stop();
    for (size_t k = 1; k < cut.pieces(); ++k) {
        const DenseTensor slab = cut.piece(k);  // materialised outside the timed region
        const TrialTimer t;
        stream.consume(slab, rng);
        out.update_seconds.push_back(t.stop());
    }
    out.updates = static_cast<Index>(out.update_seconds.size());
    for (double dt : out.update_seconds) out.stream_seconds += dt;
    out.fitness = model_fitness(full, stream.model());
    return out;
}

// Planted factors of one family, drawn in random_model's order (i outer, r inner).
KruskalModel planted_model(const Dims& dims, int rank, Rng& rng, FactorFamily family, double congruence) {
    if (family != FactorFamily::uniform) {
        KruskalModel m = random_model(dims, rank, rng);
        if (family == FactorFamily::congruent) {
            // F <- G C^T with C C^T = c 11^T + (1 - c) I (lower Cholesky factor of the
            // equicorrelation matrix): pairwise column congruence c in expectation.
            if (!(congruence > -1.0 / std::max(rank - 1, 1) && congruence < 1.0))
                throw std::domain_error("gen_synthetic: congruence must keep c 11^T + (1 - c) I positive definite");
            Matrix c(rank, rank);
            for (int j = 0; j < rank; ++j)
                for (int i = j; i < rank; ++i) {
                    double a = (i == j) ? 1.0 : congruence;
                    for (int k = 0; k < j; ++k) a -= c(i, k) * c(j, k);
                    c(i, j) = (i == j) ? std::sqrt(a) : a / c(j, j);
                }
            for (Matrix& f : m.factors) {
                const Matrix g = f;
                for (Index i = 0; i < f.rows(); ++i)
                    for (int r = 0; r < rank; ++r) {
                        double v = 0.0;
                        for (int k = 0; k <= r; ++k) v += g(i, k) * c(r, k);
                        f(i, r) = v;
                    }
            }
        }
        return m;
    }
    KruskalModel m;
    m.rank = rank;
    std::uniform_real_distribution<double> unit(0.0, 1.0);
    for (Index d : dims) {
        Matrix f(d, rank);
        for (Index i = 0; i < d; ++i)
            for (int r = 0; r < rank; ++r) f(i, r) = unit(rng);
        m.factors.push_back(std::move(f));
    }
    return m;
}

}  // namespace

std::optional<FactorFamily> parse_family(const std::string& name) {
    static const std::map<std::string, FactorFamily> names{
        {"normal", FactorFamily::normal}, {"uniform", FactorFamily::uniform}, {"congruent", FactorFamily::congruent}};
    const auto it = names.find(name);
    return it == names.end() ? std::nullopt : std::optional<FactorFamily>(it->second);
}

SyntheticTensor gen_synthetic(const Dims& dims, int rank, std::optional<double> sir_db, Rng& rng) {
    return gen_synthetic(dims, rank, sir_db, rng, FactorFamily::normal);
}

SyntheticTensor gen_synthetic(const Dims& dims, int rank, std::optional<double> sir_db, Rng& rng, FactorFamily family,
                              double congruence) {
    if (rank < 1) throw std::domain_error("gen_synthetic: rank must be positive");
    SyntheticTensor out;
    out.truth = planted_model(dims, rank, rng, family, congruence);
    // Signal and noise are formed on the device (rocp_generate_synthetic): the noise
    // comes from one 64-bit seed drawn after the factors and is scaled so the SIR of
    // the drawn noise is exact.
    const std::uint64_t noise_seed = sir_db ? rng() : 0;
    std::vector<const double*> fp;
    for (const Matrix& f : out.truth.factors) fp.push_back(f.data());
    rocp_tensor* t = nullptr;
    status_or_throw(rocp_tensor_create(device_handle(), dims.data(), static_cast<int>(dims.size()), nullptr, &t));
    DenseTensor x(dims);
    rocp_status st = rocp_generate_synthetic(device_handle(), t, fp.data(), rank, sir_db.has_value() ? 1 : 0,
                                             sir_db.value_or(0.0), noise_seed);
    if (st == ROCP_OK) st = rocp_tensor_download(device_handle(), t, x.data());
    rocp_tensor_free(t);
    status_or_throw(st);
    out.x = std::move(x);
    return out;
}

StreamSplit split_stream(const DenseTensor& x, double init_fraction, Index batch_size) {
    const SlabCutter cut(x, init_fraction, batch_size);
    StreamSplit split;
    split.init = cut.piece(0);
    for (size_t k = 1; k < cut.pieces(); ++k) split.batches.push_back(cut.piece(k));
    return split;
}

const char* algorithm_name(Algorithm a) {
    for (const auto& [alg, name] : kAlgorithmNames)
        if (alg == a) return name;
    return "?";
}

std::optional<Algorithm> parse_algorithm(const std::string& name) {
    for (const auto& [alg, label] : kAlgorithmNames)
        if (name == label) return alg;
    return std::nullopt;
}

std::vector<Aggregate> aggregate_rows(const std::vector<TrialResult>& rows) {
    // one accumulator triple per algorithm, in order of first appearance
    std::vector<std::pair<Algorithm, std::array<RunningStats, 3>>> acc;
    for (const TrialResult& r : rows) {
        auto it = acc.begin();
        while (it != acc.end() && it->first != r.algorithm) ++it;
        if (it == acc.end()) it = acc.insert(acc.end(), {r.algorithm, {}});
        it->second[0].add(r.fitness);
        it->second[1].add(r.init_seconds);
        it->second[2].add(r.stream_seconds);
    }
    std::vector<Aggregate> out;
    for (const auto& [alg, st] : acc)
        out.push_back(Aggregate{alg, st[0].mean(), st[0].stddev(), st[1].mean(), st[1].stddev(), st[2].mean(),
                                st[2].stddev()});
    return out;
}

BenchReport run_benchmark(const BenchConfig& cfg) {
    if (cfg.trials < 1) throw std::domain_error("run_benchmark: trials must be positive");
    if (cfg.algorithms.empty()) throw std::domain_error("run_benchmark: no algorithms selected");
    if (cfg.input_path.empty() && cfg.dims.size() < 2)
        throw std::domain_error("run_benchmark: dims required when no input tensor is given");
    for (Algorithm a : cfg.algorithms)
        if (a != Algorithm::rocp)
            throw std::domain_error(std::string("run_benchmark: ") + algorithm_name(a) +
                                    " is a reference baseline, not on the B200 path (DESIGN.md section 8)");
    BenchReport report;
    const size_t per_trial = cfg.algorithms.size();
    report.rows.resize(size_t(cfg.trials) * per_trial);
    auto run_trial = [&](int trial) {
        Rng data = seeded_engine(cfg.seed, trial, 0);
        const DenseTensor full = cfg.input_path.empty()
                                     ? gen_synthetic(cfg.dims, cfg.rank, cfg.sir_db, data, cfg.family, cfg.congruence).x
                                     : read_tensor_file(cfg.input_path);
        const SlabCutter cut(full, cfg.init_fraction, cfg.batch_size);
        for (size_t a = 0; a < per_trial; ++a) report.rows[size_t(trial) * per_trial + a] = rocp_trial(cfg, trial, full, cut);
    };
    // ROCP_THREADS (reference bench.cpp:190-213; default 1 = serial, which keeps the per-update
    // wall times honest): K trials at a time, each worker thread on its own device handle with
    // 1/K of the SMs for its persistent chain (rocp_set_chain_sms), so the trials share the GPU
    // side by side.  Every cell derives its generators from (seed, trial): the fitness values do
    // not depend on K.
    int workers = 1;
    if (const char* e = std::getenv("ROCP_THREADS")) workers = std::max(1, std::atoi(e));
    workers = std::min(workers, cfg.trials);
    if (workers == 1) {
        for (int trial = 0; trial < cfg.trials; ++trial) run_trial(trial);
    } else {
        const int device = current_device();
        std::atomic<int> next{0};
        std::vector<std::exception_ptr> errs(static_cast<size_t>(workers));
        std::vector<std::thread> pool;
        for (int w = 0; w < workers; ++w)
            pool.emplace_back([&, w] {
                try {
                    set_device(device);
                    int sms = 0;
                    if (rocp_sm_count(device_handle(), &sms) == ROCP_OK && sms / workers >= 16)
                        rocp_set_chain_sms(device_handle(), std::max(16, (sms - sms / 8) / workers));
                    for (int trial = next++; trial < cfg.trials; trial = next++) run_trial(trial);
                } catch (...) {
                    errs[size_t(w)] = std::current_exception();
                }
            });
        for (std::thread& t : pool) t.join();
        for (const std::exception_ptr& e : errs)
            if (e) std::rethrow_exception(e);
    }
    report.aggregates = aggregate_rows(report.rows);
    return report;
}

void write_csv(const BenchReport& report, std::ostream& out) {
    const FullPrecision guard(out);
    out << "trial,algorithm,fitness,init_seconds,stream_seconds,updates,seconds_per_update\n";
    for (const TrialResult& r : report.rows)
        CsvLine(out) << r.trial << algorithm_name(r.algorithm) << r.fitness << r.init_seconds << r.stream_seconds
                     << r.updates << r.seconds_per_update();
    for (const Aggregate& a : report.aggregates) {
        RunningStats per_update;
        for (const TrialResult& r : report.rows)
            if (r.algorithm == a.algorithm) per_update.add(r.seconds_per_update());
        CsvLine(out) << "mean" << algorithm_name(a.algorithm) << a.fitness_mean << a.init_mean << a.stream_mean << ""
                     << per_update.mean();
        CsvLine(out) << "std" << algorithm_name(a.algorithm) << a.fitness_std << a.init_std << a.stream_std << ""
                     << 0.0;
    }
}

void write_updates_csv(const BenchReport& report, std::ostream& out) {
    const FullPrecision guard(out);
    out << "trial,algorithm,update,seconds\n";
    for (const TrialResult& r : report.rows) {
        size_t u = 0;
        for (double dt : r.update_seconds) CsvLine(out) << r.trial << algorithm_name(r.algorithm) << u++ << dt;
    }
}

}  // namespace rocp
