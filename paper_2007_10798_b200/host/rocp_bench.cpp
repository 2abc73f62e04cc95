// rocp_bench.cpp -- synthetic data and the benchmark harness of the reference
// (synthetic.cpp:8-57, bench.cpp:17-264) over the B200 C++ API.  Differences
// are listed in include/rocp_b200/bench.hpp.

#include "../../include/rocp_b200/bench.hpp"

#include "../../include/rocp_b200.h"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <ostream>
#include <stdexcept>

namespace rocp {

namespace {

using Clock = std::chrono::steady_clock;

double seconds_since(Clock::time_point start) {
    return std::chrono::duration<double>(Clock::now() - start).count();
}

// One generator per (seed, trial, stream), as bench.cpp:27-31.
Rng make_rng(std::uint64_t seed, int trial, int stream) {
    std::seed_seq seq{static_cast<std::uint64_t>(seed), static_cast<std::uint64_t>(trial),
                      static_cast<std::uint64_t>(stream)};
    return Rng(seq);
}

void check(rocp_status st) {
    if (st == ROCP_OK) return;
    const std::string msg = rocp_last_error(device_handle());
    if (st == ROCP_E_DOMAIN) throw std::domain_error(msg);
    if (st == ROCP_E_NUMERICAL) throw NumericalError(msg, 0);
    throw std::runtime_error("rocp_b200 status " + std::to_string(int(st)) + ": " + msg);
}

void sync() { check(rocp_synchronize(device_handle())); }

TrialResult run_rocp_cell(const BenchConfig& cfg, int trial, const DenseTensor& full, const StreamSplit& split) {
    TrialResult row;
    row.trial = trial;
    row.algorithm = Algorithm::rocp;
    Rng rng = make_rng(cfg.seed, trial, static_cast<int>(Algorithm::rocp) + 1);
    const CprandOptions opts{cfg.samples, cfg.rocp_tol, cfg.rocp_max_iters};
    const Index s = cfg.samples > 0 ? cfg.samples : auto_sample_count(cfg.rank);
    const auto start = Clock::now();
    InitResult init = cprand_decompose(split.init, cfg.rank, opts, rng);
    RocpStream stream(std::move(init), s, RocpConfig{}, full.dims().back());
    sync();
    row.init_seconds = seconds_since(start);
    for (const DenseTensor& batch : split.batches) {  // bench.cpp:50-59 timed()
        const auto t0 = Clock::now();
        stream.consume(batch, rng);
        sync();
        const double dt = seconds_since(t0);
        row.update_seconds.push_back(dt);
        row.stream_seconds += dt;
        ++row.updates;
    }
    row.fitness = model_fitness(full, stream.model());
    return row;
}

void csv_row(std::ostream& out, const std::string& label, const std::string& algo, double fitness, double init_s,
             double stream_s, const std::string& updates, double per_update) {
    out << label << ',' << algo << ',' << fitness << ',' << init_s << ',' << stream_s << ',' << updates << ','
        << per_update << '\n';
}

}  // namespace

std::optional<FactorFamily> parse_family(const std::string& name) {
    if (name == "normal") return FactorFamily::normal;
    if (name == "uniform") return FactorFamily::uniform;
    if (name == "congruent") return FactorFamily::congruent;
    return std::nullopt;
}

SyntheticTensor gen_synthetic(const Dims& dims, int rank, std::optional<double> sir_db, Rng& rng) {
    return gen_synthetic(dims, rank, sir_db, rng, FactorFamily::normal);
}

SyntheticTensor gen_synthetic(const Dims& dims, int rank, std::optional<double> sir_db, Rng& rng, FactorFamily family,
                              double congruence) {
    if (rank < 1) throw std::domain_error("gen_synthetic: rank must be positive");
    SyntheticTensor out;
    if (family == FactorFamily::uniform) {  // random_model's draw order with U(0,1)
        std::uniform_real_distribution<double> unif(0.0, 1.0);
        out.truth.rank = rank;
        for (Index d : dims) {
            Matrix f(d, rank);
            for (Index i = 0; i < d; ++i)
                for (int r = 0; r < rank; ++r) f(i, r) = unif(rng);
            out.truth.factors.push_back(std::move(f));
        }
    } else {
        out.truth = random_model(dims, rank, rng);
    }
    if (family == FactorFamily::congruent) {  // F = G L^T, L L^T = c 11^T + (1 - c) I
        if (!(congruence > -1.0 / std::max(rank - 1, 1) && congruence < 1.0))
            throw std::domain_error("gen_synthetic: congruence must keep c 11^T + (1 - c) I positive definite");
        std::vector<double> L(size_t(rank) * rank, 0.0);
        for (int i = 0; i < rank; ++i)
            for (int j = 0; j <= i; ++j) {
                double a = (i == j) ? 1.0 : congruence;
                for (int k = 0; k < j; ++k) a -= L[size_t(i) * rank + k] * L[size_t(j) * rank + k];
                L[size_t(i) * rank + j] = (i == j) ? std::sqrt(a) : a / L[size_t(j) * rank + j];
            }
        for (Matrix& f : out.truth.factors) {
            Matrix g = f;
            for (Index i = 0; i < f.rows(); ++i)
                for (int r = 0; r < rank; ++r) {
                    double v = 0.0;
                    for (int k = 0; k <= r; ++k) v += g(i, k) * L[size_t(r) * rank + k];
                    f(i, r) = v;
                }
        }
    }
    // planted signal and exactly scaled noise on the device (rocp_generate_synthetic), one
    // noise seed drawn from rng after the factors
    const std::uint64_t noise_seed = sir_db ? rng() : 0;
    rocp_tensor* t = nullptr;
    check(rocp_tensor_create(device_handle(), dims.data(), static_cast<int>(dims.size()), nullptr, &t));
    std::vector<const double*> f;
    for (const Matrix& m : out.truth.factors) f.push_back(m.data());
    DenseTensor x(dims);
    rocp_status st = rocp_generate_synthetic(device_handle(), t, f.data(), rank, sir_db ? 1 : 0,
                                             sir_db ? *sir_db : 0.0, noise_seed);
    if (st == ROCP_OK) st = rocp_tensor_download(device_handle(), t, x.data());
    rocp_tensor_free(t);
    check(st);
    out.x = std::move(x);
    return out;
}

StreamSplit split_stream(const DenseTensor& x, double init_fraction, Index batch_size) {  // synthetic.cpp:33-57
    if (init_fraction <= 0.0 || init_fraction >= 1.0)
        throw std::domain_error("split_stream: init fraction must lie in (0,1)");
    if (batch_size < 1) throw std::domain_error("split_stream: batch size must be positive");
    const Dims& dims = x.dims();
    const Index t = dims.back();
    const Index t_init = static_cast<Index>(std::floor(init_fraction * static_cast<double>(t)));
    if (t_init < 1) throw std::domain_error("split_stream: initial slice is empty");
    const Index slice = element_count(dims) / t;
    auto take = [&](Index from, Index len) {
        Dims d = dims;
        d.back() = len;
        return DenseTensor(std::move(d), std::vector<double>(x.data() + from * slice, x.data() + (from + len) * slice));
    };
    StreamSplit split;
    split.init = take(0, t_init);
    for (Index pos = t_init; pos < t; pos += batch_size) split.batches.push_back(take(pos, std::min(batch_size, t - pos)));
    return split;
}

const char* algorithm_name(Algorithm a) {
    switch (a) {
        case Algorithm::rocp: return "rocp";
        case Algorithm::online_full: return "online_full";
        case Algorithm::batch_hot: return "batch_hot";
        case Algorithm::batch_cold: return "batch_cold";
    }
    return "?";
}

std::optional<Algorithm> parse_algorithm(const std::string& name) {
    for (Algorithm a : {Algorithm::rocp, Algorithm::online_full, Algorithm::batch_hot, Algorithm::batch_cold})
        if (name == algorithm_name(a)) return a;
    return std::nullopt;
}

std::vector<Aggregate> aggregate_rows(const std::vector<TrialResult>& rows) {  // bench.cpp:136-177
    std::vector<Aggregate> out;
    std::vector<Algorithm> seen;
    for (const TrialResult& r : rows)
        if (std::find(seen.begin(), seen.end(), r.algorithm) == seen.end()) seen.push_back(r.algorithm);
    for (Algorithm a : seen) {
        std::vector<const TrialResult*> group;
        for (const TrialResult& r : rows)
            if (r.algorithm == a) group.push_back(&r);
        const double n = static_cast<double>(group.size());
        auto mean_std = [&](auto field) {
            double mean = 0.0;
            for (const TrialResult* r : group) mean += field(*r);
            mean /= n;
            double var = 0.0;
            for (const TrialResult* r : group) {
                const double d = field(*r) - mean;
                var += d * d;
            }
            return std::pair<double, double>(mean, group.size() > 1 ? std::sqrt(var / (n - 1.0)) : 0.0);
        };
        Aggregate agg;
        agg.algorithm = a;
        std::tie(agg.fitness_mean, agg.fitness_std) = mean_std([](const TrialResult& r) { return r.fitness; });
        std::tie(agg.init_mean, agg.init_std) = mean_std([](const TrialResult& r) { return r.init_seconds; });
        std::tie(agg.stream_mean, agg.stream_std) = mean_std([](const TrialResult& r) { return r.stream_seconds; });
        out.push_back(agg);
    }
    return out;
}

BenchReport run_benchmark(const BenchConfig& cfg) {  // bench.cpp:179-213
    if (cfg.trials < 1) throw std::domain_error("run_benchmark: trials must be positive");
    if (cfg.algorithms.empty()) throw std::domain_error("run_benchmark: no algorithms selected");
    if (cfg.input_path.empty() && cfg.dims.size() < 2)
        throw std::domain_error("run_benchmark: dims required when no input tensor is given");
    for (Algorithm a : cfg.algorithms)
        if (a != Algorithm::rocp)
            throw std::domain_error(std::string("run_benchmark: ") + algorithm_name(a) +
                                    " is a reference baseline, not on the B200 path (DESIGN.md section 8)");
    BenchReport report;
    report.rows.resize(static_cast<size_t>(cfg.trials) * cfg.algorithms.size());
    for (int trial = 0; trial < cfg.trials; ++trial) {
        Rng data_rng = make_rng(cfg.seed, trial, 0);
        const DenseTensor full = cfg.input_path.empty()
                                     ? gen_synthetic(cfg.dims, cfg.rank, cfg.sir_db, data_rng, cfg.family, cfg.congruence).x
                                                        : read_tensor_file(cfg.input_path);
        const StreamSplit split = split_stream(full, cfg.init_fraction, cfg.batch_size);
        for (size_t a = 0; a < cfg.algorithms.size(); ++a)
            report.rows[static_cast<size_t>(trial) * cfg.algorithms.size() + a] = run_rocp_cell(cfg, trial, full, split);
    }
    report.aggregates = aggregate_rows(report.rows);
    return report;
}

void write_csv(const BenchReport& report, std::ostream& out) {  // bench.cpp:226-252
    const auto flags = out.flags();
    const auto prec = out.precision(17);
    out << "trial,algorithm,fitness,init_seconds,stream_seconds,updates,seconds_per_update\n";
    for (const TrialResult& r : report.rows)
        csv_row(out, std::to_string(r.trial), algorithm_name(r.algorithm), r.fitness, r.init_seconds, r.stream_seconds,
                std::to_string(r.updates), r.seconds_per_update());
    for (const Aggregate& a : report.aggregates) {
        double per_update_mean = 0.0;
        int n = 0;
        for (const TrialResult& r : report.rows)
            if (r.algorithm == a.algorithm) {
                per_update_mean += r.seconds_per_update();
                ++n;
            }
        per_update_mean /= std::max(n, 1);
        csv_row(out, "mean", algorithm_name(a.algorithm), a.fitness_mean, a.init_mean, a.stream_mean, "",
                per_update_mean);
        csv_row(out, "std", algorithm_name(a.algorithm), a.fitness_std, a.init_std, a.stream_std, "", 0.0);
    }
    out.precision(prec);
    out.flags(flags);
}

void write_updates_csv(const BenchReport& report, std::ostream& out) {  // bench.cpp:254-264
    const auto flags = out.flags();
    const auto prec = out.precision(17);
    out << "trial,algorithm,update,seconds\n";
    for (const TrialResult& r : report.rows)
        for (size_t u = 0; u < r.update_seconds.size(); ++u)
            out << r.trial << ',' << algorithm_name(r.algorithm) << ',' << u << ',' << r.update_seconds[u] << '\n';
    out.precision(prec);
    out.flags(flags);
}

}  // namespace rocp
