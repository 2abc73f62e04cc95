// C++ API tests, written against include/rocp_b200/rocp.hpp the way the
// reference's doctest suites exercise include/rocp/*.hpp (reference test
// file:line cited per case).  Runs on the GPU (tests/test_cpp_api.py, -m gpu).
#include "rocp_b200/bench.hpp"
#include "rocp_b200/rocp.hpp"

#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <functional>
#include <sstream>
#include <random>
#include <string>
#include <vector>

using namespace rocp;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                                   \
    do {                                                                              \
        if (cond) ++g_pass;                                                           \
        else { ++g_fail; std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); } \
    } while (0)
template <class E, class F>
static bool throws(F&& f) {
    try { f(); } catch (const E&) { return true; } catch (...) { return false; }
    return false;
}

static Matrix random_matrix(Index r, Index c, Rng& rng) {
    std::normal_distribution<double> g(0.0, 1.0);
    Matrix m(r, c);
    for (Index i = 0; i < m.size(); ++i) m.data()[i] = g(rng);
    return m;
}

// test-side elementwise reconstruction (reference tests/oracles.hpp:42-60 idea)
static DenseTensor reconstruct_loops(const KruskalModel& m, const Dims& dims) {
    DenseTensor t(dims);
    std::vector<Index> idx(dims.size(), 0);
    for (Index flat = 0; flat < t.size(); ++flat) {
        double sum = 0.0;
        for (int r = 0; r < m.rank; ++r) {
            double prod = 1.0;
            for (size_t n = 0; n < dims.size(); ++n) prod *= m.factors[n](idx[n], r);
            sum += prod;
        }
        t[flat] = sum;
        for (size_t n = 0; n < dims.size(); ++n) {
            if (++idx[n] < dims[n]) break;
            idx[n] = 0;
        }
    }
    return t;
}

static double frob(const Matrix& a) {
    double s = 0;
    for (Index i = 0; i < a.size(); ++i) s += a.data()[i] * a.data()[i];
    return std::sqrt(s);
}
static double diff(const Matrix& a, const Matrix& b) {
    double s = 0;
    for (Index i = 0; i < a.size(); ++i) s += (a.data()[i] - b.data()[i]) * (a.data()[i] - b.data()[i]);
    return std::sqrt(s);
}

static void test_index_map() {  // test_tensor.cpp:30-82
    const Dims d{2, 3, 4};
    const Index a[2] = {1, 1}, b[2] = {3, 4}, c[2] = {2, 1};
    CHECK(linear_index(a, d, 1) == 1);
    CHECK(linear_index(b, d, 1) == 12);
    CHECK(linear_index(c, d, 2) == 2);
    CHECK((decode_index(12, d, 1) == std::vector<Index>{3, 4}));
    CHECK((decode_index(3, Dims{5, 5}, 2) == std::vector<Index>{3}));
    CHECK(throws<std::domain_error>([&] { decode_index(13, d, 1); }));
    CHECK(auto_sample_count(1) == 1 && auto_sample_count(3) == 33 && auto_sample_count(5) == 81);
}

static void test_draws_and_gather() {  // test_factor_model.cpp:95-168
    const SampleIndexSet one = draw_samples(Dims{1, 1, 5}, 3, 8, CounterKey{1, 0, 0});
    bool all_one = true;
    for (Index j : one.rows) all_one = all_one && j == 1;
    CHECK(all_one);
    const SampleIndexSet x1 = draw_samples(Dims{4, 5, 6}, 2, 50, CounterKey{99, 0, 0});
    const SampleIndexSet x2 = draw_samples(Dims{4, 5, 6}, 2, 50, CounterKey{99, 0, 0});
    CHECK(x1.rows == x2.rows && x1.decoded == x2.decoded);
    const SampleIndexSet u = draw_samples(Dims{2, 10}, 1, 10000, CounterKey{4242, 0, 0});
    std::vector<int> freq(10, 0);
    for (Index j : u.rows) ++freq[static_cast<size_t>(j - 1)];
    bool uniform = true;
    for (int f : freq) uniform = uniform && std::abs(f - 1000.0) <= 5.0 * std::sqrt(10000 * 0.09);
    CHECK(uniform);
    Rng rng(55);
    DenseTensor t({3, 4, 5});
    std::normal_distribution<double> g;
    for (Index i = 0; i < t.size(); ++i) t[i] = g(rng);
    const Matrix dup = sample_unfolding(t, SampleIndexSet::from_rows(t.dims(), 1, {4, 4}));
    CHECK(dup(0, 0) == dup(0, 1) && dup(2, 0) == dup(2, 1));
    const Matrix col = sample_unfolding(t, SampleIndexSet::from_rows(t.dims(), 2, {7}));
    const std::vector<Index> mi = decode_index(7, t.dims(), 2);  // (i1, i3)
    bool fibre = true;
    for (Index i2 = 0; i2 < 4; ++i2) fibre = fibre && col(i2, 0) == t[(mi[0] - 1) + 3 * i2 + 12 * (mi[1] - 1)];
    CHECK(fibre);
    CHECK(throws<std::domain_error>([&] { sample_unfolding(t, SampleIndexSet::from_rows({3, 4, 6}, 1, {1})); }));
}

static void test_skr() {  // test_factor_model.cpp:172-218
    Rng rng(73);
    const Dims dims{2, 3, 4};
    const KruskalModel m = random_model(dims, 3, rng);
    for (int mode = 1; mode <= 3; ++mode) {
        const auto fs = factors_excluding(m, mode);
        const SampleIndexSet all = SampleIndexSet::all_columns(dims, mode);
        const Matrix z = sampled_khatri_rao(all, fs);
        // row c is the Hadamard product of decoded factor rows, left to right
        bool ok = true;
        for (Index c = 0; c < all.count(); ++c)
            for (int r = 0; r < 3; ++r) {
                double v = 1.0;
                for (size_t l = 0; l < fs.size(); ++l)
                    v = v * fs[l](all.decoded_at(c, static_cast<int>(fs.size() - 1 - l)) - 1, r);
                ok = ok && z(c, r) == v;
            }
        CHECK(ok);
    }
}

static void test_solve() {  // test_cprand.cpp:25-81
    Rng rng(101);
    const Matrix x = random_matrix(5, 3, rng);
    CHECK(diff(solve_sampled_ls(Matrix::Identity(3, 3), x), x) < 1e-14);
    const Matrix u0 = random_matrix(6, 3, rng), z = random_matrix(20, 3, rng);
    Matrix xs(6, 20);
    for (Index i = 0; i < 6; ++i)
        for (Index c = 0; c < 20; ++c) {
            double v = 0;
            for (int r = 0; r < 3; ++r) v += u0(i, r) * z(c, r);
            xs(i, c) = v;
        }
    CHECK(diff(solve_sampled_ls(z, xs), u0) <= 1e-10 * frob(u0));
    SolveInfo info;
    const Matrix u = solve_sampled_ls(random_matrix(2, 4, rng), random_matrix(3, 2, rng), &info);
    CHECK(info.underdetermined && info.regularized && u.allFinite());
    SolveInfo zi;
    const Matrix uz = solve_sampled_ls(Matrix::Zero(5, 2), random_matrix(3, 5, rng), &zi);
    CHECK(zi.regularized && uz == Matrix::Zero(3, 2));
    CHECK(throws<std::domain_error>([&] { solve_sampled_ls(Matrix::Zero(5, 2), Matrix::Zero(3, 4)); }));
}

static void test_cprand() {  // test_cprand.cpp:83-198
    {
        Rng gen(13);
        const Dims dims{30, 30, 30};
        const DenseTensor x = reconstruct_loops(random_model(dims, 5, gen), dims);
        Rng rng(17);
        const InitResult res = cprand_decompose(x, 5, {}, rng);
        CHECK(res.best_fitness >= 0.99);
        CHECK(std::abs(model_fitness(x, res.model) - res.best_fitness) < 1e-12);
    }
    {
        Rng gen(19);
        const Dims dims{8, 9, 10};
        const DenseTensor x = reconstruct_loops(random_model(dims, 3, gen), dims);
        Rng a(23), b(23);
        const InitResult ra = cprand_decompose(x, 3, {}, a), rb = cprand_decompose(x, 3, {}, b);
        CHECK(ra.best_fitness == rb.best_fitness && ra.iterations == rb.iterations);
        for (int n = 0; n < 3; ++n) CHECK(ra.model.factors[static_cast<size_t>(n)] == rb.model.factors[static_cast<size_t>(n)]);
    }
    Rng r1(1);
    CHECK(throws<std::domain_error>([&] { cprand_decompose(DenseTensor({3, 3}), 1, {}, r1); }));
    DenseTensor inf({3, 3, 3});
    inf[0] = INFINITY;
    int sweep = -1;
    try {
        Rng r2(1);
        cprand_decompose(inf, 2, {}, r2);
    } catch (const NumericalError& e) {
        sweep = e.sweep();
    }
    CHECK(sweep == 1);
}

static void test_stream() {  // test_rocp.cpp:235-294
    const Dims dims{20, 20, 200};
    Rng gen(383);
    const KruskalModel truth = random_model(dims, 5, gen);
    const DenseTensor x = reconstruct_loops(truth, dims);
    const Index slice = 400;
    auto take = [&](Index t0, Index len) {
        std::vector<double> v(x.data() + t0 * slice, x.data() + (t0 + len) * slice);
        return DenseTensor({20, 20, len}, std::move(v));
    };
    std::vector<DenseTensor> batches;
    for (Index t = 40; t < 200; ++t) batches.push_back(take(t, 1));
    Rng rng(389);
    const KruskalModel model = rocp_run(take(0, 40), batches, 5, {}, rng);
    CHECK(model.factors.back().rows() == 200);
    CHECK(model_fitness(x, model) >= 0.95);

    // frozen old temporal rows and constant state footprint
    Rng rng2(7);
    InitResult init = cprand_decompose(take(0, 40), 5, {}, rng2);
    RocpStream st(std::move(init), auto_sample_count(5), {}, 200);
    Matrix before = st.model().factors.back();
    const std::size_t bytes = st.state().byte_size();
    bool frozen = true, constant = true;
    for (Index t = 40; t < 60; ++t) {
        st.consume(take(t, 1), rng2);
        const Matrix now = st.model().factors.back();
        for (Index i = 0; i < before.rows(); ++i)
            for (int r = 0; r < 5; ++r) frozen = frozen && now(i, r) == before(i, r);
        constant = constant && st.state().byte_size() == bytes;
        before = now;
    }
    CHECK(frozen && constant && st.t_len() == 60);
    CHECK(st.last_residual() >= 0.0 && st.last_residual() < 1.0);
    CHECK(throws<std::domain_error>([&] { st.consume(DenseTensor({20, 21, 1}), rng2); }));
}

static void test_records() {  // test_tensor_io.cpp-style round trips; rocp.cpp:180-211
    DenseTensor t({3, 2, 4});
    for (Index i = 0; i < t.size(); ++i) t[i] = 0.5 * double(i) - 3.0;
    std::stringstream buf;
    write_tensor(t, buf);
    const std::string bytes = buf.str();
    CHECK(bytes.size() == 4 + 1 + 4 + 3 * 8 + 24 * 8 && bytes.compare(0, 4, "ROCP") == 0 && bytes[4] == 1);
    const DenseTensor back = read_tensor(buf);
    CHECK(back.dims() == t.dims());
    bool same = true;
    for (Index i = 0; i < t.size(); ++i) same = same && back[i] == t[i];
    CHECK(same);
    // 2 x 2 matrix: column-major values after the 25-byte header
    Matrix m(2, 2);
    m(0, 0) = 1.0; m(1, 0) = 3.0; m(0, 1) = 2.0; m(1, 1) = 4.0;
    std::stringstream mb;
    write_matrix(m, mb);
    double v[4];
    std::memcpy(v, mb.str().data() + 25, sizeof(v));
    CHECK(v[0] == 1.0 && v[1] == 3.0 && v[2] == 2.0 && v[3] == 4.0);
    CHECK(read_matrix(mb) == m);
    std::stringstream bad("ROCX\x01");
    CHECK(throws<std::runtime_error>([&] { read_tensor(bad); }));
    std::stringstream trunc(bytes.substr(0, bytes.size() - 8));
    CHECK(throws<std::runtime_error>([&] { read_tensor(trunc); }));
    CHECK(throws<std::runtime_error>([&] { read_tensor_file("/nonexistent/x.rocp"); }));
    // save_state / load_state of a live stream
    Rng rng(91);
    KruskalModel truth = random_model({12, 10, 40}, 3, rng);
    const DenseTensor x = reconstruct_loops(truth, {12, 10, 40});
    DenseTensor xi({12, 10, 16}), xb({12, 10, 8});
    std::copy(x.data(), x.data() + xi.size(), xi.data());
    std::copy(x.data() + xi.size(), x.data() + xi.size() + xb.size(), xb.data());
    RocpStream st(cprand_decompose(xi, 3, {}, rng), auto_sample_count(3), {}, 64);
    st.consume(xb, rng);
    const ComplementaryState s0 = st.state();
    std::stringstream sb;
    save_state(s0, sb);
    const ComplementaryState s1 = load_state(sb);
    CHECK(s1.t_len == s0.t_len && s1.t_len == 24 && s1.dims_head == s0.dims_head);
    bool eq = s1.p.size() == 2 && s1.q.size() == 2;
    for (size_t n = 0; eq && n < 2; ++n) eq = s1.p[n] == s0.p[n] && s1.q[n] == s0.q[n];
    CHECK(eq);
}

static void test_synthetic() {  // test_bench.cpp:15-91
    {
        Rng rng(501);  // no noise level: the exact low-rank signal
        const SyntheticTensor d = gen_synthetic({5, 6, 7}, 3, std::nullopt, rng);
        const DenseTensor sig = reconstruct_loops(d.truth, {5, 6, 7});
        double worst = 0.0;
        for (Index i = 0; i < d.x.size(); ++i) worst = std::max(worst, std::abs(d.x[i] - sig[i]));
        CHECK(worst <= 1e-12);
    }
    for (double sir : {20.0, 6.0, 40.0}) {  // noise scaled to the requested level exactly
        Rng rng(503);
        const SyntheticTensor d = gen_synthetic({8, 9, 10}, 4, sir, rng);
        const DenseTensor sig = reconstruct_loops(d.truth, {8, 9, 10});
        double ss = 0.0, nn = 0.0;
        for (Index i = 0; i < d.x.size(); ++i) {
            ss += sig[i] * sig[i];
            nn += (d.x[i] - sig[i]) * (d.x[i] - sig[i]);
        }
        CHECK(std::abs(10.0 * std::log10(ss / nn) - sir) <= 1e-6 * sir);
    }
    {
        Rng rng(507);
        const SyntheticTensor d = gen_synthetic({60, 60, 60, 200}, 5, 20.0, rng);
        CHECK((d.x.dims() == Dims{60, 60, 60, 200}) && d.truth.rank == 5 && d.x.size() == 60 * 60 * 60 * 200);
    }
    Rng rng(509);
    {
        const SyntheticTensor d = gen_synthetic({4, 5, 200}, 2, std::nullopt, rng);
        const StreamSplit sp = split_stream(d.x, 0.2, 1);
        bool ones = sp.batches.size() == 160;
        for (const DenseTensor& b : sp.batches) ones = ones && b.dims().back() == 1;
        CHECK(sp.init.dims().back() == 40 && ones);
    }
    {
        const SyntheticTensor d = gen_synthetic({3, 3, 10}, 2, std::nullopt, rng);
        const StreamSplit sp = split_stream(d.x, 0.2, 4);
        CHECK(sp.init.dims().back() == 2 && sp.batches.size() == 2 && sp.batches[0].dims().back() == 4 &&
              sp.batches[1].dims().back() == 4);
    }
    {
        const SyntheticTensor d = gen_synthetic({4, 3, 11}, 2, 20.0, rng);
        const StreamSplit sp = split_stream(d.x, 0.3, 2);
        std::vector<double> joined = sp.init.values();
        for (const DenseTensor& b : sp.batches) joined.insert(joined.end(), b.values().begin(), b.values().end());
        CHECK(joined == d.x.values());
    }
    {
        const SyntheticTensor d = gen_synthetic({3, 3, 4}, 1, std::nullopt, rng);
        CHECK(throws<std::domain_error>([&] { split_stream(d.x, 0.1, 1); }));
        CHECK(throws<std::domain_error>([&] { split_stream(d.x, 0.0, 1); }));
        CHECK(throws<std::domain_error>([&] { split_stream(d.x, 0.5, 0); }));
    }
}

static void test_factor_families() {  // BASELINE configs[2] (U(0,1)) and configs[4] (congruence 0.9)
    Rng r1(601);
    const SyntheticTensor u = gen_synthetic({30, 20, 10}, 4, 30.0, r1, FactorFamily::uniform);
    bool in01 = true;
    for (const Matrix& f : u.truth.factors)
        for (Index i = 0; i < f.size(); ++i) in01 = in01 && f.data()[i] >= 0.0 && f.data()[i] < 1.0;
    CHECK(in01 && u.x.size() == 30 * 20 * 10);
    Rng r2(603);
    const SyntheticTensor c = gen_synthetic({4000, 8, 6}, 3, std::nullopt, r2, FactorFamily::congruent, 0.9);
    const Matrix& f = c.truth.factors[0];
    double worst = 0.0;
    for (int a = 0; a < 3; ++a)
        for (int b = a + 1; b < 3; ++b) {
            double ab = 0, aa = 0, bb = 0;
            for (Index i = 0; i < f.rows(); ++i) {
                ab += f(i, a) * f(i, b);
                aa += f(i, a) * f(i, a);
                bb += f(i, b) * f(i, b);
            }
            worst = std::max(worst, std::abs(ab / std::sqrt(aa * bb) - 0.9));
        }
    CHECK(worst < 0.03);  // sample column congruence of 4000 rows
    Rng r3(605), r4(605);  // the normal family is the reference's gen_synthetic
    const SyntheticTensor n1 = gen_synthetic({5, 6, 7}, 2, 20.0, r3), n2 = gen_synthetic({5, 6, 7}, 2, 20.0, r4, FactorFamily::normal);
    CHECK(n1.x.values() == n2.x.values());
    CHECK(throws<std::domain_error>([&] { Rng r(1); gen_synthetic({4, 4, 4}, 3, std::nullopt, r, FactorFamily::congruent, 1.0); }));
    CHECK(parse_family("uniform") == FactorFamily::uniform && !parse_family("gamma").has_value());
}

static void test_bench_harness() {  // test_bench.cpp:114-207
    {
        BenchConfig cfg;  // single-trial smoke run
        cfg.dims = {8, 8, 20};
        cfg.rank = 2;
        cfg.trials = 1;
        cfg.algorithms = {Algorithm::rocp};
        cfg.seed = 7;
        const BenchReport r = run_benchmark(cfg);
        CHECK(r.rows.size() == 1);
        const TrialResult& row = r.rows.front();
        CHECK(row.fitness > 0.0 && row.fitness <= 1.0);
        CHECK(row.updates == 16 && row.update_seconds.size() == 16);
        CHECK(r.aggregates.size() == 1 && r.aggregates[0].fitness_mean == row.fitness);
    }
    {
        BenchConfig cfg;  // fitness is deterministic for a fixed config
        cfg.dims = {6, 6, 15};
        cfg.rank = 2;
        cfg.trials = 3;
        cfg.seed = 11;
        const BenchReport a = run_benchmark(cfg), b = run_benchmark(cfg);
        bool same = a.rows.size() == b.rows.size() && a.rows.size() == 3;
        for (size_t i = 0; same && i < a.rows.size(); ++i) same = a.rows[i].fitness == b.rows[i].fitness;
        CHECK(same);
        cfg.algorithms = {Algorithm::rocp, Algorithm::batch_hot};  // baselines are not on this path
        CHECK(throws<std::domain_error>([&] { run_benchmark(cfg); }));
    }
    {
        BenchConfig cfg;  // ROCP_THREADS: trials side by side on one GPU, fitness independent of the parallelism
        cfg.dims = {10, 9, 24};
        cfg.rank = 3;
        cfg.trials = 5;
        cfg.seed = 19;
        const BenchReport serial = run_benchmark(cfg);
        setenv("ROCP_THREADS", "3", 1);
        const BenchReport par = run_benchmark(cfg);
        unsetenv("ROCP_THREADS");
        bool same = serial.rows.size() == 5 && par.rows.size() == 5;
        for (size_t i = 0; same && i < 5; ++i)
            same = serial.rows[i].trial == int(i) && par.rows[i].trial == int(i) &&
                   serial.rows[i].fitness == par.rows[i].fitness && par.rows[i].updates == serial.rows[i].updates;
        CHECK(same);
        CHECK(par.aggregates.size() == 1 && par.aggregates[0].fitness_mean == serial.aggregates[0].fitness_mean);
    }
    {
        BenchConfig cfg;  // aggregates are recomputable from the rows
        cfg.dims = {6, 6, 15};
        cfg.rank = 2;
        cfg.trials = 4;
        cfg.seed = 13;
        const BenchReport r = run_benchmark(cfg);
        double mean = 0.0, var = 0.0;
        for (const TrialResult& t : r.rows) mean += t.fitness;
        mean /= 4.0;
        for (const TrialResult& t : r.rows) var += (t.fitness - mean) * (t.fitness - mean);
        CHECK(std::abs(r.aggregates[0].fitness_mean - mean) <= 1e-12);
        CHECK(std::abs(r.aggregates[0].fitness_std - std::sqrt(var / 3.0)) <= 1e-12);
    }
    {
        BenchConfig cfg;  // CSV report carries the mean/std block
        cfg.dims = {6, 6, 12};
        cfg.rank = 2;
        cfg.trials = 2;
        cfg.seed = 17;
        const BenchReport r = run_benchmark(cfg);
        std::stringstream csv, upd;
        write_csv(r, csv);
        const std::string text = csv.str();
        CHECK(text.find("trial,algorithm,fitness,init_seconds,stream_seconds,updates,seconds_per_update") !=
              std::string::npos);
        CHECK(text.find("\nmean,rocp,") != std::string::npos && text.find("\nstd,rocp,") != std::string::npos);
        write_updates_csv(r, upd);
        CHECK(upd.str().find("trial,algorithm,update,seconds") != std::string::npos);
    }
    {
        BenchConfig cfg;  // config errors are rejected
        cfg.dims = {6, 6, 12};
        cfg.trials = 0;
        CHECK(throws<std::domain_error>([&] { run_benchmark(cfg); }));
        cfg.trials = 1;
        cfg.algorithms.clear();
        CHECK(throws<std::domain_error>([&] { run_benchmark(cfg); }));
    }
    for (Algorithm a : {Algorithm::rocp, Algorithm::online_full, Algorithm::batch_hot, Algorithm::batch_cold})
        CHECK(parse_algorithm(algorithm_name(a)) == a);
    CHECK(!parse_algorithm("onlinecp").has_value());
}

static bool bitwise(const Matrix& a, const Matrix& b) {
    return a.rows() == b.rows() && a.cols() == b.cols() &&
           std::memcmp(a.data(), b.data(), static_cast<size_t>(a.size()) * sizeof(double)) == 0;
}

// The reference's free functions (rocp.hpp:35-81) replay RocpStream::consume bit for bit
// (consume = update_last_mode + append + update_other_modes, rocp.cpp:144-160).
static void test_free_functions_replay_consume() {
    const Dims dims{16, 14, 60};
    const int R = 4;
    Rng gen(71);
    const KruskalModel truth = random_model(dims, R, gen);
    const DenseTensor x = reconstruct_loops(truth, dims);
    const Index slice = 16 * 14, t_init = 20, B = 5;
    auto take = [&](Index t0, Index len) {
        std::vector<double> v(x.data() + t0 * slice, x.data() + (t0 + len) * slice);
        return DenseTensor({16, 14, len}, std::move(v));
    };
    Rng rng(73);
    InitResult init = cprand_decompose(take(0, t_init), R, {}, rng);
    const Index s = auto_sample_count(R);
    ComplementaryState state = init_state(init, s);  // rocp.cpp:45-69
    CHECK(state.t_len == t_init && state.sample_count == s && state.p.size() == 2 && state.q.size() == 2);
    KruskalModel model = init.model;
    RocpStream stream(init, s);
    {
        const ComplementaryState direct = stream.state();
        for (size_t n = 0; n < 2; ++n) CHECK(bitwise(state.p[n], direct.p[n]) && bitwise(state.q[n], direct.q[n]));
    }
    std::vector<Matrix> temporal_rows;
    bool all_equal = true;
    const std::uint64_t seed = 0x5eedULL;
    for (Index t = t_init, b = 1; t + B <= 60; t += B, ++b) {
        const DenseTensor xb = take(t, B);
        const CounterKey key{seed, static_cast<std::uint32_t>(b), 0};
        const LastModeUpdate lm = update_last_mode(model, xb, s, key);
        CHECK(lm.idx.mode == 3 && lm.idx.count() == s && lm.z_s.rows() == s && lm.u_new.rows() == B);
        UpdateTrace tr;
        update_other_modes(state, model, xb, lm.u_new, key, &tr);
        CHECK(tr.mode_idx.size() == 2 && tr.mode_z.size() == 2 && tr.mode_x.size() == 2);
        temporal_rows.push_back(lm.u_new);
        stream.consume(xb, seed, static_cast<std::uint32_t>(b));
        const KruskalModel m = stream.model();
        const ComplementaryState cs = stream.state();
        for (size_t n = 0; n < 2; ++n)
            all_equal = all_equal && bitwise(m.factors[n], model.factors[n]) && bitwise(cs.p[n], state.p[n]) &&
                        bitwise(cs.q[n], state.q[n]);
        const Matrix& tf = m.factors.back();
        for (Index i = 0; i < B; ++i)
            for (int r = 0; r < R; ++r) all_equal = all_equal && tf(t + i, r) == lm.u_new(i, r);
    }
    CHECK(all_equal);
    CHECK(stream.t_len() == 60);
    // update_mode_with / update_last_mode_with contracts (rocp.cpp:75,100-101)
    const DenseTensor xb = take(20, B);
    CHECK(throws<std::domain_error>(
        [&] { update_last_mode_with(model, xb, draw_samples(xb.dims(), 1, s, CounterKey{1, 1, 0})); }));
    CHECK(throws<std::domain_error>([&] {
        update_mode_with(state, model, xb, Matrix(B, R), draw_samples(xb.dims(), 3, s, CounterKey{1, 1, 0}));
    }));
    CHECK(throws<std::domain_error>(
        [&] { update_other_modes(state, model, xb, Matrix(B + 1, R), CounterKey{1, 1, 0}); }));
    CHECK(throws<std::domain_error>([&] { update_last_mode(model, DenseTensor({16, 15, 2}), s, CounterKey{}); }));
    InitResult bad = init;
    bad.best_sampled_kr.pop_back();
    CHECK(throws<std::domain_error>([&] { init_state(bad, s); }));
    CHECK(throws<std::domain_error>([&] { init_state(init, s + 1); }));
}

// Traces are filled (cprand.cpp:34,44; rocp.cpp:125-129) and a traced consume equals an
// untraced one bit for bit.
static void test_traces() {
    const Dims dims{12, 10, 40};
    const int R = 3;
    Rng gen(91);
    const DenseTensor x = reconstruct_loops(random_model(dims, R, gen), dims);
    const Index slice = 120;
    auto take = [&](Index t0, Index len) {
        std::vector<double> v(x.data() + t0 * slice, x.data() + (t0 + len) * slice);
        return DenseTensor({12, 10, len}, std::move(v));
    };
    Rng a(97), b(97);
    CprandTrace ct;
    const InitResult ia = cprand_decompose(take(0, 10), R, {}, a, &ct);
    const InitResult ib = cprand_decompose(take(0, 10), R, {}, b);
    CHECK(static_cast<int>(ct.sweeps.size()) == ia.iterations);
    bool shapes = true, fresh = false;
    for (const auto& sw : ct.sweeps) {
        shapes = shapes && sw.size() == 3;
        for (int n = 0; n < 3 && sw.size() == 3; ++n)
            shapes = shapes && sw[static_cast<size_t>(n)].mode == n + 1 && sw[static_cast<size_t>(n)].count() == auto_sample_count(R);
    }
    for (size_t k = 1; k < ct.sweeps.size(); ++k) fresh = fresh || ct.sweeps[k][0].rows != ct.sweeps[0][0].rows;
    CHECK(shapes);
    CHECK(ct.sweeps.size() < 2 || fresh);  // fresh draws each sweep (test_cprand.cpp:165-180)
    CHECK(ia.best_fitness == ib.best_fitness);
    const Index s = auto_sample_count(R);
    RocpStream sa(ia, s), sb(ib, s);
    std::vector<UpdateTrace> traces;
    for (Index t = 10; t + 5 <= 40; t += 5) {
        traces.emplace_back();
        sa.consume(take(t, 5), a, &traces.back());
        sb.consume(take(t, 5), b);
    }
    const KruskalModel ma = sa.model(), mb = sb.model();
    bool eq = true;
    for (size_t n = 0; n < 3; ++n) eq = eq && bitwise(ma.factors[n], mb.factors[n]);
    CHECK(eq);
    CHECK(sa.regularized() == sb.regularized());
    bool tr_ok = true;
    for (const UpdateTrace& tr : traces) {
        tr_ok = tr_ok && tr.mode_idx.size() == 2 && tr.mode_z.size() == 2 && tr.mode_x.size() == 2;
        for (size_t n = 0; n < tr.mode_x.size(); ++n)
            tr_ok = tr_ok && tr.mode_x[n].rows() == dims[n] && tr.mode_x[n].cols() == s && tr.mode_z[n].rows() == s;
    }
    CHECK(tr_ok);
}

// Constant streaming footprint over 500 batches through the 3-argument constructor
// (acceptance.cpp:427-471): the temporal factor grows geometrically (rocp.cpp:152-155)
// instead of failing on stream length.
static void test_long_stream_growth() {
    Rng gen(10001);
    const Dims head{20, 20, 20};
    Dims dims = head;
    dims.push_back(20);
    const KruskalModel truth = random_model(dims, 5, gen);
    const DenseTensor x_init = reconstruct_loops(truth, dims);
    Rng rng(10003);
    InitResult init = cprand_decompose(x_init, 5, {}, rng);
    RocpStream stream(std::move(init), auto_sample_count(5));
    const std::size_t bytes = stream.state().byte_size();
    bool constant = true;
    Dims slab_dims = head;
    slab_dims.push_back(1);
    for (int k = 0; k < 500; ++k) {
        KruskalModel slab_model = truth;
        slab_model.factors.back() = random_matrix(1, 5, rng);
        stream.consume(reconstruct_loops(slab_model, slab_dims), rng);
        constant = constant && stream.state().byte_size() == bytes;
    }
    CHECK(constant);
    CHECK(stream.t_len() == 520);
    const KruskalModel m = stream.model();
    CHECK(m.factors.back().rows() == 520 && m.factors.back().allFinite());
}

int main() {
    const std::vector<std::pair<const char*, std::function<void()>>> cases = {
        {"index_map", test_index_map}, {"draws_and_gather", test_draws_and_gather}, {"skr", test_skr},
        {"solve", test_solve},         {"cprand", test_cprand},                     {"stream", test_stream},
        {"records", test_records},     {"synthetic", test_synthetic},               {"bench_harness", test_bench_harness},
        {"factor_families", test_factor_families},
        {"free_functions_replay_consume", test_free_functions_replay_consume},
        {"traces", test_traces},
        {"long_stream_growth", test_long_stream_growth}};
    for (const auto& [name, fn] : cases) {
        const int before = g_fail;
        try {
            fn();
        } catch (const std::exception& e) {
            ++g_fail;
            std::printf("FAIL %s: exception %s\n", name, e.what());
        }
        std::printf("%s %s\n", g_fail == before ? "[PASS]" : "[FAIL]", name);
    }
    std::printf("%d checks passed, %d failed\n", g_pass, g_fail);
    return g_fail == 0 ? 0 : 1;
}
