// rocp_bench -- the reference CLI's `bench` subcommand (tools/rocp_main.cpp:
// 176-190, report writing :80-121) on the B200 path: same options, same CSV
// reports (write_csv / write_updates_csv).  Only --algorithms rocp runs
// (include/rocp_b200/bench.hpp).  Plain argv parsing (CLI11 is not vendored).
//
//   rocp_bench --dims 1000 1000 1000 --rank 20 --init-frac 0.1 --batch 25
//              --trials 1 --seed 0 --sir-db 20 [--csv out.csv] [--updates-csv u.csv]

#include "../../include/rocp_b200/bench.hpp"

#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <string>
#include <vector>

namespace {

[[noreturn]] void usage(const char* msg) {
    std::fprintf(stderr,
                 "rocp_bench: %s\n"
                 "options: --dims I1 .. IN | --input FILE, --rank R, --samples S, --init-frac F, --batch B,\n"
                 "         --algorithms rocp, --trials T, --seed N, --sir-db DB|none, --rocp-tol X,\n"
                 "         --rocp-max-iters K, --als-tol X, --als-max-iters K, --csv FILE, --updates-csv FILE,\n"
                 "         --device D, --family normal|uniform|congruent, --congruence C\n",
                 msg);
    std::exit(2);
}

}  // namespace

int main(int argc, char** argv) {
    rocp::BenchConfig cfg;
    std::string csv, updates_csv;
    std::vector<std::string> args(argv + 1, argv + argc);
    auto value = [&](size_t& i) -> const std::string& {
        if (i + 1 >= args.size() || args[i + 1].rfind("--", 0) == 0) usage(("missing value for " + args[i]).c_str());
        return args[++i];
    };
    for (size_t i = 0; i < args.size(); ++i) {
        const std::string& a = args[i];
        if (a == "--dims") {
            cfg.dims.clear();
            while (i + 1 < args.size() && args[i + 1].rfind("--", 0) != 0) cfg.dims.push_back(std::stoll(args[++i]));
        } else if (a == "--algorithms") {
            cfg.algorithms.clear();
            while (i + 1 < args.size() && args[i + 1].rfind("--", 0) != 0) {
                const auto alg = rocp::parse_algorithm(args[++i]);
                if (!alg) usage(("unknown algorithm " + args[i]).c_str());
                cfg.algorithms.push_back(*alg);
            }
        } else if (a == "--input") cfg.input_path = value(i);
        else if (a == "--rank") cfg.rank = std::stoi(value(i));
        else if (a == "--samples") cfg.samples = std::stoll(value(i));
        else if (a == "--init-frac") cfg.init_fraction = std::stod(value(i));
        else if (a == "--batch") cfg.batch_size = std::stoll(value(i));
        else if (a == "--trials") cfg.trials = std::stoi(value(i));
        else if (a == "--seed") cfg.seed = std::stoull(value(i));
        else if (a == "--sir-db") {
            const std::string& v = value(i);
            if (v == "none") cfg.sir_db.reset();
            else cfg.sir_db = std::stod(v);
        } else if (a == "--rocp-tol") cfg.rocp_tol = std::stod(value(i));
        else if (a == "--rocp-max-iters") cfg.rocp_max_iters = std::stoi(value(i));
        else if (a == "--als-tol") cfg.als_tol = std::stod(value(i));
        else if (a == "--als-max-iters") cfg.als_max_iters = std::stoi(value(i));
        else if (a == "--csv") csv = value(i);
        else if (a == "--updates-csv") updates_csv = value(i);
        else if (a == "--device") rocp::set_device(std::stoi(value(i)));
        else if (a == "--family") {
            const auto f = rocp::parse_family(value(i));
            if (!f) usage(("unknown factor family " + args[i]).c_str());
            cfg.family = *f;
        } else if (a == "--congruence") cfg.congruence = std::stod(value(i));
        else usage(("unknown option " + a).c_str());
    }
    try {
        const rocp::BenchReport report = rocp::run_benchmark(cfg);
        if (!csv.empty()) {
            std::ofstream out(csv);
            if (!out) throw std::runtime_error("cannot open " + csv);
            rocp::write_csv(report, out);
        } else {
            rocp::write_csv(report, std::cout);
        }
        if (!updates_csv.empty()) {
            std::ofstream out(updates_csv);
            if (!out) throw std::runtime_error("cannot open " + updates_csv);
            rocp::write_updates_csv(report, out);
        }
    } catch (const std::exception& e) {
        std::fprintf(stderr, "rocp_bench: %s\n", e.what());
        return 1;
    }
    return 0;
}
