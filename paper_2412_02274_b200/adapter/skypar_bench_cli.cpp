// skypar_bench_cli.cpp — the `skypar-bench` front end (proj/tools/bench_main.cpp:47-63
// flags; CLI11 is absent here, so the parser is hand-written).  It prints the
// same two tables as the reference tool: the dataset skyline per strategy
// (serial SFS first) and the grid-resistance scan per strategy, with the
// dominance-test accounting (parallel_max, final_tests, simulated cost) and
// wall times.  Built by oracle/build_ref.sh over the GPU drop-in
// (oracle/_ref/skypar_bench_gpu) and over the CPU library
// (oracle/_ref/skypar_bench_ref): the count columns agree exactly, the wall
// columns show the speed-up.
#include <cerrno>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "skypar/datagen.hpp"
#include "skypar/gres.hpp"
#include "skypar/harness.hpp"

namespace {

struct Row {
    std::string name;
    std::uint64_t pmax = 0, fin = 0, cost = 0;
    double ms = 0;
};

void table(const char* title, const std::vector<Row>& rows) {
    std::printf("%s\n", title);
    std::printf("  %-10s %15s %15s %15s %12s %9s\n", "strategy", "parallel_max", "final_tests",
                "simulated", "wall_ms", "speedup");
    const double base = rows.empty() ? 0.0 : rows[0].ms;
    for (const Row& r : rows)
        std::printf("  %-10s %15llu %15llu %15llu %12.2f %8.2fx\n", r.name.c_str(),
                    (unsigned long long)r.pmax, (unsigned long long)r.fin,
                    (unsigned long long)r.cost, r.ms, r.ms > 0 ? base / r.ms : 0.0);
}

[[noreturn]] void usage(const std::string& msg) {
    std::fprintf(stderr, "%s\nRun with --help for more information.\n", msg.c_str());
    std::exit(2);
}

template <class T>
T number(const std::string& flag, const char* text) {
    char* end = nullptr;
    errno = 0;
    const long long v = std::strtoll(text, &end, 10);
    if (!*text || *end || errno) usage(flag + ": " + text + " is not a valid number");
    if (std::is_unsigned_v<T> && v < 0) usage(flag + ": " + text + " is not a valid number");
    return static_cast<T>(v);
}

}  // namespace

int main(int argc, char** argv) {
    std::size_t n = 100000, reps = 0;
    int dims = 3, cores = 16, cap = 25;
    long long partitions = 16;
    std::uint64_t seed = 1;
    std::string gen = "ant";
    for (int i = 1; i < argc; ++i) {
        std::string flag = argv[i];
        std::string val;
        const auto eq = flag.find('=');
        if (eq != std::string::npos) {
            val = flag.substr(eq + 1);
            flag = flag.substr(0, eq);
        }
        if (flag == "-h" || flag == "--help") {
            std::printf(
                "compare the serial skyline reference with the partitioned path\n"
                "Usage: skypar-bench [--n N] [--d D] [--gen uni|ant] [--seed S] "
                "[--partitions P] [--cores C] [--cap G] [--reps K]\n");
            return 0;
        }
        if (eq == std::string::npos) {
            if (i + 1 >= argc) usage(flag + ": requires a value");
            val = argv[++i];
        }
        const char* v = val.c_str();
        if (flag == "--n") n = number<std::size_t>(flag, v);
        else if (flag == "--d") dims = number<int>(flag, v);
        else if (flag == "--seed") seed = number<std::uint64_t>(flag, v);
        else if (flag == "--partitions") partitions = number<long long>(flag, v);
        else if (flag == "--cores") cores = number<int>(flag, v);
        else if (flag == "--cap") cap = number<int>(flag, v);
        else if (flag == "--reps") reps = number<std::size_t>(flag, v);
        else if (flag == "--gen") {
            if (val != "uni" && val != "ant") usage("--gen: " + val + " not in {uni,ant}");
            gen = val;
        } else usage("unknown option: " + flag);
    }
    using namespace skypar;
    using Clock = std::chrono::steady_clock;
    try {
        const Relation data = generate(GenSpec{n, dims, distribution_from_name(gen), seed});
        std::printf("dataset %s n=%zu d=%d, partitions=%lld cores=%d cap=%d reps=%zu\n\n",
                    gen.c_str(), n, dims, partitions, cores, cap, reps);
        const Strategy all[] = {Strategy::None, Strategy::Grid, Strategy::Angular,
                                Strategy::Sliced};
        std::vector<Row> sky;
        Relation skyline(data.dims);
        {
            DominanceCounter c;
            const auto t0 = Clock::now();
            skyline = skyline_sfs(data, c);  // the serial baseline (core.cpp)
            const double ms = std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
            sky.push_back({"serial", c.count, 0, c.count, ms});
        }
        for (Strategy s : all) {
            const PartitionPlan plan = make_plan(s, partitions, dims);
            DominanceCounter rc;
            const RepresentativeSet rs = select_representatives(data, reps, sum_score, rc);
            const ParallelSkylineResult r = parallel_skyline(data, plan, rs, cores);
            sky.push_back({strategy_name(s), r.metrics.parallel_max, r.metrics.final_tests,
                           r.metrics.simulated_cost, r.metrics.wall_total_ms});
        }
        std::printf("dataset skyline: %zu tuples\n", skyline.size());
        table("phase: skyline of the full dataset", sky);
        std::vector<Row> gres;
        for (Strategy s : all) {
            const PartitionPlan plan = make_plan(s, partitions, dims);
            const GridResistanceResult g =
                grid_resistance(skyline, plan, reps, s == Strategy::None ? 1 : cores, cap);
            gres.push_back({s == Strategy::None ? "serial" : strategy_name(s),
                            g.metrics.parallel_max_sum, g.metrics.final_sum,
                            g.metrics.simulated_cost, g.metrics.wall_total_ms});
        }
        std::printf("\n");
        table("phase: grid-resistance scan over the skyline", gres);
        return 0;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
}
