// refdrive — repo-owned TEST/BASELINE driver that links the UNMODIFIED
// reference library (compiled from /root/reference/proj/src by
// oracle/build_ref.sh into oracle/_ref/).  It is test infrastructure: only
// tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
// reference legs execute it.
//
// Modes
//   golden : run parallel_skyline + grid_resistance on one seeded input and
//            print the results as one JSON object (sorted skyline ids, the
//            skyline in output order, g_max, the denominators map, per-g rows).
//   dump   : write the generated input as raw float64 (generator parity).
//   pids   : the reference's assign_partitions on the generated input (golden
//            partition ids for the device assign_partitions).
//   csv    : parse --input with the reference's load_dataset_csv
//            (harness.cpp:93-134) and print the relation (value bits in hex,
//            ids) or the exception text — golden vectors for the device CSV
//            parser.
//   bench  : time parallel_skyline + grid_resistance with steady_clock on the
//            given core budget, the way proj/tools/bench_main.cpp:66-101 does,
//            generation excluded; print one JSON line.
//
// Inputs: --gen uni|ant (reference generators, proj/src/datagen.cpp:41-94),
// --gen corr (the BASELINE C3 generator, which the reference does not have:
// base = next_unit; v_j = clamp_unit(base + 0.05 * next_normal); identical
// arithmetic to paper_2412_02274_b200's host generator and to oracle/skyoracle.c),
// --gen lattice (testutil::random_relation with coarse=true,
// proj/tests/test_util.hpp:38-54), or --input file.bin (raw little-endian
// float64, n*d row-major; ids = row index).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "skypar/datagen.hpp"
#include "skypar/gres.hpp"
#include "skypar/harness.hpp"
#include "skypar/oracle.hpp"
#include "skypar/parallel.hpp"

using namespace skypar;

namespace {

struct Args {
    std::string mode = "golden";
    std::string gen = "uni";
    std::string input;
    std::size_t n = 1000;
    int d = 3;
    std::uint64_t seed = 1;
    std::string strategy = "none";
    long long p = 1;
    int cores = 1;
    int cap = 25;  // 0 = uncapped
    std::size_t reps = 0;
    bool brute = false;  // also emit brute-force skyline ids / resistance
    bool no_gres = false;
    int repeat = 1;
    std::string out;  // dump mode: raw float64 values written here
};

double unit(std::mt19937_64& e) { return static_cast<double>(e() >> 11) * 0x1.0p-53; }

double normal12(std::mt19937_64& e) {
    double s = 0.0;
    for (int i = 0; i < 12; ++i) s += unit(e);
    return s - 6.0;
}

Relation gen_corr(std::size_t n, int d, std::uint64_t seed) {
    const double below_one = std::nextafter(1.0, 0.0);
    std::mt19937_64 eng(seed);
    Relation r(d);
    r.tuples.reserve(n);
    for (std::size_t i = 0; i < n; ++i) {
        Tuple t;
        t.id = static_cast<std::int64_t>(i);
        double base = unit(eng);
        for (int j = 0; j < d; ++j) {
            double nz = normal12(eng);
            double scaled = 0.05 * nz;
            double v = base + scaled;
            t.values.push_back(std::min(std::max(v, 0.0), below_one));
        }
        r.tuples.push_back(std::move(t));
    }
    return r;
}

Relation gen_lattice(std::size_t n, int d, std::uint64_t seed) {
    std::mt19937_64 rng(seed);
    Relation r(d);
    for (std::size_t i = 0; i < n; ++i) {
        Tuple t;
        t.id = static_cast<std::int64_t>(i);
        for (int j = 0; j < d; ++j) {
            double v = static_cast<double>(rng() >> 11) * 0x1.0p-53;
            v = std::floor(v * 16.0) / 16.0;
            t.values.push_back(v);
        }
        r.tuples.push_back(std::move(t));
    }
    return r;
}

Relation load_input(const Args& a) {
    if (!a.input.empty()) {
        std::ifstream in(a.input, std::ios::binary);
        if (!in) throw std::runtime_error("cannot open " + a.input);
        std::vector<double> buf(a.n * static_cast<std::size_t>(a.d));
        in.read(reinterpret_cast<char*>(buf.data()),
                static_cast<std::streamsize>(buf.size() * sizeof(double)));
        if (!in) throw std::runtime_error("short read from " + a.input);
        Relation r(a.d);
        r.tuples.reserve(a.n);
        for (std::size_t i = 0; i < a.n; ++i) {
            Tuple t;
            t.id = static_cast<std::int64_t>(i);
            t.values.assign(buf.begin() + static_cast<long>(i * a.d),
                            buf.begin() + static_cast<long>((i + 1) * a.d));
            r.add(std::move(t));
        }
        return r;
    }
    if (a.gen == "uni") return generate(GenSpec{a.n, a.d, Distribution::Uniform, a.seed});
    if (a.gen == "ant") return generate(GenSpec{a.n, a.d, Distribution::Anticorrelated, a.seed});
    if (a.gen == "corr") return gen_corr(a.n, a.d, a.seed);
    if (a.gen == "lattice") return gen_lattice(a.n, a.d, a.seed);
    throw std::runtime_error("unknown --gen " + a.gen);
}

Args parse(int argc, char** argv) {
    Args a;
    for (int i = 1; i < argc; ++i) {
        std::string f = argv[i];
        auto next = [&]() -> std::string {
            if (i + 1 >= argc) throw std::runtime_error("missing value for " + f);
            return argv[++i];
        };
        if (f == "--mode") a.mode = next();
        else if (f == "--gen") a.gen = next();
        else if (f == "--input") a.input = next();
        else if (f == "--n") a.n = std::stoull(next());
        else if (f == "--d") a.d = std::stoi(next());
        else if (f == "--seed") a.seed = std::stoull(next());
        else if (f == "--strategy") a.strategy = next();
        else if (f == "--p") a.p = std::stoll(next());
        else if (f == "--cores") a.cores = std::stoi(next());
        else if (f == "--cap") a.cap = std::stoi(next());
        else if (f == "--reps") a.reps = std::stoull(next());
        else if (f == "--repeat") a.repeat = std::stoi(next());
        else if (f == "--out") a.out = next();
        else if (f == "--brute") a.brute = true;
        else if (f == "--no-gres") a.no_gres = true;
        else throw std::runtime_error("unknown flag " + f);
    }
    if (a.cores <= 0) a.cores = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
    return a;
}

std::string cpu_model() {
    std::ifstream in("/proc/cpuinfo");
    std::string line;
    while (std::getline(in, line))
        if (line.rfind("model name", 0) == 0) {
            auto c = line.find(':');
            std::string m = line.substr(c + 2);
            std::string out;
            for (char ch : m) out += (ch == '"' ? '\'' : ch);
            return out;
        }
    return "unknown";
}

void print_ids(const char* key, const std::vector<std::int64_t>& v) {
    std::printf("\"%s\":[", key);
    for (std::size_t i = 0; i < v.size(); ++i) std::printf(i ? ",%lld" : "%lld", (long long)v[i]);
    std::printf("]");
}

int run_golden(const Args& a) {
    Relation data = load_input(a);
    PartitionPlan plan = make_plan(strategy_from_name(a.strategy), a.p, a.d);
    DominanceCounter rc;
    RepresentativeSet reps = select_representatives(data, a.reps, sum_score, rc);
    ParallelSkylineResult sky = parallel_skyline(data, plan, reps, a.cores);
    std::vector<std::int64_t> order, sorted;
    for (const Tuple& t : sky.skyline.tuples) order.push_back(t.id);
    sorted = order;
    std::sort(sorted.begin(), sorted.end());
    std::printf("{\"n\":%zu,\"d\":%d,\"gen\":\"%s\",\"seed\":%llu,\"strategy\":\"%s\",\"p\":%lld,"
                "\"slices\":%d,\"partitions\":%lld,\"cap\":%d,\"reps\":%zu,",
                data.size(), a.d, a.input.empty() ? a.gen.c_str() : "file",
                (unsigned long long)a.seed, a.strategy.c_str(), a.p, plan.slices, plan.partitions,
                a.cap, a.reps);
    print_ids("skyline_ids", sorted);
    std::printf(",");
    print_ids("skyline_order", order);
    if (a.brute) {
        std::vector<std::int64_t> bf;
        for (const Tuple& t : skyline_bruteforce(data).tuples) bf.push_back(t.id);
        std::sort(bf.begin(), bf.end());
        std::printf(",");
        print_ids("bruteforce_ids", bf);
    }
    if (!a.no_gres) {
        std::optional<int> cap;
        if (a.cap > 0) cap = a.cap;
        GridResistanceResult g;
        try {
            g = grid_resistance(sky.skyline, plan, a.reps, a.cores, cap);
        } catch (const std::exception& e) {
            std::printf(",\"gres_error\":\"%s\"}\n", e.what());
            return 0;
        }
        std::printf(",\"g_max\":%d,\"den\":[", g.metrics.g_max);
        bool first = true;
        for (const auto& [id, den] : g.denominators) {
            std::printf(first ? "[%lld,%d]" : ",[%lld,%d]", (long long)id, den);
            first = false;
        }
        std::printf("],\"rows\":[");
        for (std::size_t i = 0; i < g.metrics.iterations.size(); ++i)
            std::printf(i ? ",%d" : "%d", g.metrics.iterations[i].intervals);
        std::printf("]");
        if (a.brute) {
            std::printf(",\"bruteforce_den\":[");
            bool f2 = true;
            for (const Tuple& t : sky.skyline.tuples) {
                int den = grid_resistance_bruteforce(t, data, cap);
                std::printf(f2 ? "[%lld,%d]" : ",[%lld,%d]", (long long)t.id, den);
                f2 = false;
            }
            std::printf("]");
        }
    }
    std::printf("}\n");
    return 0;
}

// pids: the reference's own assign_partitions (partition.cpp:183-213) on the
// generated input — golden partition ids for the device assign_partitions
int run_pids(const Args& a) {
    Relation data = load_input(a);
    PartitionPlan plan = make_plan(strategy_from_name(a.strategy), a.p, a.d);
    std::printf("{\"n\":%zu,\"d\":%d,\"gen\":\"%s\",\"seed\":%llu,\"strategy\":\"%s\","
                "\"p\":%lld,\"slices\":%d,\"partitions\":%lld,",
                data.size(), a.d, a.input.empty() ? a.gen.c_str() : "file",
                (unsigned long long)a.seed, a.strategy.c_str(), a.p, plan.slices, plan.partitions);
    try {
        const std::vector<long long> ids = assign_partitions(data, plan);
        std::printf("\"pids\":[");
        for (std::size_t i = 0; i < ids.size(); ++i) std::printf(i ? ",%lld" : "%lld", ids[i]);
        std::printf("]}\n");
    } catch (const std::exception& e) {
        std::printf("\"pids_error\":\"%s\"}\n", e.what());
    }
    return 0;
}

int run_dump(const Args& a) {
    Relation data = load_input(a);
    std::ofstream out(a.out, std::ios::binary);
    if (!out) throw std::runtime_error("cannot write " + a.out);
    for (const Tuple& t : data.tuples)
        out.write(reinterpret_cast<const char*>(t.values.data()),
                  static_cast<std::streamsize>(t.values.size() * sizeof(double)));
    std::printf("{\"n\":%zu,\"d\":%d}\n", data.size(), a.d);
    return 0;
}

int run_bench(const Args& a) {
    Relation data = load_input(a);
    PartitionPlan plan = make_plan(strategy_from_name(a.strategy), a.p, a.d);
    std::optional<int> cap;
    if (a.cap > 0) cap = a.cap;
    double best_sky = 1e300, best_gres = 1e300, tot_sky = 0, tot_gres = 0;
    std::size_t S = 0;
    int g_max = 0;
    std::uint64_t gres_tests = 0, sky_tests = 0;
    for (int rep = 0; rep < a.repeat; ++rep) {
        auto t0 = std::chrono::steady_clock::now();
        DominanceCounter rc;
        RepresentativeSet reps = select_representatives(data, a.reps, sum_score, rc);
        ParallelSkylineResult sky = parallel_skyline(data, plan, reps, a.cores);
        auto t1 = std::chrono::steady_clock::now();
        double gms = 0;
        if (!a.no_gres) {
            GridResistanceResult g = grid_resistance(sky.skyline, plan, a.reps, a.cores, cap);
            auto t2 = std::chrono::steady_clock::now();
            gms = std::chrono::duration<double, std::milli>(t2 - t1).count();
            g_max = g.metrics.g_max;
            gres_tests = 0;
            for (const auto& it : g.metrics.iterations) gres_tests += it.final_tests;
            for (const auto& it : g.metrics.iterations) gres_tests += it.parallel_max;
        }
        double sms = std::chrono::duration<double, std::milli>(t1 - t0).count();
        S = sky.skyline.size();
        sky_tests = sky.metrics.final_tests;
        for (auto c : sky.metrics.per_partition_tests) sky_tests += c;
        best_sky = std::min(best_sky, sms);
        best_gres = std::min(best_gres, gms);
        tot_sky += sms;
        tot_gres += gms;
    }
    std::printf("{\"n\":%zu,\"d\":%d,\"gen\":\"%s\",\"strategy\":\"%s\",\"partitions\":%lld,"
                "\"cores\":%d,\"hw_threads\":%u,\"cpu\":\"%s\",\"skyline_size\":%zu,\"g_max\":%d,"
                "\"repeat\":%d,\"skyline_ms_mean\":%.6f,\"gres_ms_mean\":%.6f,"
                "\"skyline_ms_best\":%.6f,\"gres_ms_best\":%.6f,\"skyline_tests\":%llu,"
                "\"gres_tests_partition_max_plus_final\":%llu}\n",
                data.size(), a.d, a.input.empty() ? a.gen.c_str() : "file", a.strategy.c_str(),
                plan.partitions, a.cores, std::thread::hardware_concurrency(), cpu_model().c_str(),
                S, g_max, a.repeat, tot_sky / a.repeat, tot_gres / a.repeat, best_sky, best_gres,
                (unsigned long long)sky_tests, (unsigned long long)gres_tests);
    return 0;
}

std::string json_escape(const std::string& in) {
    std::string out;
    for (unsigned char ch : in) {
        if (ch == '"' || ch == '\\') {
            out += '\\';
            out += (char)ch;
        } else if (ch < 0x20 || ch >= 0x7f) {
            char buf[8];
            std::snprintf(buf, sizeof(buf), "\\u%04x", ch);
            out += buf;
        } else {
            out += (char)ch;
        }
    }
    return out;
}

int run_csv(const Args& a) {
    try {
        const Relation r = load_dataset_csv(a.input);
        std::printf("{\"rows\":%zu,\"dims\":%zu,\"ids\":[", r.size(), r.dims);
        for (std::size_t i = 0; i < r.size(); ++i)
            std::printf("%s%lld", i ? "," : "", (long long)r.tuples[i].id);
        std::printf("],\"bits\":[");
        bool first = true;
        for (const Tuple& t : r.tuples)
            for (double v : t.values) {
                std::uint64_t b;
                std::memcpy(&b, &v, 8);
                std::printf("%s\"%016llx\"", first ? "" : ",", (unsigned long long)b);
                first = false;
            }
        std::printf("]}\n");
    } catch (const std::exception& e) {
        std::printf("{\"csv_error\":\"%s\"}\n", json_escape(e.what()).c_str());
    }
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    try {
        Args a = parse(argc, argv);
        if (a.mode == "golden") return run_golden(a);
        if (a.mode == "bench") return run_bench(a);
        if (a.mode == "dump") return run_dump(a);
        if (a.mode == "pids") return run_pids(a);
        if (a.mode == "csv") return run_csv(a);
        throw std::runtime_error("unknown --mode " + a.mode);
    } catch (const std::exception& e) {
        std::printf("{\"error\":\"%s\"}\n", e.what());
        return 3;
    }
}
