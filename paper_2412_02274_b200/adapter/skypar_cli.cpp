// skypar_cli.cpp — the `skypar` command-line front end (SURVEY.md §8(f) rank
// 1) with a hand-written argument parser (the reference's CLI11 is absent
// here).  Same flags, list semantics and defaults as proj/tools/skypar_main.cpp:28-77:
// every list flag takes comma-separated values (or several values) and the
// full cross-product is run through the reference's own run_sweep
// (proj/src/harness.cpp:299-310), one report per combination.
//
// Linked two ways by oracle/build_ref.sh:
//   oracle/_ref/skypar_gpu — reference harness/metrics objects + the GPU
//                            drop-in (adapter/skypar_gpu.cpp, libskygpu.so)
//   oracle/_ref/skypar_ref — the same main over the unmodified CPU library
// so the two binaries' report files can be compared byte for byte.
#include <cstdint>
#include <cstdlib>
#include <iostream>
#include <optional>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "skypar/harness.hpp"

namespace {

struct UsageError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

const char* kHelp =
    "skyline and grid-resistance benchmark\n"
    "Usage: skypar [OPTIONS]\n\n"
    "Options:\n"
    "  -h,--help            Print this help message and exit\n"
    "  --dataset TEXT       CSV dataset file (header + numeric rows); excludes --gen\n"
    "  --gen TEXT           generate a synthetic dataset: uni|ant; excludes --dataset\n"
    "  --n UINT,...         generated tuple count (list sweeps) [1000000]\n"
    "  --d UINT,...         generated dimension count (list sweeps) [3]\n"
    "  --seed UINT          base seed; instance i uses seed+i [1]\n"
    "  --strategy TEXT,...  partitioning: none|grid|angular|sliced (list sweeps) [none]\n"
    "  --partitions UINT,.. target partition count (list sweeps) [16]\n"
    "  --reps UINT,...      representative tuples for pre-filtering (list sweeps) [0]\n"
    "  --cores UINT,...     core budget for the parallel phase (list sweeps) [16]\n"
    "  --cap INT            ceiling for the grid interval bound, in [2, 1000000] [25]\n"
    "  --repeat UINT        instances to generate and average [1]\n"
    "  --normalize          min-max scale each attribute to [0,1]\n"
    "  --out TEXT           report file (stdout when omitted)\n"
    "  --format TEXT        report format: csv|jsonl [csv]\n"
    "  --mode TEXT          skyline: stop after the dataset skyline; gres: full scan [gres]\n"
    "  --oracle             cross-check results against the brute-force reference\n";

template <class T>
T parse_number(const std::string& flag, const std::string& text) {
    if (text.empty()) throw UsageError(flag + ": empty value");
    std::istringstream in(text);
    T v{};
    in >> v;
    if (!in || !in.eof()) throw UsageError(flag + ": " + text + " is not a valid number");
    if constexpr (std::is_unsigned_v<T>)
        if (text[0] == '-') throw UsageError(flag + ": " + text + " is not a valid number");
    return v;
}

void require_member(const std::string& flag, const std::string& v,
                    const std::vector<std::string>& allowed) {
    for (const std::string& a : allowed)
        if (v == a) return;
    std::string set;
    for (const std::string& a : allowed) set += (set.empty() ? "" : ",") + a;
    throw UsageError(flag + ": " + v + " not in {" + set + "}");
}

// split "a,b" and gather further non-flag arguments into one list
std::vector<std::string> split_values(const std::vector<std::string>& raw) {
    std::vector<std::string> out;
    for (const std::string& r : raw) {
        std::size_t start = 0;
        while (true) {
            const std::size_t comma = r.find(',', start);
            out.push_back(r.substr(start, comma == std::string::npos ? std::string::npos
                                                                     : comma - start));
            if (comma == std::string::npos) break;
            start = comma + 1;
        }
    }
    return out;
}

}  // namespace

int main(int argc, char** argv) {
    std::string dataset_path, gen_name, format_name = "csv", out_path;
    std::vector<std::string> strategy_names;
    skypar::SweepConfig sweep;
    skypar::ExperimentConfig& cfg = sweep.base;
    int cap = 25;
    try {
        std::vector<std::string> args(argv + 1, argv + argc);
        bool saw_dataset = false, saw_gen = false;
        for (std::size_t i = 0; i < args.size(); ++i) {
            std::string flag = args[i];
            std::vector<std::string> vals;
            const std::size_t eq = flag.find('=');
            if (flag.rfind("--", 0) == 0 && eq != std::string::npos) {
                vals.push_back(flag.substr(eq + 1));
                flag = flag.substr(0, eq);
            }
            if (flag == "-h" || flag == "--help") {
                std::cout << kHelp;
                return 0;
            }
            const bool is_flag = flag == "--normalize" || flag == "--oracle";
            if (is_flag) {
                if (!vals.empty()) throw UsageError(flag + ": takes no value");
                (flag == "--normalize" ? cfg.normalize_input : cfg.oracle_check) = true;
                continue;
            }
            if (flag.rfind("--", 0) != 0) throw UsageError("unexpected argument: " + flag);
            static const char* kKnown[] = {"--dataset", "--gen",  "--n",   "--d",      "--seed",
                                           "--strategy", "--partitions", "--reps", "--cores",
                                           "--cap",     "--repeat", "--out", "--format", "--mode"};
            bool known = false;
            for (const char* k : kKnown) known |= flag == k;
            if (!known) throw UsageError("unknown option: " + flag);
            const bool is_list = flag == "--n" || flag == "--d" || flag == "--strategy" ||
                                 flag == "--partitions" || flag == "--reps" || flag == "--cores";
            if (vals.empty()) {
                while (i + 1 < args.size() && args[i + 1].rfind("--", 0) != 0) {
                    vals.push_back(args[++i]);
                    if (!is_list) break;
                }
            }
            if (vals.empty()) throw UsageError(flag + ": requires a value");
            const std::vector<std::string> items = is_list ? split_values(vals) : vals;
            if (flag == "--dataset") {
                dataset_path = items[0];
                saw_dataset = true;
            } else if (flag == "--gen") {
                require_member(flag, items[0], {"uni", "ant"});
                gen_name = items[0];
                saw_gen = true;
            } else if (flag == "--n") {
                for (const auto& v : items) sweep.n_values.push_back(parse_number<std::size_t>(flag, v));
            } else if (flag == "--d") {
                for (const auto& v : items) {
                    const int x = parse_number<int>(flag, v);
                    if (x <= 0) throw UsageError(flag + ": value " + v + " is not positive");
                    sweep.dim_values.push_back(x);
                }
            } else if (flag == "--seed") {
                cfg.seed = parse_number<std::uint64_t>(flag, items[0]);
            } else if (flag == "--strategy") {
                for (const auto& v : items) {
                    require_member(flag, v, {"none", "grid", "angular", "sliced"});
                    strategy_names.push_back(v);
                }
            } else if (flag == "--partitions") {
                for (const auto& v : items) {
                    const long long x = parse_number<long long>(flag, v);
                    if (x <= 0) throw UsageError(flag + ": value " + v + " is not positive");
                    sweep.partition_targets.push_back(x);
                }
            } else if (flag == "--reps") {
                for (const auto& v : items) {
                    const int x = parse_number<int>(flag, v);
                    if (x < 0) throw UsageError(flag + ": value " + v + " is negative");
                    sweep.rep_counts.push_back(x);
                }
            } else if (flag == "--cores") {
                for (const auto& v : items) {
                    const int x = parse_number<int>(flag, v);
                    if (x <= 0) throw UsageError(flag + ": value " + v + " is not positive");
                    sweep.core_budgets.push_back(x);
                }
            } else if (flag == "--cap") {
                cap = parse_number<int>(flag, items[0]);
                if (cap < 2 || cap > 1000000)
                    throw UsageError(flag + ": value " + items[0] + " not in range [2 - 1000000]");
            } else if (flag == "--repeat") {
                cfg.repetitions = parse_number<int>(flag, items[0]);
                if (cfg.repetitions <= 0)
                    throw UsageError(flag + ": value " + items[0] + " is not positive");
            } else if (flag == "--out") {
                out_path = items[0];
            } else if (flag == "--format") {
                require_member(flag, items[0], {"csv", "jsonl"});
                format_name = items[0];
            } else if (flag == "--mode") {
                require_member(flag, items[0], {"skyline", "gres"});
                cfg.mode = items[0];
            } else {
                throw UsageError("unknown option: " + flag);
            }
        }
        if (saw_dataset && saw_gen) throw UsageError("--dataset excludes --gen");
    } catch (const UsageError& e) {
        std::cerr << e.what() << "\nRun with --help for more information.\n";
        return 2;
    }

    try {
        if (!dataset_path.empty()) cfg.dataset_path = dataset_path;
        if (!gen_name.empty()) cfg.gen = skypar::distribution_from_name(gen_name);
        if (!cfg.dataset_path && !cfg.gen)
            throw std::runtime_error("one of --dataset and --gen is required");
        for (const std::string& name : strategy_names)
            sweep.strategies.push_back(skypar::strategy_from_name(name));
        cfg.format = skypar::report_format_from_name(format_name);
        cfg.cap = cap;
        if (!out_path.empty()) cfg.out_path = out_path;
        const std::vector<skypar::RunReport> reports = skypar::run_sweep(sweep);
        if (!cfg.out_path) std::cout << skypar::serialize_reports(reports, cfg.format);
        for (const skypar::RunReport& r : reports)
            std::cerr << r.dataset << " " << r.strategy << " p=" << r.partitions
                      << " rep=" << r.rep_requested << " cores=" << r.cores << ": skyline size "
                      << r.skyline_size << ", simulated cost " << r.simulated_cost << " over "
                      << r.instances << " instance(s)\n";
        return 0;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << '\n';
        return 1;
    }
}
