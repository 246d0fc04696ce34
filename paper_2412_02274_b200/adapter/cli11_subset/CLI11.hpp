// CLI11.hpp — an ORIGINAL, minimal stand-in for the subset of the CLI11
// command-line library that the reference's two tools use
// (proj/tools/skypar_main.cpp:17-79, proj/tools/bench_main.cpp:43-62).  The
// real CLI11 is not vendored in the reference tree (proj/.gitignore:2) and
// there is no network, so the UNMODIFIED tool sources are compiled against
// this header instead (oracle/build_ref.sh: -I .../adapter/cli11_subset).
//
// Covered: CLI::App{description}; add_option(name, var[, description]) for
// integral, std::string and std::vector<...> variables; add_flag(name,
// bool&[, description]); Option::check / delimiter / default_str /
// capture_default_str / excludes; the validators IsMember, PositiveNumber,
// NonNegativeNumber, Range; CLI11_PARSE.  Accepted syntax: "--name value",
// "--name=value", repeated list options append, "-h" / "--help".
// Behaviour on bad input: a one-line message on stderr, exit status 2
// (this shim's own convention); --help prints the option table, status 0.
// default_str only changes the text shown by --help — the variable keeps its
// value (an unset list stays empty, which run_sweep reads as "use the
// default").
#pragma once

// (the real CLI11 is header-only and pulls in these standard headers; the
// reference tools rely on that, e.g. bench_main.cpp uses std::chrono and
// std::printf without including <chrono>/<cstdio> itself)
#include <algorithm>
#include <charconv>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <iomanip>
#include <map>
#include <set>
#include <utility>
#include <cstdint>
#include <cstdio>
#include <functional>
#include <initializer_list>
#include <iostream>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

namespace CLI {

// a failed parse: what to print and the process exit status
struct Error : std::runtime_error {
    int status;
    Error(const std::string& m, int s) : std::runtime_error(m), status(s) {}
};
struct HelpRequest : Error {
    HelpRequest() : Error("help", 0) {}
};

// A validator maps one raw value to "" (accepted) or a message.
struct Validator {
    std::function<std::string(const std::string&)> fn;
    std::string label;  // shown in --help
};

namespace detail {
inline bool to_number(const std::string& s, long double* out) {
    if (s.empty()) return false;
    std::size_t used = 0;
    try {
        *out = std::stold(s, &used);
    } catch (...) {
        return false;
    }
    return used == s.size();
}
inline std::string join(const std::vector<std::string>& xs, const char* sep) {
    std::string r;
    for (std::size_t i = 0; i < xs.size(); ++i) r += (i ? sep : "") + xs[i];
    return r;
}
}  // namespace detail

inline Validator IsMember(std::initializer_list<const char*> allowed) {
    std::vector<std::string> set(allowed.begin(), allowed.end());
    const std::string shown = "{" + detail::join(set, ",") + "}";
    return Validator{[set, shown](const std::string& v) -> std::string {
                         for (const std::string& a : set)
                             if (a == v) return "";
                         return v + " not in " + shown;
                     },
                     shown};
}

inline Validator Range(double lo, double hi) {
    auto num = [](double x) {
        std::ostringstream o;
        if (x == static_cast<double>(static_cast<long long>(x)))
            o << static_cast<long long>(x);
        else
            o << x;
        return o.str();
    };
    std::ostringstream label;
    label << "[" << num(lo) << " - " << num(hi) << "]";
    const std::string shown = label.str();
    return Validator{[lo, hi, shown](const std::string& v) -> std::string {
                         long double x = 0;
                         if (!detail::to_number(v, &x) || x < lo || x > hi)
                             return "value " + v + " not in range " + shown;
                         return "";
                     },
                     shown};
}

inline const Validator PositiveNumber{[](const std::string& v) -> std::string {
                                          long double x = 0;
                                          if (!detail::to_number(v, &x) || !(x > 0))
                                              return "value " + v + " is not positive";
                                          return "";
                                      },
                                      "POSITIVE"};

inline const Validator NonNegativeNumber{[](const std::string& v) -> std::string {
                                             long double x = 0;
                                             if (!detail::to_number(v, &x) || x < 0)
                                                 return "value " + v + " is negative";
                                             return "";
                                         },
                                         "NONNEGATIVE"};

namespace detail {

template <class T>
struct is_vector : std::false_type {};
template <class T, class A>
struct is_vector<std::vector<T, A>> : std::true_type {};

// one raw token -> T (the whole token must be consumed)
template <class T>
bool convert(const std::string& s, T* out) {
    if constexpr (std::is_same_v<T, std::string>) {
        *out = s;
        return true;
    } else if constexpr (std::is_same_v<T, bool>) {
        if (s == "true" || s == "1" || s == "on" || s == "yes") return *out = true, true;
        if (s == "false" || s == "0" || s == "off" || s == "no") return *out = false, true;
        return false;
    } else if constexpr (std::is_integral_v<T>) {
        if (s.empty() || (std::is_unsigned_v<T> && s[0] == '-')) return false;
        const char* b = s.data();
        if (*b == '+') ++b;
        T v{};
        auto r = std::from_chars(b, s.data() + s.size(), v);
        if (r.ec != std::errc() || r.ptr != s.data() + s.size()) return false;
        *out = v;
        return true;
    } else if constexpr (std::is_floating_point_v<T>) {
        long double x = 0;
        if (!to_number(s, &x)) return false;
        *out = static_cast<T>(x);
        return true;
    } else {
        static_assert(sizeof(T) == 0, "CLI11 subset: unsupported option type");
        return false;
    }
}

template <class T>
std::string show(const T& v) {
    if constexpr (std::is_same_v<T, std::string>) {
        return v;
    } else if constexpr (is_vector<T>::value) {
        std::string r;
        for (std::size_t i = 0; i < v.size(); ++i) r += (i ? "," : "") + show(v[i]);
        return r;
    } else if constexpr (std::is_same_v<T, bool>) {
        return v ? "true" : "false";
    } else {
        std::ostringstream o;
        o << v;
        return o.str();
    }
}

}  // namespace detail

class App;

class Option {
  public:
    Option* check(const Validator& v) {
        checks_.push_back(v);
        return this;
    }
    Option* delimiter(char c) {
        delim_ = c;
        return this;
    }
    Option* default_str(const std::string& s) {
        default_ = s;
        return this;
    }
    Option* capture_default_str() {
        if (capture_) default_ = capture_();
        return this;
    }
    Option* excludes(Option* other) {
        excludes_.push_back(other);
        other->excludes_.push_back(this);
        return this;
    }
    const std::string& name() const { return name_; }
    std::size_t count() const { return count_; }

  private:
    friend class App;
    std::string name_, help_, type_, default_;
    bool flag_ = false, list_ = false;
    char delim_ = 0;
    std::size_t count_ = 0;
    std::vector<Validator> checks_;
    std::vector<Option*> excludes_;
    std::function<bool(const std::string&)> store_;  // convert + assign/append one value
    std::function<std::string()> capture_;
};

class App {
  public:
    explicit App(std::string description = "") : desc_(std::move(description)) {}

    template <class T>
    Option* add_option(const std::string& name, T& var, const std::string& help = "") {
        Option* o = make(name, help);
        if constexpr (detail::is_vector<T>::value) {
            using E = typename T::value_type;
            o->list_ = true;
            o->type_ = type_of<E>();
            o->store_ = [&var](const std::string& s) {
                E e{};
                if (!detail::convert(s, &e)) return false;
                var.push_back(e);
                return true;
            };
        } else {
            o->type_ = type_of<T>();
            o->store_ = [&var](const std::string& s) { return detail::convert(s, &var); };
        }
        o->capture_ = [&var] { return detail::show(var); };
        return o;
    }

    Option* add_flag(const std::string& name, bool& var, const std::string& help = "") {
        Option* o = make(name, help);
        o->flag_ = true;
        o->store_ = [&var](const std::string&) {
            var = true;
            return true;
        };
        return o;
    }

    void parse(int argc, char** argv) {
        prog_ = argc > 0 ? argv[0] : "app";
        for (int i = 1; i < argc; ++i) {
            std::string tok = argv[i];
            if (tok == "-h" || tok == "--help") throw HelpRequest();
            std::string val;
            bool has_val = false;
            const std::size_t eq = tok.find('=');
            if (tok.rfind("--", 0) == 0 && eq != std::string::npos) {
                val = tok.substr(eq + 1);
                tok = tok.substr(0, eq);
                has_val = true;
            }
            Option* o = find(tok);
            if (!o) throw Error("unknown option: " + std::string(argv[i]), 2);
            for (Option* x : o->excludes_)
                if (x->count_) throw Error(o->name_ + " excludes " + x->name_, 2);
            ++o->count_;
            if (o->flag_) {
                if (has_val) throw Error(o->name_ + " is a flag and takes no value", 2);
                o->store_("");
                continue;
            }
            if (!has_val) {
                if (i + 1 >= argc) throw Error(o->name_ + " requires a value", 2);
                val = argv[++i];
            }
            std::vector<std::string> parts;
            if (o->list_ && o->delim_) {
                std::size_t a = 0;
                for (;;) {
                    const std::size_t b = val.find(o->delim_, a);
                    parts.push_back(val.substr(a, b == std::string::npos ? b : b - a));
                    if (b == std::string::npos) break;
                    a = b + 1;
                }
            } else {
                parts.push_back(val);
            }
            for (const std::string& p : parts) {
                if (!o->store_(p))
                    throw Error(o->name_ + ": " + p + " is not a valid number / value of type " +
                                    o->type_,
                                2);
                for (const Validator& v : o->checks_) {
                    const std::string m = v.fn(p);
                    if (!m.empty()) throw Error(o->name_ + ": " + m, 2);
                }
            }
        }
    }

    int exit(const Error& e) const {
        if (e.status == 0) {
            std::cout << help();
            return 0;
        }
        std::cerr << e.what() << "\nRun with --help for more information.\n";
        return e.status;
    }

    std::string help() const {
        std::ostringstream o;
        if (!desc_.empty()) o << desc_ << "\n";
        o << "Usage: " << prog_ << " [OPTIONS]\n\nOptions:\n";
        o << "  -h,--help                Print this help message and exit\n";
        for (const auto& p : opts_) {
            std::string left = p->name_;
            if (!p->flag_) left += " " + p->type_ + (p->list_ ? " ..." : "");
            o << "  " << left;
            for (std::size_t k = left.size(); k < 24; ++k) o << ' ';
            o << " " << p->help_;
            for (const Validator& v : p->checks_) o << " " << v.label;
            if (!p->default_.empty()) o << " [" << p->default_ << "]";
            for (const Option* x : p->excludes_) o << " Excludes: " << x->name_;
            o << "\n";
        }
        return o.str();
    }

  private:
    template <class T>
    static std::string type_of() {
        if constexpr (std::is_same_v<T, std::string>) return "TEXT";
        else if constexpr (std::is_integral_v<T> && std::is_unsigned_v<T>) return "UINT";
        else if constexpr (std::is_integral_v<T>) return "INT";
        else return "FLOAT";
    }
    Option* make(const std::string& name, const std::string& help) {
        opts_.push_back(std::make_unique<Option>());
        Option* o = opts_.back().get();
        o->name_ = name;
        o->help_ = help;
        return o;
    }
    Option* find(const std::string& name) {
        for (auto& p : opts_)
            if (p->name_ == name) return p.get();
        return nullptr;
    }
    std::string desc_, prog_ = "app";
    std::vector<std::unique_ptr<Option>> opts_;
};

}  // namespace CLI

#define CLI11_PARSE(app, argc, argv)          \
    try {                                     \
        (app).parse((argc), (argv));          \
    } catch (const CLI::Error& cli_error_) {  \
        return (app).exit(cli_error_);        \
    }
