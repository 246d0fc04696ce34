// hostgen.cpp — product-side seeded input generators (host, untimed input
// preparation).  Same recipes as the reference (proj/src/datagen.cpp:11-94):
// std::mt19937_64, unit = (x >> 11) * 2^-53, normal = sum of 12 units - 6,
// compiled with -ffp-contract=off so no a*b+c is fused (the reference is
// built without -march; contraction changes ANT bits).
// Kind 2 is the BASELINE C3 correlated generator, which the reference lacks:
// base = unit; v_j = clamp_unit(base + 0.05 * normal).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "skygpu.h"

namespace {

inline double unit(std::mt19937_64& e) { return static_cast<double>(e() >> 11) * 0x1.0p-53; }

inline double normal12(std::mt19937_64& e) {
    double s = 0.0;
    for (int i = 0; i < 12; ++i) s += unit(e);
    return s - 6.0;
}

void put_err(char* err, size_t errlen, const std::string& m) {
    if (!err || !errlen) return;
    size_t k = std::min(errlen - 1, m.size());
    std::memcpy(err, m.data(), k);
    err[k] = 0;
}

}  // namespace

extern "C" int skygpu_generate(int kind, uint64_t n, int d, uint64_t seed, double* out,
                               char* err, size_t errlen) {
    if (d < 1) {
        put_err(err, errlen, "generate: dims must be >= 1");
        return SKYGPU_EINVAL;
    }
    const double below_one = std::nextafter(1.0, 0.0);
    std::mt19937_64 eng(seed);
    std::vector<double> coords(d);
    for (uint64_t i = 0; i < n; ++i) {
        double* row = out + i * static_cast<uint64_t>(d);
        switch (kind) {
            case 0:  // gen_uniform, datagen.cpp:41-54
                for (int j = 0; j < d; ++j) row[j] = unit(eng);
                break;
            case 1: {  // gen_anticorrelated, datagen.cpp:56-90
                double plane = 0.5 * d + 0.015625 * d * normal12(eng);
                plane = std::min(std::max(plane, 0.0), static_cast<double>(d));
                for (int j = 0; j < d; ++j) coords[j] = plane / d;
                if (d > 1) {
                    for (int step = 0; step < 4 * d; ++step) {
                        uint64_t from = eng() % static_cast<uint64_t>(d);
                        uint64_t to = eng() % static_cast<uint64_t>(d - 1);
                        if (to >= from) ++to;
                        double amount = unit(eng) * std::min(coords[from], below_one - coords[to]);
                        coords[from] -= amount;
                        coords[to] += amount;
                    }
                }
                for (int j = 0; j < d; ++j) row[j] = std::min(std::max(coords[j], 0.0), below_one);
                break;
            }
            case 2: {  // BASELINE C3 correlated (new)
                double base = unit(eng);
                for (int j = 0; j < d; ++j) {
                    double nz = normal12(eng);
                    double scaled = 0.05 * nz;
                    row[j] = std::min(std::max(base + scaled, 0.0), below_one);
                }
                break;
            }
            case 3:  // testutil::random_relation(coarse=true), test_util.hpp:38-54
                for (int j = 0; j < d; ++j) {
                    double v = static_cast<double>(eng() >> 11) * 0x1.0p-53;
                    row[j] = std::floor(v * 16.0) / 16.0;
                }
                break;
            default:
                put_err(err, errlen, "generate: unknown kind");
                return SKYGPU_EINVAL;
        }
    }
    put_err(err, errlen, "");
    return SKYGPU_OK;
}
