/*
 * skyoracle.c — CPU restatement of the reference's hot path, used ONLY as the
 * parity checker (tests/, __graft_entry__.smoke(), bench.py cpu_baseline).
 * It is TEST INFRASTRUCTURE: the product path (paper_2412_02274_b200) never
 * links, imports or executes it.
 *
 * Parity is PINNED: tests/test_oracle_golden.py checks every function below
 * against golden vectors emitted by the unmodified reference library
 * (oracle/build_ref.sh + oracle/refdrive.cpp -> tests/golden/*.json, script
 * tests/golden/make_golden.py) and against the reference's own known-answer
 * tests (proj/tests/test_gres.cpp:26-73, test_core.cpp:61-133,
 * test_datagen.cpp:43-58, test_partition.cpp:109-131).
 *
 * Compile with -ffp-contract=off: the reference is built without -march, so
 * its x86-64 code never contracts a*b+c (proj/CMakeLists.txt:8-14), and the
 * generators contain contractible expressions (datagen.cpp:67,77-79).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- PRNG --- */
/* std::mt19937_64 as fixed by the C++ standard ([rand.predef]); the
 * reference draws all randomness from it (datagen.cpp:1-27). */
typedef struct {
    uint64_t mt[312];
    int idx;
} so_mt64;

static void mt_seed(so_mt64* m, uint64_t seed) {
    m->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        m->mt[i] = 6364136223846793005ULL * (m->mt[i - 1] ^ (m->mt[i - 1] >> 62)) + (uint64_t)i;
    m->idx = 312;
}

static uint64_t mt_next(so_mt64* m) {
    if (m->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            uint64_t x = (m->mt[i] & 0xFFFFFFFF80000000ULL) | (m->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
            uint64_t xa = x >> 1;
            if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
            m->mt[i] = m->mt[(i + 156) % 312] ^ xa;
        }
        m->idx = 0;
    }
    uint64_t y = m->mt[m->idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}

uint64_t so_mt64_nth(uint64_t seed, uint64_t n) { /* n-th draw, 1-based */
    so_mt64 m;
    mt_seed(&m, seed);
    uint64_t v = 0;
    for (uint64_t i = 0; i < n; ++i) v = mt_next(&m);
    return v;
}

/* datagen.cpp:11-13 */
static double next_unit(so_mt64* m) { return (double)(mt_next(m) >> 11) * 0x1.0p-53; }
/* datagen.cpp:19-23 */
static double next_normal(so_mt64* m) {
    double s = 0.0;
    for (int i = 0; i < 12; ++i) s += next_unit(m);
    return s - 6.0;
}
static double below_one(void) { return nextafter(1.0, 0.0); }
/* datagen.cpp:25-27: std::min(std::max(v, 0.0), kBelowOne) */
static double clamp_unit(double v) {
    double a = (v < 0.0) ? 0.0 : v; /* std::max(v, 0.0) returns v unless v < 0 */
    double b1 = below_one();
    return (b1 < a) ? b1 : a;        /* std::min(a, b) returns b iff b < a */
}

/* kind: 0 = uni (datagen.cpp:41-54), 1 = ant (datagen.cpp:56-90),
 *       2 = corr (BASELINE C3, new: base = unit; v_j = clamp(base + 0.05*normal)),
 *       3 = lattice (proj/tests/test_util.hpp:38-54, coarse = true) */
int so_generate(int kind, uint64_t n, int d, uint64_t seed, double* out) {
    if (d < 1) return -1;
    so_mt64 m;
    mt_seed(&m, seed);
    const double b1 = below_one();
    double coords[64];
    if (d > 64) return -1;
    for (uint64_t i = 0; i < n; ++i) {
        double* row = out + i * (uint64_t)d;
        if (kind == 0) {
            for (int j = 0; j < d; ++j) row[j] = next_unit(&m);
        } else if (kind == 1) {
            double plane = 0.5 * d + 0.015625 * d * next_normal(&m);
            /* std::min(std::max(plane, 0.0), double(d)) */
            if (plane < 0.0) plane = 0.0;
            if ((double)d < plane) plane = (double)d;
            for (int j = 0; j < d; ++j) coords[j] = plane / d;
            if (d > 1) {
                for (int step = 0; step < 4 * d; ++step) {
                    uint64_t from = mt_next(&m) % (uint64_t)d;
                    uint64_t to = mt_next(&m) % (uint64_t)(d - 1);
                    if (to >= from) ++to;
                    double room = b1 - coords[to];
                    double lim = (room < coords[from]) ? room : coords[from]; /* std::min */
                    double amount = next_unit(&m) * lim;
                    coords[from] -= amount;
                    coords[to] += amount;
                }
            }
            for (int j = 0; j < d; ++j) row[j] = clamp_unit(coords[j]);
        } else if (kind == 2) {
            double base = next_unit(&m);
            for (int j = 0; j < d; ++j) {
                double nz = next_normal(&m);
                double scaled = 0.05 * nz;
                row[j] = clamp_unit(base + scaled);
            }
        } else if (kind == 3) {
            for (int j = 0; j < d; ++j) {
                double v = (double)(mt_next(&m) >> 11) * 0x1.0p-53;
                row[j] = floor(v * 16.0) / 16.0;
            }
        } else {
            return -1;
        }
    }
    return 0;
}

/* ------------------------------------------------------------ dominance --- */
/* core.hpp:55-67 (without the counter): t dominates s */
static int dominates(const double* t, const double* s, int d) {
    int strict = 0;
    for (int i = 0; i < d; ++i) {
        if (t[i] > s[i]) return 0;
        if (t[i] < s[i]) strict = 1;
    }
    return strict;
}

/* core.cpp:21-23: std::accumulate from 0.0, left to right */
static double sum_score(const double* t, int d) {
    double s = 0.0;
    for (int i = 0; i < d; ++i) s += t[i];
    return s;
}

typedef struct {
    double score;
    int64_t id;
    uint64_t idx;
} scored;

static int cmp_scored(const void* a, const void* b) {
    const scored* x = (const scored*)a;
    const scored* y = (const scored*)b;
    if (x->score != y->score) return x->score < y->score ? -1 : 1;
    if (x->id != y->id) return x->id < y->id ? -1 : 1;
    /* equal (score, id) only with duplicate ids: std::sort leaves this
     * unspecified; fix it to input order */
    return x->idx < y->idx ? -1 : (x->idx > y->idx);
}

/* core.cpp:48-73 skyline_sfs: sort by (sum, id), window filter; the window
 * only grows.  parallel_skyline (parallel.cpp:22-101) returns the same set
 * in the same (sum, id) order for every plan (predecessor rule).
 * out_pos receives input positions of skyline tuples in output order. */
int so_skyline_sfs(const double* v, const int64_t* ids, uint64_t n, int d, uint64_t* out_pos,
                   uint64_t* out_n, uint64_t* tests) {
    scored* o = (scored*)malloc(sizeof(scored) * (n ? n : 1));
    uint64_t* win = (uint64_t*)malloc(sizeof(uint64_t) * (n ? n : 1));
    if (!o || !win) return -2;
    for (uint64_t i = 0; i < n; ++i) {
        o[i].score = sum_score(v + i * d, d);
        o[i].id = ids[i];
        o[i].idx = i;
    }
    qsort(o, n, sizeof(scored), cmp_scored);
    uint64_t w = 0, cnt = 0;
    for (uint64_t k = 0; k < n; ++k) {
        const double* t = v + o[k].idx * d;
        int dom = 0;
        for (uint64_t j = 0; j < w; ++j) {
            ++cnt;
            if (dominates(v + win[j] * d, t, d)) {
                dom = 1;
                break;
            }
        }
        if (!dom) win[w++] = o[k].idx;
    }
    memcpy(out_pos, win, sizeof(uint64_t) * w);
    *out_n = w;
    if (tests) *tests = cnt;
    free(o);
    free(win);
    return 0;
}

/* oracle.cpp:34-47 skyline_bruteforce: keep t iff no s dominates t (input order) */
int so_skyline_bruteforce(const double* v, uint64_t n, int d, uint64_t* out_pos, uint64_t* out_n) {
    uint64_t w = 0;
    for (uint64_t i = 0; i < n; ++i) {
        int dom = 0;
        for (uint64_t j = 0; j < n && !dom; ++j) dom = dominates(v + j * d, v + i * d, d);
        if (!dom) out_pos[w++] = i;
    }
    *out_n = w;
    return 0;
}

/* ------------------------------------------------------------------ gres --- */
static int cmp_double(const void* a, const void* b) {
    double x = *(const double*)a, y = *(const double*)b;
    return (x < y) ? -1 : (y < x);
}

/* gres.cpp:15-28 min_positive_gap; returns 1 and *gap when a gap exists */
int so_min_positive_gap(const double* v, uint64_t n, int d, double* gap) {
    double best = INFINITY;
    double* col = (double*)malloc(sizeof(double) * (n ? n : 1));
    for (int j = 0; j < d; ++j) {
        for (uint64_t i = 0; i < n; ++i) col[i] = v[i * d + j];
        qsort(col, n, sizeof(double), cmp_double);
        for (uint64_t i = 1; i < n; ++i) {
            double g = col[i] - col[i - 1];
            if (g > 0.0 && g < best) best = g;
        }
    }
    free(col);
    if (!isfinite(best)) return 0;
    *gap = best;
    return 1;
}

/* gres.cpp:30-37 intervals_from_gap; cap <= 0 means "no cap".
 * returns 0, or -3 on the overflow error */
int so_intervals_from_gap(double gap, int cap, int* out) {
    if (cap > 0 && 1.0 / gap >= (double)cap) {
        *out = cap;
        return 0;
    }
    double bound = floor(1.0 / gap);
    if (bound > 2147483647.0) return -3;
    *out = (int)bound;
    return 0;
}

/* gres.cpp:57-63 max_grid_intervals: -4 = all attributes constant, -3 = overflow */
int so_max_grid_intervals(const double* v, uint64_t n, int d, int cap, int* out) {
    double gap;
    if (!so_min_positive_gap(v, n, d, &gap)) return -4;
    return so_intervals_from_gap(gap, cap, out);
}

/* gres.cpp:41-48 snap_to_grid */
void so_snap(const double* v, uint64_t cnt, int g, double* out) {
    for (uint64_t i = 0; i < cnt; ++i) out[i] = floor(v[i] * (double)g) / (double)g;
}

/* gres.cpp:65-129 grid_resistance: descending-g scan, each step the SFS
 * skyline of the projected relation (parallel.cpp:22-101 == skyline_sfs
 * set-wise); den[i] for sky tuple i (input order) = the largest g whose
 * projection ejects it, else 1.  Returns 0 or -3 (overflow, no cap). */
int so_grid_resistance(const double* sky, const int64_t* ids, uint64_t s, int d, int cap,
                       int32_t* den, int* g_max_out, uint64_t* tests) {
    int g_max = 1;
    *g_max_out = 1;
    if (s == 0) return 0;
    double gap;
    if (so_min_positive_gap(sky, s, d, &gap)) {
        int rc = so_intervals_from_gap(gap, cap, &g_max);
        if (rc) return rc;
    }
    *g_max_out = g_max;
    double* proj = (double*)malloc(sizeof(double) * s * d);
    uint64_t* pos = (uint64_t*)malloc(sizeof(uint64_t) * s);
    char* alive = (char*)malloc(s);
    for (uint64_t i = 0; i < s; ++i) den[i] = 0;
    uint64_t total = 0;
    for (int g = g_max; g >= 2; --g) {
        so_snap(sky, s * d, g, proj);
        uint64_t m = 0, t = 0;
        so_skyline_sfs(proj, ids, s, d, pos, &m, &t);
        total += t;
        memset(alive, 0, s);
        for (uint64_t k = 0; k < m; ++k) alive[pos[k]] = 1;
        for (uint64_t i = 0; i < s; ++i)
            if (!alive[i] && den[i] == 0) den[i] = g;
    }
    for (uint64_t i = 0; i < s; ++i)
        if (den[i] == 0) den[i] = 1;
    if (tests) *tests = total;
    free(proj);
    free(pos);
    free(alive);
    return 0;
}

/* oracle.cpp:49-86 grid_resistance_bruteforce for tuple t against relation r.
 * returns den >= 1, or -5 when the uncapped bound is too large */
int so_gres_bruteforce(const double* t, const double* r, uint64_t n, int d, int cap) {
    double min_gap = INFINITY;
    for (uint64_t a = 0; a < n; ++a)
        for (uint64_t b = a + 1; b < n; ++b)
            for (int j = 0; j < d; ++j) {
                double gp = fabs(r[a * d + j] - r[b * d + j]);
                if (gp > 0.0 && gp < min_gap) min_gap = gp;
            }
    int g_max;
    if (!isfinite(min_gap)) g_max = 1;
    else if (cap > 0 && 1.0 / min_gap >= (double)cap) g_max = cap;
    else if (1.0 / min_gap > 1e6) return -5;
    else g_max = (int)floor(1.0 / min_gap);
    double pt[64], ps[64];
    int best = 1;
    for (int g = 2; g <= g_max; ++g) {
        so_snap(t, d, g, pt);
        int dom = 0;
        for (uint64_t k = 0; k < n && !dom; ++k) {
            so_snap(r + k * d, d, g, ps);
            dom = dominates(ps, pt, d);
        }
        if (dom) best = g;
    }
    return best;
}

/* Independent S-independent check of the gres stage:
 * at step g, t is ejected iff some occupied code cell c' <= c(t), c' != c(t),
 * i.e. OR_j P[c(t) - e_j] with P the inclusive prefix-OR of the occupancy.
 * Codes k = floor(v*g) (strict order of k == strict order of k/g for
 * k < 2^52).  Rows are u64 bitmasks along attribute 0 (extent <= 64).
 * den must be pre-sized s; g_max given.  Returns 0, or -6 if unsupported. */
/* The same scan over a SUBSET of the steps (descending list): a shard of the
 * step-split resistance engine; den = the largest listed step at which the
 * tuple is dominated, else 1 (the MAX over shards covering every step is
 * the full scan's map). */
int so_gres_cells_steps(const double* sky, uint64_t s, int d, const int* steps, int nsteps,
                        int32_t* den);

int so_gres_cells(const double* sky, uint64_t s, int d, int g_max, int32_t* den) {
    int steps[4096];
    int n = 0;
    for (int g = g_max; g >= 2 && n < 4096; --g) steps[n++] = g;
    if (g_max - 1 > 4096) return -6;
    return so_gres_cells_steps(sky, s, d, steps, n, den);
}

int so_gres_cells_steps(const double* sky, uint64_t s, int d, const int* steps, int nsteps,
                        int32_t* den) {
    for (uint64_t i = 0; i < s; ++i) den[i] = 0;
    if (d < 1 || d > 16) return -6;
    uint32_t* codes = (uint32_t*)malloc(sizeof(uint32_t) * (s ? s : 1) * d);
    for (int si = 0; si < nsteps; ++si) {
        const int g = steps[si];
        uint64_t ext[16];
        for (int j = 0; j < d; ++j) ext[j] = 1;
        for (uint64_t i = 0; i < s; ++i)
            for (int j = 0; j < d; ++j) {
                double k = floor(sky[i * d + j] * (double)g);
                if (k > 4.0e9) {
                    free(codes);
                    return -6;
                }
                codes[i * d + j] = (uint32_t)k;
                if (codes[i * d + j] + 1 > ext[j]) ext[j] = codes[i * d + j] + 1;
            }
        if (ext[0] > 64) {
            free(codes);
            return -6;
        }
        uint64_t rows = 1, stride[16];
        for (int j = 1; j < d; ++j) {
            stride[j] = rows;
            rows *= ext[j];
            if (rows > (1ULL << 34)) {
                free(codes);
                return -6;
            }
        }
        uint64_t* P = (uint64_t*)calloc(rows, sizeof(uint64_t));
        if (!P) {
            free(codes);
            return -6;
        }
        for (uint64_t i = 0; i < s; ++i) {
            uint64_t r = 0;
            for (int j = 1; j < d; ++j) r += codes[i * d + j] * stride[j];
            P[r] |= 1ULL << codes[i * d];
        }
        for (uint64_t r = 0; r < rows; ++r) { /* prefix-OR along attribute 0 */
            uint64_t x = P[r];
            x |= x << 1; x |= x << 2; x |= x << 4; x |= x << 8; x |= x << 16; x |= x << 32;
            P[r] = x;
        }
        for (int j = 1; j < d; ++j) { /* prefix-OR along attribute j */
            uint64_t st = stride[j];
            for (uint64_t r = 0; r < rows; ++r) {
                uint64_t cj = (r / st) % ext[j];
                if (cj) P[r] |= P[r - st];
            }
        }
        for (uint64_t i = 0; i < s; ++i) {
            if (den[i]) continue;
            uint64_t r = 0;
            for (int j = 1; j < d; ++j) r += codes[i * d + j] * stride[j];
            uint32_t c0 = codes[i * d];
            int hit = 0;
            if (c0 > 0 && ((P[r] >> (c0 - 1)) & 1ULL)) hit = 1;
            for (int j = 1; j < d && !hit; ++j)
                if (codes[i * d + j] > 0 && ((P[r - stride[j]] >> c0) & 1ULL)) hit = 1;
            if (hit) den[i] = g;
        }
        free(P);
    }
    for (uint64_t i = 0; i < s; ++i)
        if (den[i] == 0) den[i] = 1;
    free(codes);
    return 0;
}

/* ------------------------------------------------------------ partition --- */
#define SO_MAX_PARTS (1LL << 20)
static long long ipow_cap(long long b, int e) { /* partition.cpp:15-22 */
    long long v = 1;
    for (int i = 0; i < e; ++i) {
        v *= b;
        if (v > SO_MAX_PARTS) return SO_MAX_PARTS + 1;
    }
    return v;
}
static int closest_slices(long long target, int e) { /* partition.cpp:24-31 */
    int m = 2;
    while (ipow_cap(m + 1, e) <= target) ++m;
    long long lo = ipow_cap(m, e), hi = ipow_cap(m + 1, e);
    return (target - lo <= hi - target) ? m : m + 1;
}
/* partition.cpp:53-83 make_plan; strategy 0 none,1 grid,2 angular,3 sliced.
 * returns 0 or -1 (invalid argument) */
int so_make_plan(int strategy, long long target, int dims, int* slices, long long* parts) {
    if (dims < 1) return -1;
    if (target < 1 || target > SO_MAX_PARTS) return -1;
    *slices = 1;
    *parts = 1;
    if (strategy == 1) {
        *slices = closest_slices(target, dims);
        *parts = ipow_cap(*slices, dims);
    } else if (strategy == 2) {
        if (dims < 2) return -1;
        *slices = closest_slices(target, dims - 1);
        *parts = ipow_cap(*slices, dims - 1);
    } else if (strategy == 3) {
        *parts = target;
    }
    if (*parts > SO_MAX_PARTS) return -1;
    return 0;
}

/* ------------------------------------------------- assign_partitions --- */
/* partition.cpp:183-213 with grid_cell + cell_partition_id (:85-109),
 * to_hyperspherical + assign_angular (:139-174) and assign_sliced
 * (:176-181; order by (attribute 0, id)).  Returns 0, or 1 + the first flat
 * index of a Grid value outside [0,1] (grid_cell's throw, :91-94). */
static const double* g_sl_v;
static const int64_t* g_sl_ids;
static int g_sl_d;
static int cmp_sliced(const void* a, const void* b) {
    const uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
    const double va = g_sl_v[x * g_sl_d], vb = g_sl_v[y * g_sl_d];
    if (va != vb) return va < vb ? -1 : 1;
    const int64_t ia = g_sl_ids ? g_sl_ids[x] : (int64_t)x, ib = g_sl_ids ? g_sl_ids[y] : (int64_t)y;
    return ia < ib ? -1 : (ia > ib ? 1 : 0);
}

long long so_assign_partitions(const double* v, const int64_t* ids, uint64_t n, int d,
                               int strategy, int slices, long long parts, int64_t* out) {
    const double kPi = 3.14159265358979323846; /* partition.cpp:13 */
    if (strategy == 0) {
        for (uint64_t i = 0; i < n; ++i) out[i] = 0;
        return 0;
    }
    if (strategy == 1) {
        for (uint64_t i = 0; i < n; ++i) {
            long long id = 0, w = 1;
            for (int j = 0; j < d; ++j) {
                const double x = v[i * d + j];
                if (x < 0.0 || x > 1.0) return 1 + (long long)(i * d + j);
                int idx = (int)(x * slices);
                if (idx >= slices) idx = slices - 1;
                id += (long long)idx * w;
                w *= slices;
            }
            out[i] = id;
        }
        return 0;
    }
    if (strategy == 2) {
        double tail[65];
        for (uint64_t i = 0; i < n; ++i) {
            const double* t = v + i * d;
            int all_zero = 1;
            for (int j = 0; j < d; ++j)
                if (t[j] != 0.0) { all_zero = 0; break; }
            if (all_zero) { out[i] = 0; continue; }
            tail[d] = 0.0;
            for (int j = d - 1; j >= 0; --j) tail[j] = tail[j + 1] + t[j] * t[j];
            long long id = 0, w = 1;
            for (int j = 0; j + 1 < d; ++j) {
                const double ang = atan2(sqrt(tail[j + 1]), t[j]);
                int idx = (int)((2.0 * ang / kPi) * slices);
                if (idx >= slices) idx = slices - 1;
                id += (long long)idx * w;
                w *= slices;
            }
            out[i] = id;
        }
        return 0;
    }
    /* sliced */
    uint64_t* order = (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t));
    if (!order) return -1;
    for (uint64_t i = 0; i < n; ++i) order[i] = i;
    g_sl_v = v;
    g_sl_ids = ids;
    g_sl_d = d;
    qsort(order, n, sizeof(uint64_t), cmp_sliced);
    for (uint64_t r = 0; r < n; ++r) out[order[r]] = (long long)r * parts / (long long)n;
    free(order);
    return 0;
}
