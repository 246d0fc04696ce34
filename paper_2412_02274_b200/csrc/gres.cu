// gres.cu — the grid-resistance stage on sm_100a (north_star (b)).
//
// Reference: grid_resistance (proj/src/gres.cpp:65-129).  g_max comes from the
// smallest non-zero same-attribute gap of the skyline (gres.cpp:15-37,
// :89-90); then for g = g_max .. 2 every tuple is projected to
// floor(v*g)/g (gres.cpp:41-55) and the projected skyline is recomputed
// (parallel_skyline, :102); a tuple's denominator is the first (largest) g
// whose projected skyline does not contain it, else 1 (:112-121).
//
// By the predecessor rule (skyline.cu) the projected skyline drops t at g
// iff some tuple s before t in (projected sum, id) order has q(s) dominating
// q(t), q = floor(v*g)/g.  Two exact reductions make this a pure code test:
//  * codes: with k = floor(v*g) (k < 2^52), correctly rounded k/g is
//    strictly increasing in k, so q(s) dominates q(t) iff k(s) dominates k(t);
//  * order: q(s) dominating q(t) forces psum(s) <= psum(t); a tie (which would
//    let a later-id dominator NOT eject t) needs sums that differ by >= 1/g to
//    round to the same double, impossible while g*d*(d+1)*(max|v|+1) < 2^50.
//    Outside that bound the float64 path re-checks (psum, id) order exactly.
// So at step g, t is ejected iff some skyline tuple's code vector dominates
// t's — every skyline tuple is a comparator; no order bookkeeping.
//
// Engines:
//  - pair engine, u8 codes (d <= 8, max code <= 127): a tuple's codes of
//    every step packed one byte per attribute (u32 words for d <= 4, u64 for
//    d <= 8); ONE launch covers all steps — the resident kernel (all steps'
//    codes of a comparator range staged once in shared memory, S <= 2^21) or
//    the tiled one; one test = SWAR subtract + mask + compare; a candidate
//    leaves at its first (largest) dominating step.
//  - cell engine (cells.cu), same codes, O(cells + S) per step: huge S;
//    its small-grid variant (d <= 4, code extent <= 32) runs every step in
//    ONE launch with each step's grid in shared memory and is preferred
//    whenever it applies (C1, C2).
//  - f64 path (anything else): one launch per step on the reference's own
//    projections floor(v*g)/g compared as float64, with the exact (psum, id)
//    order check when ties are possible.
#include <cub/cub.cuh>

#include <cmath>
#include <limits>

#include "sky_common.cuh"

namespace skygpu {

namespace {

constexpr int kBlock = 256;

template <class F>
void dispatch_d(int d, F&& f) {
    switch (d) {
        case 1: f(std::integral_constant<int, 1>{}); break;
        case 2: f(std::integral_constant<int, 2>{}); break;
        case 3: f(std::integral_constant<int, 3>{}); break;
        case 4: f(std::integral_constant<int, 4>{}); break;
        case 5: f(std::integral_constant<int, 5>{}); break;
        case 6: f(std::integral_constant<int, 6>{}); break;
        case 7: f(std::integral_constant<int, 7>{}); break;
        case 8: f(std::integral_constant<int, 8>{}); break;
        default: f(std::integral_constant<int, 0>{}); break;
    }
}

// column j of the SoA skyline into a contiguous buffer (for the gap sort)
__global__ void k_copy(const double* __restrict__ src, uint64_t n, double* __restrict__ dst) {
    pdl_wait();
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
}

// gres.cpp:20-24: min positive adjacent difference of a sorted column
__global__ void k_min_gap(const double* __restrict__ col, uint64_t n,
                          unsigned long long* __restrict__ slots) {
    pdl_wait();
    unsigned long long best = 0x7FF0000000000000ULL;  // +inf
    for (uint64_t i = 1 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        double gap = __dsub_rn(col[i], col[i - 1]);
        if (gap > 0.0) {
            unsigned long long b = (unsigned long long)__double_as_longlong(gap);
            best = b < best ? b : best;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        unsigned long long x = __shfl_down_sync(0xffffffffu, best, o);
        best = x < best ? x : best;
    }
    if ((threadIdx.x & 31) == 0) atomicMin(&slots[S_MINGAP], best);
}

__global__ void k_max_value(const double* __restrict__ v, uint64_t n,
                            unsigned long long* __restrict__ slots) {
    pdl_wait();
    unsigned long long best = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        unsigned long long b = ord_bits(v[i]);
        best = b > best ? b : best;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        unsigned long long x = __shfl_down_sync(0xffffffffu, best, o);
        best = x > best ? x : best;
    }
    if ((threadIdx.x & 31) == 0) atomicMax(&slots[S_MAXV], best);
}

// gres.cpp:70-80 (checked builds): the first (a, b) in input order with
// a dominating b.  Per candidate b the smallest dominating a; global min of
// a*S + b gives the lexicographically first pair.
template <int D>
__global__ void __launch_bounds__(kBlock)
k_check_skyline(const double* __restrict__ v, uint64_t S, int d,
                unsigned long long* __restrict__ slots) {
    pdl_wait();
    constexpr int TILE = D > 0 ? 256 : 128;
    constexpr int DM = D > 0 ? D : kMaxDims;
    extern __shared__ double tile[];
    const int dd = D > 0 ? D : d;
    const uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const bool valid = b < S;
    double t[DM];
#pragma unroll
    for (int k = 0; k < DM; ++k)
        if (k < dd) t[k] = valid ? v[k * S + b] : 0.0;
    bool alive = valid;
    for (uint64_t base = 0; base < S; base += TILE) {
        const uint32_t nt = (uint32_t)min((uint64_t)TILE, S - base);
        for (uint32_t k = threadIdx.x; k < nt; k += blockDim.x)
            for (int a = 0; a < dd; ++a) tile[a * TILE + k] = v[a * S + base + k];
        __syncthreads();
        if (alive) {
            for (uint32_t k = 0; k < nt; ++k) {
                double s[DM];
#pragma unroll
                for (int a = 0; a < DM; ++a)
                    if (a < dd) s[a] = tile[a * TILE + k];
                bool dm = D > 0 ? dom_f64<(D > 0 ? D : 1)>(s, t) : dom_f64_dyn(s, t, dd);
                if (dm) {
                    atomicMin(&slots[S_PAIR], (unsigned long long)((base + k) * S + b));
                    alive = false;
                    break;
                }
            }
        }
        if (!__syncthreads_or(alive)) break;
    }
}

// projections at step g exactly as the reference: floor(v*g)/g (gres.cpp:46)
__global__ void k_project(const double* __restrict__ v, uint64_t total, int g,
                          double* __restrict__ q) {
    pdl_wait();
    const double gd = (double)g;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
         i += (uint64_t)gridDim.x * blockDim.x)
        q[i] = __ddiv_rn(floor(__dmul_rn(v[i], gd)), gd);
}

// candidate list of this shard, ascending: the k-th owned tuple of the
// interleaved 256-tuple chunks rank, rank + world, rank + 2*world, ...
__global__ void k_shard_iota(uint64_t na, int rank, int world, uint32_t* __restrict__ act) {
    pdl_wait();
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < na;
         k += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t chunk = (uint64_t)rank + (uint64_t)world * (k >> 8);
        act[k] = (uint32_t)(chunk * 256 + (k & 255));
    }
}

// the speculative path's set-up in one launch: flags, the witness table,
// den = 0 and the identity candidate list
__global__ void k_gres_spec_init(unsigned long long* __restrict__ slots,
                                 unsigned long long* __restrict__ table, uint64_t ntab,
                                 int32_t* __restrict__ den, uint64_t S, uint32_t* __restrict__ act) {
    pdl_wait();
    const uint64_t i0 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i0 == 0) {
        slots[S_FLAG] = 0;
        slots[S_MAXV] = 0;
        slots[S_SPEC] = 0;
    }
    for (uint64_t i = i0; i < S || i < ntab; i += (uint64_t)gridDim.x * blockDim.x) {
        if (i < ntab) table[i] = 0;
        if (i < S) {
            den[i] = 0;
            act[i] = (uint32_t)i;
        }
    }
}

__global__ void k_fill_den(const uint32_t* __restrict__ act, uint64_t na, int value,
                           int32_t* __restrict__ den) {
    pdl_wait();
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < na;
         i += (uint64_t)gridDim.x * blockDim.x)
        den[act[i]] = value;
}

// ---- pair engine, u8 path, all steps in ONE launch ----------------------
// codes of every step: codes[gi*S + t] for g = g_max - gi (gi = 0 .. G-1),
// one byte per attribute (u32 words for d <= 4, u64 for d <= 8)
// Tiled pair kernel (all steps, one launch).  Block = 8 warps x 8
// candidates each, over one comparator range.  For each step g (descending)
// the range's codes at g are staged through shared memory in 2048-code tiles;
// every lane loads one comparator code and tests it against all of its
// warp's still-undecided candidates (register blocking: 1 LDS per 8 tests),
// and one redux.or per 32 comparators tells the warp which candidates were
// hit (warp-level early exit).  A hit at g is the candidate's final answer
// (atomicMax(den, g)); candidates re-read den every step, so exits found by
// blocks working on other comparator ranges prune this block too.
constexpr int kTileCodes = 2048;
constexpr int kCandPerWarp = 8;
constexpr int kCandPerBlock = (kBlock / 32) * kCandPerWarp;

template <class W>
__device__ __forceinline__ bool dom_w(W s, W t, W tg) {
    constexpr W H = (W)kGuard;
    return (((tg - s) & H) == H) & (s != t);
}

template <class W>
__global__ void k_codes_all(const double* __restrict__ v, uint64_t S, int d, int g_max, int G,
                            W* __restrict__ codes) {
    pdl_wait();
    const uint64_t total = S * (uint64_t)G;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t gi = i / S, t = i - gi * S;
        const double gd = (double)(g_max - (int)gi);
        W w = 0;
        for (int k = 0; k < d; ++k) {
            double q = floor(__dmul_rn(v[k * S + t], gd));
            w |= (W)(unsigned)q << (8 * k);
        }
        codes[i] = w;
    }
}

template <class W>
__global__ void __launch_bounds__(kBlock)
k_gres_pairs_tiled(const W* __restrict__ codes, uint32_t S, int G, int g_max,
                   const uint32_t* __restrict__ act, uint32_t na, uint32_t range,
                   int32_t* __restrict__ den, unsigned long long* __restrict__ tests) {
    pdl_wait();
    constexpr W H = (W)kGuard;
    __shared__ W tile[kTileCodes];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t r0 = blockIdx.y * range;
    const uint32_t r1 = min(S, r0 + range);
    volatile int32_t* vden = den;
    uint32_t t[kCandPerWarp];
    int best[kCandPerWarp];
    unsigned valid = 0;
#pragma unroll
    for (int c = 0; c < kCandPerWarp; ++c) {
        const uint32_t idx = blockIdx.x * kCandPerBlock + warp * kCandPerWarp + c;
        t[c] = idx < na ? act[idx] : 0;
        best[c] = idx < na ? 0 : 0x7fffffff;
        if (idx < na) valid |= 1u << c;
    }
    unsigned long long cnt = 0;
    for (int gi = 0; gi < G; ++gi) {
        const int g = g_max - gi;
        unsigned alive = 0;
#pragma unroll
        for (int c = 0; c < kCandPerWarp; ++c) {
            if (((valid >> c) & 1) && best[c] < g) best[c] = max(best[c], vden[t[c]]);
            if (best[c] < g) alive |= 1u << c;
        }
        // (den moves under other blocks' atomicMax; the loads above are ONE
        // instruction of a converged warp — every branch before them is on
        // warp-uniform values and the scan ends in a warp vote — so all lanes
        // read the same value and leave the scan loops together.  A lane-0
        // broadcast of alive was measured: resident kernel 1.39 -> 1.75 ms,
        // the mask no longer lives in predicates.)
        if (!__syncthreads_or(alive != 0)) break;
        const W* cg = codes + (uint64_t)gi * S;
        W tc[kCandPerWarp], tg[kCandPerWarp];
#pragma unroll
        for (int c = 0; c < kCandPerWarp; ++c) {
            tc[c] = ((alive >> c) & 1) ? cg[t[c]] : (W)0;
            tg[c] = tc[c] | H;
        }
        for (uint32_t base = r0; base < r1; base += kTileCodes) {
            const uint32_t nt = min((uint32_t)kTileCodes, r1 - base);
            for (uint32_t k = threadIdx.x; k < nt; k += kBlock) tile[k] = cg[base + k];
            __syncthreads();
            for (uint32_t k0 = 0; k0 < nt && alive; k0 += 32) {
                const uint32_t k = k0 + lane;
                unsigned hits = 0;
                if (k < nt) {
                    const W s = tile[k];
#pragma unroll
                    for (int c = 0; c < kCandPerWarp; ++c)
                        if ((alive >> c) & 1) hits |= (unsigned)dom_w<W>(s, tc[c], tg[c]) << c;
                    cnt += __popc(alive);
                }
                hits = __reduce_or_sync(0xffffffffu, hits);
                if (hits) {
                    alive &= ~hits;
#pragma unroll
                    for (int c = 0; c < kCandPerWarp; ++c)
                        if ((hits >> c) & 1) {
                            best[c] = g;
                            if (lane == 0) atomicMax(&den[t[c]], g);
                        }
                }
            }
            if (!__syncthreads_or(alive != 0)) break;
        }
    }
    add_count(tests, cnt);
}

// Resident pair kernel (default for S <= 2^21).  A block = 64 candidates
// (8 warps x 8) x one comparator range of <= 512 tuples.  The block stages
// ONCE the codes of every step for its range (<= 48 KB of shared memory) and
// for its candidates; after that single barrier the 8 warps run through the
// steps independently — no further barrier, no global load on the critical
// path: for each g (descending) every lane tests one comparator against the
// warp's still-undecided candidates (register-blocked, one LDS per 8 tests),
// one redux.or per 32 comparators retires the hit candidates (answer g,
// atomicMax(den, g)).  Exits found by blocks on other ranges arrive through
// den, read one step ahead so the latency overlaps the scan.
constexpr int kResCand = kCandPerWarp * (kBlock / 32);  // 64

template <class W>
__global__ void __launch_bounds__(kBlock)
k_gres_pairs_resident(const W* __restrict__ codes, uint32_t S, int G, int g_max,
                      const uint32_t* __restrict__ act, uint32_t na, uint32_t range,
                      int32_t* __restrict__ den, unsigned long long* __restrict__ tests) {
    pdl_wait();
    constexpr W H = (W)kGuard;
    extern __shared__ __align__(16) unsigned char smraw[];
    const uint32_t r0 = blockIdx.y * range;
    const uint32_t rl = min(range, S - r0);
    W* comp = reinterpret_cast<W*>(smraw);      // [G][rl]
    W* cand = comp + (size_t)G * rl;             // [G][64]
    for (uint32_t i = threadIdx.x; i < (uint32_t)G * rl; i += kBlock) {
        const uint32_t gi = i / rl, k = i - gi * rl;
        comp[i] = codes[(uint64_t)gi * S + r0 + k];
    }
    for (uint32_t i = threadIdx.x; i < (uint32_t)G * kResCand; i += kBlock) {
        const uint32_t gi = i / kResCand, l = i - gi * kResCand;
        const uint32_t idx = blockIdx.x * kResCand + l;
        cand[i] = idx < na ? codes[(uint64_t)gi * S + act[idx]] : (W)0;
    }
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    volatile int32_t* vden = den;
    uint32_t t[kCandPerWarp];
    int best[kCandPerWarp];
#pragma unroll
    for (int c = 0; c < kCandPerWarp; ++c) {
        const uint32_t idx = blockIdx.x * kResCand + warp * kCandPerWarp + c;
        t[c] = idx < na ? act[idx] : 0;
        best[c] = idx < na ? vden[t[c]] : 0x7fffffff;
    }
    unsigned long long cnt = 0;
    for (int gi = 0; gi < G; ++gi) {
        const int g = g_max - gi;
        unsigned alive = 0;
#pragma unroll
        for (int c = 0; c < kCandPerWarp; ++c)
            if (best[c] < g) alive |= 1u << c;
        // (same argument as in the tiled kernel: one load instruction of a
        // converged warp per candidate, warp-uniform control flow around it)
        if (!alive) break;
        W tc[kCandPerWarp], tg[kCandPerWarp];
        int nb[kCandPerWarp];
#pragma unroll
        for (int c = 0; c < kCandPerWarp; ++c) {
            tc[c] = cand[gi * kResCand + warp * kCandPerWarp + c];
            tg[c] = tc[c] | H;
            nb[c] = ((alive >> c) & 1) ? vden[t[c]] : best[c];  // consumed after the scan
        }
        const W* cg = comp + (size_t)gi * rl;
        // branch-free inner loop: every lane tests its comparator against all
        // 8 candidates (x = tg - s: every guard bit set <=> s <= t bytewise;
        // x > H <=> additionally s != t), one ballot per candidate, and the
        // already-decided candidates are masked out afterwards.  Lanes past
        // the range use the neutral code 0x7F..7F, which dominates nothing.
        constexpr W kNeutral = (W)0x7F7F7F7F7F7F7F7FULL;
        for (uint32_t k0 = 0; k0 < rl && alive; k0 += 32) {
            const uint32_t k = k0 + lane;
            const W s = k < rl ? cg[k] : kNeutral;
            unsigned hits = 0;
#pragma unroll
            for (int c = 0; c < kCandPerWarp; ++c) {
                const W x = tg[c] - s;
                const bool le = (x & H) == H;  // s <= t in every byte
                unsigned bl;
                if constexpr (sizeof(W) == 8) {
                    // u64 words: the 64-bit strictness compare only when some
                    // lane passed (warp-uniform branch) — fewer ALU ops per test
                    bl = __ballot_sync(0xffffffffu, le);
                    if (bl) bl = __ballot_sync(0xffffffffu, le & (x != H));
                } else {
                    bl = __ballot_sync(0xffffffffu, le & (x != H));
                }
                hits |= (bl != 0u ? 1u : 0u) << c;
            }
            hits &= alive;
            if (k < rl) cnt += __popc(alive);
            if (hits) {
                alive &= ~hits;
#pragma unroll
                for (int c = 0; c < kCandPerWarp; ++c)
                    if ((hits >> c) & 1) {
                        best[c] = g;
                        if (lane == 0) atomicMax(&den[t[c]], g);
                    }
            }
        }
#pragma unroll
        for (int c = 0; c < kCandPerWarp; ++c) best[c] = max(best[c], nb[c]);
    }
    add_count(tests, cnt);
}

__global__ void k_finalize_den(const uint32_t* __restrict__ act, uint64_t na,
                               int32_t* __restrict__ den) {
    pdl_wait();
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < na;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t t = act[i];
        if (den[t] == 0) den[t] = 1;
    }
}

// ---- pair engine, float64 path ------------------------------------------
// psum (core.cpp:21-23 on the projection) and the (psum, id) predecessor
// order, only consulted when ties are possible.
__device__ __forceinline__ bool before(const double* __restrict__ q, uint64_t S, int d,
                                       const int64_t* __restrict__ ids, uint32_t s, uint32_t t) {
    double ps = 0.0, pt = 0.0;
    for (int k = 0; k < d; ++k) {
        ps = __dadd_rn(ps, q[k * S + s]);
        pt = __dadd_rn(pt, q[k * S + t]);
    }
    if (ps != pt) return ps < pt;
    if (ids[s] != ids[t]) return ids[s] < ids[t];
    return s < t;
}

template <int D>
__global__ void __launch_bounds__(kBlock)
k_gres_pairs_f64(const double* __restrict__ q, uint32_t S, int d,
                 const int64_t* __restrict__ ids, const uint32_t* __restrict__ act,
                 uint32_t na, int g, int tiecheck, int32_t* __restrict__ den,
                 uint8_t* __restrict__ still, unsigned long long* __restrict__ tests) {
    pdl_wait();
    constexpr int TILE = D > 0 ? 256 : 128;
    constexpr int DM = D > 0 ? D : kMaxDims;
    extern __shared__ double tile[];
    const int dd = D > 0 ? D : d;
    const uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x;
    const bool valid = idx < na;
    const uint32_t ti = valid ? act[idx] : 0;
    double t[DM];
#pragma unroll
    for (int k = 0; k < DM; ++k)
        if (k < dd) t[k] = valid ? q[(uint64_t)k * S + ti] : 0.0;
    bool alive = valid;
    unsigned long long cnt = 0;
    for (uint32_t base = 0; base < S; base += TILE) {
        const uint32_t nt = min((uint32_t)TILE, S - base);
        for (uint32_t k = threadIdx.x; k < nt; k += blockDim.x)
            for (int a = 0; a < dd; ++a) tile[a * TILE + k] = q[(uint64_t)a * S + base + k];
        __syncthreads();
        if (alive) {
            for (uint32_t k = 0; k < nt; ++k) {
                double s[DM];
#pragma unroll
                for (int a = 0; a < DM; ++a)
                    if (a < dd) s[a] = tile[a * TILE + k];
                ++cnt;
                bool dm = D > 0 ? dom_f64<(D > 0 ? D : 1)>(s, t) : dom_f64_dyn(s, t, dd);
                if (dm && tiecheck) dm = before(q, S, dd, ids, base + k, ti);
                if (dm) {
                    alive = false;
                    break;
                }
            }
        }
        if (!__syncthreads_or(alive)) break;
    }
    if (valid) {
        still[idx] = alive;
        if (!alive) den[ti] = g;
    }
    add_count(tests, cnt);
}

uint64_t select_flagged(Ctx& c, const uint32_t* in, const uint8_t* flags, uint32_t* out,
                        uint64_t n) {
    if (n == 0) return 0;
    size_t tmp = 0;
    SKY_CUDA(cub::DeviceSelect::Flagged(nullptr, tmp, in, flags, out, c.d_slots + S_SEL,
                                         (int64_t)n, c.stream));
    void* t = c.buf[B_CUB].get(tmp);
    SKY_CUDA(cub::DeviceSelect::Flagged(t, tmp, in, flags, out, c.d_slots + S_SEL, (int64_t)n,
                                         c.stream));
    note_launch(c, 2);
    read_slots(c, S_SEL, 1);
    return c.h_slots[S_SEL];
}

}  // namespace

// gres.cpp:30-37 intervals_from_gap, same float64 arithmetic
static int intervals_from_gap(double gap, int cap) {
    if (cap > 0 && 1.0 / gap >= static_cast<double>(cap)) return cap;
    double bound = std::floor(1.0 / gap);
    if (bound > static_cast<double>(std::numeric_limits<int>::max()))
        invalid("max_grid_intervals: bound overflows the integer range; set a cap");
    return static_cast<int>(bound);
}

// Witness for the capped branch of intervals_from_gap (gres.cpp:31): two
// DISTINCT values of one attribute in the same bucket of width 1/(2 cap)
// have an FP gap with 1.0/gap >= cap, and the reference's min adjacent gap
// is <= that gap (rounding is monotone), so g_max = cap exactly.  Values
// outside [0,1) are simply not bucketed (the witness is then inconclusive
// only if no other pair qualifies).  Also reduces max value (code range).
__global__ void k_gap_witness(const double* __restrict__ v, uint64_t S, int d, int cap,
                              unsigned long long* __restrict__ table,
                              unsigned long long* __restrict__ slots) {
    pdl_wait();
    const int nb = 2 * cap;
    unsigned long long mx = 0;
    bool found = false;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < S * d;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t j = i / S;
        const double x = v[i];
        const unsigned long long bits = ord_bits(x);
        mx = bits > mx ? bits : mx;
        if (!(x >= 0.0 && x < 1.0) || found) continue;
        int b = (int)floor(__dmul_rn(x, (double)nb));
        b = b < 0 ? 0 : (b >= nb ? nb - 1 : b);
        // a plain read first: the 2*cap buckets per attribute fill at once,
        // after that a CAS per value would serialise on a few addresses
        unsigned long long old = *(volatile unsigned long long*)&table[j * nb + b];
        if (old == 0ULL) old = atomicCAS(&table[j * nb + b], 0ULL, bits + 1);
        if (old != 0ULL && old != bits + 1) {
            const unsigned long long ob = old - 1;
            const double w = __longlong_as_double((long long)ob);
            const double gap = x > w ? __dsub_rn(x, w) : __dsub_rn(w, x);
            if (gap > 0.0 && __ddiv_rn(1.0, gap) >= (double)cap) found = true;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        unsigned long long x = __shfl_down_sync(0xffffffffu, mx, o);
        mx = x > mx ? x : mx;
    }
    if ((threadIdx.x & 31) == 0) atomicMax(&slots[S_MAXV], mx);
    if (found) atomicOr(&slots[S_FLAG], 1ULL);
}

// The same witness with the buckets in shared memory, one attribute per
// blockIdx.y (cap <= kWitnessSmemCap): each block looks for a pair in its own
// share of the column — no global CAS contention (the global-table form
// serialises millions of CAS on d x 2cap addresses at C5).  Any pair proves
// the cap, so block-local detection is exact; S <= 4096 runs one block per
// attribute (the whole column, like the global table); a block per 1024
// values otherwise (any pigeonhole pair of distinct values proves the cap).
constexpr int kWitnessSmemCap = 2048;

__global__ void __launch_bounds__(256)
    k_gap_witness_smem(const double* __restrict__ v, uint64_t S, int cap,
                       unsigned long long* __restrict__ slots) {
    pdl_wait();
    __shared__ unsigned long long tab[2 * kWitnessSmemCap];
    __shared__ int any;
    const int nb = 2 * cap;
    for (int b = threadIdx.x; b < nb; b += blockDim.x) tab[b] = 0;
    if (threadIdx.x == 0) any = 0;
    __syncthreads();
    const double* col = v + (uint64_t)blockIdx.y * S;
    unsigned long long mx = 0;
    bool found = false;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < S;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const double x = col[i];
        const unsigned long long bits = ord_bits(x);
        mx = bits > mx ? bits : mx;
        if (!(x >= 0.0 && x < 1.0) || found) continue;
        int b = (int)floor(__dmul_rn(x, (double)nb));
        b = b < 0 ? 0 : (b >= nb ? nb - 1 : b);
        unsigned long long old = tab[b];
        if (old == 0ULL) old = atomicCAS(&tab[b], 0ULL, bits + 1);
        if (old != 0ULL && old != bits + 1) {
            const double w = __longlong_as_double((long long)(old - 1));
            const double gap = x > w ? __dsub_rn(x, w) : __dsub_rn(w, x);
            if (gap > 0.0 && __ddiv_rn(1.0, gap) >= (double)cap) found = true;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        unsigned long long x = __shfl_down_sync(0xffffffffu, mx, o);
        mx = x > mx ? x : mx;
    }
    if ((threadIdx.x & 31) == 0) atomicMax(&slots[S_MAXV], mx);
    if (found) any = 1;
    __syncthreads();
    if (threadIdx.x == 0 && any) atomicOr(&slots[S_FLAG], 1ULL);
}

// one launch of the witness (shared-memory buckets when cap allows)
void launch_gap_witness(Ctx& c, const double* d_soa, uint64_t S, int d, int cap,
                        unsigned long long* table) {
    if (cap <= kWitnessSmemCap) {
        const uint64_t want = S <= 4096 ? 1 : (S + 1023) / 1024;
        const unsigned bx = (unsigned)std::max<uint64_t>(
            1, std::min<uint64_t>(want, (uint64_t)c.num_sms * 8 / (uint64_t)d + 1));
        pdl_launch(k_gap_witness_smem, dim3(bx, (unsigned)d), 256, 0, c.stream, d_soa, S, cap,
                   c.d_slots);
    } else {
        SKY_CUDA(cudaMemsetAsync(table, 0, sizeof(unsigned long long) * d * 2 * cap, c.stream));
        pdl_launch(k_gap_witness, grid_for(S * d, kBlock), kBlock, 0, c.stream, d_soa, S, d, cap,
                   table,
                                                                         c.d_slots);
    }
    SKY_LAUNCH_CHECK();
    note_launch(c);
}

// gres.cpp:15-28 on the device: per column sort + adjacent-difference min.
// Returns false when every attribute is constant.
bool min_positive_gap_device(Ctx& c, const double* d_soa, uint64_t S, int d, double* gap,
                             double* maxv) {
    zero_slots(c);
    double* col = c.buf[B_GTMP0].as<double>(S);
    double* srt = c.buf[B_GTMP1].as<double>(S);
    const unsigned gb = grid_for(S, kBlock);
    for (int j = 0; j < d; ++j) {
        pdl_launch(k_copy, gb, kBlock, 0, c.stream, d_soa + (uint64_t)j * S, S, col);
        SKY_LAUNCH_CHECK();
        size_t tmp = 0;
        SKY_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp, col, srt, (int64_t)S, 0, 64,
                                                 c.stream));
        void* t = c.buf[B_CUB].get(tmp);
        SKY_CUDA(cub::DeviceRadixSort::SortKeys(t, tmp, col, srt, (int64_t)S, 0, 64, c.stream));
        pdl_launch(k_min_gap, gb, kBlock, 0, c.stream, srt, S, c.d_slots);
        SKY_LAUNCH_CHECK();
        note_launch(c, 6);
    }
    pdl_launch(k_max_value, grid_for(S * d, kBlock), kBlock, 0, c.stream, d_soa, S * d, c.d_slots);
    SKY_LAUNCH_CHECK();
    note_launch(c);
    read_slots(c, S_MINGAP, 2);
    unsigned long long gb_bits = c.h_slots[S_MINGAP], mb = c.h_slots[S_MAXV];
    double g, m;
    memcpy(&g, &gb_bits, 8);
    memcpy(&m, &mb, 8);
    *maxv = m;
    if (!std::isfinite(g)) return false;
    *gap = g;
    return true;
}

// g_max of gres.cpp:89-90: the cap witness when it fires, else the exact
// per-column sort.  Also returns the max value (code range).
int g_max_device(Ctx& c, const double* d_soa, uint64_t S, int d, int cap, double* maxv) {
    if (cap > 0 && cap <= 65536 && S >= 2) {
        zero_slots(c);
        unsigned long long* table = c.buf[B_CELLS].as<unsigned long long>((uint64_t)d * 2 * cap);
        launch_gap_witness(c, d_soa, S, d, cap, table);
        read_slots(c, S_MAXV, 3);  // S_MAXV, S_BAD, S_FLAG
        if (c.h_slots[S_FLAG] & 1ULL) {
            unsigned long long mb = c.h_slots[S_MAXV];
            memcpy(maxv, &mb, 8);
            return cap;
        }
    }
    double gap = 0;
    if (!min_positive_gap_device(c, d_soa, S, d, &gap, maxv)) return 1;
    return intervals_from_gap(gap, cap);
}

void gres_spec_fetch(Ctx& c) {
    if (c.gres_spec)
        SKY_CUDA(cudaMemcpyAsync(c.h_slots + S_SPEC, c.d_slots + S_SPEC, sizeof(unsigned long long),
                                 cudaMemcpyDeviceToHost, c.stream));
}

bool gres_spec_failed(Ctx& c) {
    if (!c.gres_spec) return false;
    c.gres_spec = false;
    return c.h_slots[S_SPEC] != 0;
}

GresOut gres_device(Ctx& c, const double* d_skyv, const int64_t* d_ids, uint64_t S, int d,
                    int cap, int engine, int shard_rank, int shard_world, bool check_skyline,
                    int32_t* d_den, bool allow_spec) {
    GresOut out;
    skygpu_stats& st = *c.st;
    if (S >= 0x7FFFFFFFull) invalid("grid_resistance: more than 2^31-1 skyline tuples");
    if (S == 0) return out;
    if (shard_world < 1) shard_world = 1;

    // speculative capped scan without a host round trip: the gap witness,
    // then the shared-memory cell kernel reading g_max (= cap when the
    // witness fired) and the value maximum from the device; if either does
    // not hold the kernel raises S_SPEC and the caller re-runs this call
    // with allow_spec = false after its final synchronisation
    c.gres_spec = false;
    if (allow_spec && !check_skyline && shard_world == 1 && engine != SKYGPU_GRES_PAIRS &&
        cap >= 2 && cap <= 31 && S >= 2 && d >= 1 && d <= 4) {
        const uint64_t ntab = (uint64_t)d * 2 * cap;
        unsigned long long* table = c.buf[B_CELLS].as<unsigned long long>(ntab);
        uint32_t* act = c.buf[B_ACT0].as<uint32_t>(S);
        trace_mark(c, "gres: start (speculative)");
        pdl_launch(k_gres_spec_init, grid_for(S > ntab ? S : ntab, kBlock), kBlock, 0, c.stream,
            c.d_slots, table, ntab, d_den, S, act);
        SKY_LAUNCH_CHECK();
        note_launch(c);
        launch_gap_witness(c, d_skyv, S, d, cap, table);
        cudaEvent_t e0 = c.ev[10], e1 = c.ev[11];
        SKY_CUDA(cudaEventRecord(e0, c.stream));
        if (gres_cells_smem_spec(c, d_skyv, S, d, cap, act, S, d_den)) {
            SKY_CUDA(cudaEventRecord(e1, c.stream));
            trace_mark(c, "gres: shared-memory cell kernel");
            pdl_launch(k_finalize_den, grid_for(S, kBlock), kBlock, 0, c.stream, act, S, d_den);
            SKY_LAUNCH_CHECK();
            note_launch(c);
            c.gres_timing_pending = true;
            c.gres_spec = true;
            out.g_max = cap;
            out.steps = cap - 1;
            st.g_max = cap;
            st.code_bits = 8;
            st.gres_engine = SKYGPU_GRES_CELLS;
            st.gres_cells = 0;
            st.gres_steps = cap - 1;
            st.gres_kernel_launches += 1;
            return out;
        }
    }

    if (check_skyline) {
        zero_slots(c);
        dispatch_d(d, [&](auto DC) {
            constexpr int D = decltype(DC)::value;
            const size_t smem = sizeof(double) * (D > 0 ? 256 : 128) * (D > 0 ? D : d);
            pdl_launch(k_check_skyline<D>, grid_for(S, kBlock, 1 << 30), kBlock, smem, c.stream,
                d_skyv, S, d, c.d_slots);
        });
        SKY_LAUNCH_CHECK();
        note_launch(c);
        read_slots(c, S_PAIR, 1);
        if (c.h_slots[S_PAIR] != ~0ULL) {
            const uint64_t key = c.h_slots[S_PAIR];
            int64_t ia = 0, ib = 0;
            SKY_CUDA(cudaMemcpyAsync(&ia, d_ids + key / S, 8, cudaMemcpyDeviceToHost, c.stream));
            SKY_CUDA(cudaMemcpyAsync(&ib, d_ids + key % S, 8, cudaMemcpyDeviceToHost, c.stream));
            SKY_CUDA(cudaStreamSynchronize(c.stream));
            invalid("grid_resistance: input is not a skyline (tuple " + std::to_string(ia) +
                    " dominates tuple " + std::to_string(ib) + ")");
        }
    }

    double maxv = 0;
    trace_mark(c, "gres: start");
    out.g_max = g_max_device(c, d_skyv, S, d, cap, &maxv);
    trace_mark(c, "gres: g_max (witness/sort + sync)");
    st.g_max = out.g_max;

    // candidate list of this shard
    uint32_t* act = c.buf[B_ACT0].as<uint32_t>(S);
    uint32_t* act2 = c.buf[B_ACT1].as<uint32_t>(S);
    uint8_t* still = c.buf[B_FLAGS].as<uint8_t>(S);
    const unsigned gb = grid_for(S, kBlock);
    SKY_CUDA(cudaMemsetAsync(d_den, 0, S * sizeof(int32_t), c.stream));
    uint64_t na = 0;  // owned tuples: interleaved 256-tuple chunks (load balance)
    for (uint64_t ch = shard_rank; ch * 256 < S; ch += shard_world)
        na += std::min<uint64_t>(256, S - ch * 256);
    pdl_launch(k_shard_iota, grid_for(na ? na : 1, kBlock), kBlock, 0, c.stream, na, shard_rank,
                                                                           shard_world, act);
    SKY_LAUNCH_CHECK();
    note_launch(c);

    // path selection (see file header)
    const double code_max = std::floor(maxv * (double)out.g_max);
    const double tie_bound = (double)out.g_max * d * (d + 1) * (maxv + 1.0);
    const bool ties_possible = !(tie_bound < 1125899906842624.0);  // 2^50
    const bool u8 = d <= 8 && code_max <= 127.0 && !ties_possible;
    st.code_bits = u8 ? 8 : 64;
    st.gres_engine = SKYGPU_GRES_PAIRS;

    cudaEvent_t e0 = c.ev[10], e1 = c.ev[11];
    double kms = 0;
    uint64_t klaunch = 0;
    int steps = 0;
    const int G = out.g_max - 1;
    // cell-occupancy engine (cells.cu): asked for, or AUTO on huge skylines
    // where the pair engine's O(S^2) tests dominate
    const bool want_cells = u8 && G >= 1 && (na > 0 || shard_world > 1) &&
                            (engine == SKYGPU_GRES_CELLS ||
                             (engine == SKYGPU_GRES_AUTO && S >= (1u << 18)));
    // small grids (d <= 4): every step in one launch, grids in shared memory
    // — the cheapest engine whenever it applies
    if (u8 && G >= 1 && na > 0 && engine != SKYGPU_GRES_PAIRS) {
        SKY_CUDA(cudaEventRecord(e0, c.stream));
        if (gres_cells_smem_device(c, d_skyv, S, d, out.g_max, maxv, act, na, d_den)) {
            SKY_CUDA(cudaEventRecord(e1, c.stream));
            trace_mark(c, "gres: shared-memory cell kernel");
            pdl_launch(k_finalize_den, grid_for(na, kBlock), kBlock, 0, c.stream, act, na, d_den);
            SKY_LAUNCH_CHECK();
            note_launch(c);
            c.gres_timing_pending = true;
            st.gres_engine = SKYGPU_GRES_CELLS;
            st.gres_cells = 0;  // no HBM sweeps (bench.py reads 0 as this variant)
            out.steps = G;
            st.gres_steps = G;
            st.gres_kernel_launches += 1;
            return out;
        }
    }
    if (want_cells) {
        uint64_t swept = 0;
        int steps_run = 0;
        // sharded: the cell engine splits the STEPS over the shards (every
        // candidate on every rank; a rank's den = its largest dominated step,
        // 1 if none — the MAX over ranks is the reference's map), instead of
        // the tuples: the grid build of a step is the cost, not its queries
        uint32_t* cact = act;
        uint64_t cna = na;
        if (shard_world > 1) {
            cact = c.buf[B_ACT1].as<uint32_t>(S);
            cna = S;
            pdl_launch(k_shard_iota, grid_for(S, kBlock), kBlock, 0, c.stream, S, 0, 1, cact);
            SKY_LAUNCH_CHECK();
            note_launch(c);
        }
        SKY_CUDA(cudaEventRecord(e0, c.stream));
        if (gres_cells_device(c, d_skyv, S, d, out.g_max, cact, cna, d_den, &swept, &steps_run,
                              shard_rank, shard_world)) {
            SKY_CUDA(cudaEventRecord(e1, c.stream));
            pdl_launch(k_finalize_den, grid_for(cna, kBlock), kBlock, 0, c.stream, cact, cna,
                       d_den);
            SKY_LAUNCH_CHECK();
            note_launch(c);
            c.gres_timing_pending = true;
            st.gres_engine = SKYGPU_GRES_CELLS;
            st.gres_cells = swept;
            out.steps = G;
            st.gres_steps = G;
            st.gres_kernel_launches += steps_run;
            return out;
        }
    }
    if (u8 && G >= 1 && na > 0) {
        // one launch for every step (north_star (b)): (candidate tile x
        // comparator range) blocks, per-step dominance with early exit
        const bool w32 = d <= 4;
        void* codes = c.buf[B_CODES].get(S * (uint64_t)G * (w32 ? 4 : 8));
        const unsigned cgrid = grid_for(S * (uint64_t)G, kBlock);
        if (w32)
            pdl_launch(k_codes_all<uint32_t>, cgrid, kBlock, 0, c.stream, d_skyv, S, d, out.g_max,
                       G,
                                                                  (uint32_t*)codes);
        else
            pdl_launch(k_codes_all<unsigned long long>, cgrid, kBlock, 0, c.stream,
                d_skyv, S, d, out.g_max, G, (unsigned long long*)codes);
        SKY_LAUNCH_CHECK();
        const bool resident = S <= (1u << 21) && !getenv("SKYGPU_GRES_TILED");
        trace_mark(c, "gres: shard list + codes");
        if (resident) {
            const size_t wb = w32 ? 4 : 8;
            const uint64_t tiles = (na + kResCand - 1) / kResCand;
            // comparator range: <= 48 KB of codes per block, and enough blocks
            // for ~8 per SM
            uint64_t range = (48 * 1024) / ((uint64_t)G * wb);
            range = std::max<uint64_t>(32, std::min<uint64_t>(range, 512));
            const uint64_t want_ranges = ((uint64_t)c.num_sms * 8 + tiles - 1) / tiles;
            range = std::min<uint64_t>(range, std::max<uint64_t>(32, (S + want_ranges - 1) / want_ranges));
            range = (range + 31) / 32 * 32;
            const uint64_t nranges = (S + range - 1) / range;
            const size_t smem = ((size_t)G * range + (size_t)G * kResCand) * wb;
            dim3 grid((unsigned)tiles, (unsigned)nranges);
            if (nranges > 65535) throw Error(SKYGPU_ERUNTIME, "gres: too many comparator ranges");
            SKY_CUDA(cudaEventRecord(e0, c.stream));
            if (w32) {
                SKY_CUDA(cudaFuncSetAttribute(k_gres_pairs_resident<uint32_t>,
                                              cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
                pdl_launch(k_gres_pairs_resident<uint32_t>, grid, kBlock, smem, c.stream,
                    (const uint32_t*)codes, (uint32_t)S, G, out.g_max, act, (uint32_t)na,
                    (uint32_t)range, d_den, c.d_slots + S_TESTS_GRES);
            } else {
                SKY_CUDA(cudaFuncSetAttribute(k_gres_pairs_resident<unsigned long long>,
                                              cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
                pdl_launch(k_gres_pairs_resident<unsigned long long>, grid, kBlock, smem, c.stream,
                    (const unsigned long long*)codes, (uint32_t)S, G, out.g_max, act, (uint32_t)na,
                    (uint32_t)range, d_den, c.d_slots + S_TESTS_GRES);
            }
        } else {
            const uint64_t cand_tiles = (na + kCandPerBlock - 1) / kCandPerBlock;
            const uint64_t target_blocks = (uint64_t)c.num_sms * 8;
            uint64_t ranges = (target_blocks + cand_tiles - 1) / cand_tiles;
            const uint64_t max_ranges = (S + 255) / 256;
            ranges = std::max<uint64_t>(1, std::min(ranges, max_ranges));
            uint64_t range = (S + ranges - 1) / ranges;
            range = (range + 31) / 32 * 32;
            ranges = (S + range - 1) / range;
            if (ranges > 65535) {
                ranges = 65535;
                range = (S + ranges - 1) / ranges;
            }
            dim3 grid((unsigned)cand_tiles, (unsigned)ranges);
            SKY_CUDA(cudaEventRecord(e0, c.stream));
            if (w32)
                pdl_launch(k_gres_pairs_tiled<uint32_t>, grid, kBlock, 0, c.stream,
                    (const uint32_t*)codes, (uint32_t)S, G, out.g_max, act, (uint32_t)na,
                    (uint32_t)range, d_den, c.d_slots + S_TESTS_GRES);
            else
                pdl_launch(k_gres_pairs_tiled<unsigned long long>, grid, kBlock, 0, c.stream,
                    (const unsigned long long*)codes, (uint32_t)S, G, out.g_max, act, (uint32_t)na,
                    (uint32_t)range, d_den, c.d_slots + S_TESTS_GRES);
        }
        SKY_CUDA(cudaEventRecord(e1, c.stream));
        SKY_LAUNCH_CHECK();
        trace_mark(c, "gres: tiled pair kernel");
        pdl_launch(k_finalize_den, grid_for(na, kBlock), kBlock, 0, c.stream, act, na, d_den);
        SKY_LAUNCH_CHECK();
        note_launch(c, 3);
        c.gres_timing_pending = true;  // resolved after the call's final sync
        out.steps = G;
        st.gres_steps = G;
        st.gres_kernel_launches += 1;
        return out;
    }
    // float64 path (codes above 127, d > 8, or projected-sum ties possible):
    // one step at a time on the reference's own projections floor(v*g)/g
    double* q = c.buf[B_PROJ].as<double>(S * d);
    for (int g = out.g_max; g >= 2 && na > 0; --g) {
        ++steps;
        pdl_launch(k_project, grid_for(S * d, kBlock), kBlock, 0, c.stream, d_skyv, S * d, g, q);
        SKY_LAUNCH_CHECK();
        dispatch_d(d, [&](auto DC) {
            constexpr int D = decltype(DC)::value;
            const size_t smem = sizeof(double) * (D > 0 ? 256 : 128) * (D > 0 ? D : d);
            SKY_CUDA(cudaEventRecord(e0, c.stream));
            pdl_launch(k_gres_pairs_f64<D>, grid_for(na, kBlock, 1 << 30), kBlock, smem, c.stream,
                q, (uint32_t)S, d, d_ids, act, (uint32_t)na, g, ties_possible ? 1 : 0, d_den,
                still, c.d_slots + S_TESTS_GRES);
            SKY_CUDA(cudaEventRecord(e1, c.stream));
        });
        SKY_LAUNCH_CHECK();
        note_launch(c, 2);
        na = select_flagged(c, act, still, act2, na);
        std::swap(act, act2);
        float ms = 0;
        SKY_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        kms += ms;
        ++klaunch;
    }
    if (na > 0) {
        pdl_launch(k_fill_den, grid_for(na, kBlock), kBlock, 0, c.stream, act, na, 1, d_den);
        SKY_LAUNCH_CHECK();
        note_launch(c);
    }
    out.steps = steps;
    st.gres_steps = steps;
    st.ms_gres_kernel += kms;
    st.gres_kernel_launches += klaunch;
    return out;
}

}  // namespace skygpu

namespace skygpu {

namespace {
// Grid plan inside the scan (gres.cpp:94-102 -> partition.cpp:88-95): the
// first projection floor(v*g)/g outside [0,1], in input (tuple, attribute)
// order, at the first step g = g_max.
__global__ void k_grid_projection_range(const double* __restrict__ v, uint64_t S, int d, int g,
                                        unsigned long long* __restrict__ slots) {
    pdl_wait();
    const double gd = (double)g;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < S * d;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t a = i / S, t = i - a * S;
        const double q = __ddiv_rn(floor(__dmul_rn(v[i], gd)), gd);
        if (q < 0.0 || q > 1.0) atomicMin(&slots[S_GRIDBAD], t * d + a);
    }
}
}  // namespace

void check_grid_projection(Ctx& c, const double* d_skyv, uint64_t S, int d, int g) {
    zero_slots(c);
    pdl_launch(k_grid_projection_range, grid_for(S * d, 256), 256, 0, c.stream, d_skyv, S, d, g,
                                                                         c.d_slots);
    SKY_LAUNCH_CHECK();
    note_launch(c);
    read_slots(c, S_GRIDBAD, 1);
    if (c.h_slots[S_GRIDBAD] != ~0ULL) {
        const uint64_t flat = c.h_slots[S_GRIDBAD];
        const uint64_t t = flat / d, a = flat % d;
        double v = 0;
        SKY_CUDA(cudaMemcpyAsync(&v, d_skyv + a * S + t, sizeof(double), cudaMemcpyDeviceToHost,
                                 c.stream));
        SKY_CUDA(cudaStreamSynchronize(c.stream));
        const double q = std::floor(v * g) / g;
        invalid("grid_cell: value " + std::to_string(q) + " in attribute " +
                std::to_string(a + 1) + " outside [0,1]; normalize the data first");
    }
}

}  // namespace skygpu
