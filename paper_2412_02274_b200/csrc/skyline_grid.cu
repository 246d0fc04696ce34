// skyline_grid.cu — one-pass skyline for LARGE skylines (SkyAlign-style static
// rank grid; the GPU recast of the paper's partition-level pruning,
// parallel.cpp:32-42 / partition.cpp:115-137, for data where most tuples
// survive, e.g. BASELINE config 5: 10 M anti-correlated tuples, d = 7).
//
// The round engine (skyline.cu) decides a prefix of the (sum, id) order and
// then filters every remaining tuple against the prefix's skyline; when the
// skyline is most of the input that is ~n^2/2 dominance tests.  Here every
// tuple is decided at once by the predecessor rule over the undecided set R:
//
//   t in R is kept  <=>  no s in R that precedes t in (sum, id, position)
//                        order dominates t
//
// (equivalent to the reference's SFS over R: a dominated s that dominates t
// is itself dominated by an earlier kept tuple, which then dominates t.)
//
// Pruning.  Every attribute value gets a 7-bit RANK code — the number of
// per-attribute sample quantiles (127 of them) <= the value.  Codes are
// monotone, so s dominates t  =>  code_j(s) <= code_j(t) for every j.  The
// codes of a tuple pack one byte per attribute into a u32 (d <= 4) or u64
// (d <= 8) word; the all-bytes-<= test is one SWAR subtraction (the guard-bit
// trick of the gres kernels).  Tuples are bucketed by bins of their codes:
// k0 fine bins along attribute 0 and k coarse bins along attributes 1..d-1;
// the cell order makes attribute 0 the fastest-varying, so the cells of one
// ROW (equal bins in attributes 1..d-1) are contiguous.  A comparator can
// only dominate a candidate from a cell <= the candidate's in every
// attribute, so a warp holding up to 128 candidates of one row streams, for
// every row <= its own (mixed-radix countdown over attributes 1..d-1), the
// ONE contiguous range of cells with attribute-0 bin <= its largest
// candidate's.  On C5 that visits ~0.1% of all pairs.  Code tests that pass
// (rare) take the exact float64 dominance test plus the precedence check —
// the only place exact values are read.
#include <cub/cub.cuh>

#include <cmath>
#include <cstdlib>
#include <type_traits>

#include "sky_common.cuh"

namespace skygpu {
namespace {

constexpr int kGB = 256;          // threads per block
constexpr int kBounds = 127;      // rank bounds per attribute -> codes 0..127
constexpr int kCand = 4;          // candidates per lane -> 128 per warp item
constexpr uint32_t kItem = 32 * kCand;

template <int D>
using GridWord = typename std::conditional<(D <= 4), uint32_t, unsigned long long>::type;

// Rank codes need only be MONOTONE in the value (s dominates t => every code
// of s <= t's; every pass is confirmed exactly), so they are read from a
// table: the value rounded to float (monotone), its bucket among 1024 equal
// buckets spanning the attribute's central sample quantiles (monotone), and
// T[j][bucket] = the number of quantiles falling in buckets <= it
// (non-decreasing) — one shared-memory byte instead of a 7-step binary
// search over float64 bounds.
constexpr int kRankBuckets = 1024;

struct RankTable {
    float lo[8], scale[8];
    uint8_t t[8][kRankBuckets];
};

__device__ __forceinline__ int rank_bucket(double x, float lo, float scale) {
    float u = __fmul_rn(__fsub_rn(__double2float_rn(x), lo), scale);
    u = fminf(fmaxf(u, 0.0f), (float)(kRankBuckets - 1));
    return (int)u;
}

// bounds[j][b] (b < 127) = the sample of rank 32(b+1)-1 among 4096 strided
// samples of attribute j over R (one CTA per attribute), and attribute j's
// code table
__global__ void __launch_bounds__(1024)
k_rank_bounds(const double* __restrict__ v, int d, const uint32_t* __restrict__ R, uint64_t r,
              double* __restrict__ bounds, RankTable* __restrict__ tab) {
    pdl_wait();
    using Sort = cub::BlockRadixSort<unsigned long long, 1024, 4>;
    __shared__ typename Sort::TempStorage tmp;
    const int j = blockIdx.x;
    unsigned long long items[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const uint64_t s = threadIdx.x * 4 + u;
        const uint64_t i = s * r / 4096;
        const uint64_t p = R ? R[i] : i;
        items[u] = ord_bits(v[p * d + j]);
    }
    Sort(tmp).Sort(items);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const uint32_t rank = threadIdx.x * 4 + u;
        if ((rank + 1) % 32 == 0 && rank < 4095)
            bounds[j * 128 + (rank + 1) / 32 - 1] = __longlong_as_double((long long)items[u]);
    }
    __shared__ float fb[kBounds];
    __shared__ int bk[kBounds];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const uint32_t rank = threadIdx.x * 4 + u;
        if ((rank + 1) % 32 == 0 && rank < 4095)
            fb[(rank + 1) / 32 - 1] = __double2float_rn(__longlong_as_double((long long)items[u]));
    }
    __syncthreads();
    const float lo = fb[0], hi = fb[kBounds - 1];
    const float scale = hi > lo ? __fdiv_rn((float)kRankBuckets, __fsub_rn(hi, lo)) : 0.0f;
    if (threadIdx.x < kBounds) bk[threadIdx.x] = rank_bucket((double)fb[threadIdx.x], lo, scale);
    __syncthreads();
    for (int b = threadIdx.x; b < kRankBuckets; b += blockDim.x) {
        int n = 0;
        for (int q = 0; q < kBounds; ++q) n += bk[q] <= b;
        tab->t[j][b] = (uint8_t)n;
    }
    if (threadIdx.x == 0) {
        tab->lo[j] = lo;
        tab->scale[j] = scale;
    }
}

// rank codes, cell of every tuple of R (bin0 + k0 * row), cell histogram
template <int D>
__global__ void __launch_bounds__(kGB)
k_rank_codes(const double* __restrict__ v, const uint32_t* __restrict__ R, uint32_t r,
             const RankTable* __restrict__ tab, int k0, int k, GridWord<D>* __restrict__ code,
             uint32_t* __restrict__ cell, uint32_t* __restrict__ count,
             uint32_t* __restrict__ iota) {
    pdl_wait();
    using W = GridWord<D>;
    __shared__ uint8_t st[D][kRankBuckets];
    __shared__ float slo[D], ssc[D];
    for (int i = threadIdx.x; i < D * kRankBuckets / 4; i += blockDim.x)
        reinterpret_cast<uint32_t*>(&st[0][0])[i] =
            reinterpret_cast<const uint32_t*>(&tab->t[0][0])[i];
    if (threadIdx.x < D) {
        slo[threadIdx.x] = tab->lo[threadIdx.x];
        ssc[threadIdx.x] = tab->scale[threadIdx.x];
    }
    __syncthreads();
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < r; i += gridDim.x * blockDim.x) {
        const uint64_t p = R ? R[i] : i;
        W w = 0;
        uint32_t row = 0, mul = 1, b0 = 0;
#pragma unroll
        for (int j = 0; j < D; ++j) {
            const double x = v[p * D + j];
            const int lo = st[j][rank_bucket(x, slo[j], ssc[j])];
            w |= (W)lo << (8 * j);
            if (j == 0) {
                b0 = (uint32_t)((lo * k0) >> 7);
            } else {
                row += (uint32_t)((lo * k) >> 7) * mul;
                mul *= (uint32_t)k;
            }
        }
        const uint32_t cl = b0 + (uint32_t)k0 * row;
        code[i] = w;
        cell[i] = cl;
        if (iota) iota[i] = i;
        else atomicAdd(&count[cl], 1u);
    }
}

template <class W>
__global__ void k_cell_scatter(const W* __restrict__ code, const uint32_t* __restrict__ cell,
                               uint32_t r, const uint32_t* __restrict__ seg,
                               uint32_t* __restrict__ cursor, W* __restrict__ scode,
                               uint32_t* __restrict__ sidx) {
    pdl_wait();
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < r; i += gridDim.x * blockDim.x) {
        const uint32_t cl = cell[i];
        const uint32_t pos = seg[cl] + atomicAdd(&cursor[cl], 1u);
        scode[pos] = code[i];
        sidx[pos] = i;
    }
}

// sorted-cell form of the bucketing (default): the cells sorted by a stable
// radix sort (no per-tuple atomics on a 4M-entry histogram), then the
// segment table from the run boundaries: seg[c] = first sorted position with
// cell >= c, for every c in [0, ncells]
__global__ void k_seg_bounds(const uint32_t* __restrict__ skey, uint32_t r, uint32_t ncells,
                             uint32_t* __restrict__ seg) {
    pdl_wait();
    for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q <= r; q += gridDim.x * blockDim.x) {
        const uint32_t hi = q < r ? skey[q] : ncells;
        const uint32_t lo = q > 0 ? skey[q - 1] + 1 : 0;
        for (uint32_t c = lo; c <= hi; ++c) seg[c] = q;
    }
}

template <class W>
__global__ void k_gather_codes(const uint32_t* __restrict__ sidx, uint32_t r,
                               const W* __restrict__ code, W* __restrict__ scode) {
    pdl_wait();
    for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < r; q += gridDim.x * blockDim.x)
        scode[q] = code[sidx[q]];
}

// each tuple's exact record in cell order: its D float64 values at
// rec[pos * (D + 1)] (stride D + 1 doubles: 64-byte records for D = 7; the
// sum key is recomputed by exact_rec when it matters) — the TMA decide kernel's
// exact follow-up then reads one contiguous record per side instead of
// chasing sidx -> R -> values and keys.  Gathered (writes coalesced, the
// 64-byte reads random) after the scatter.
template <int D>
__global__ void k_gather_rec(const uint32_t* __restrict__ sidx, uint32_t r,
                             const double* __restrict__ v,
                             const unsigned long long* __restrict__ key,
                             const uint32_t* __restrict__ R, double* __restrict__ rec,
                             const GridWord<D>* __restrict__ code, GridWord<D>* __restrict__ scode) {
    pdl_wait();
    for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < r; q += gridDim.x * blockDim.x) {
        const uint32_t i = sidx[q];
        if (code) scode[q] = code[i];
        const uint64_t p = R ? R[i] : i;
        double x[D];
#pragma unroll
        for (int j = 0; j < D; ++j) x[j] = v[p * D + j];
        double* o = rec + (uint64_t)q * (D + 1);  // (slot D unused: 64-byte records for D = 7)
#pragma unroll
        for (int j = 0; j < D; ++j) o[j] = x[j];
    }
}

// the scatter and the record gather in one pass (default):
// a thread reads its own row (coalesced: consecutive threads, consecutive
// rows), takes its slot, and the warp writes its 32 records through shared
// memory so that every record leaves as whole 32-byte sectors (a thread
// storing its D + 1 doubles one by one makes D + 1 partial-sector writes —
// the form round 2 measured at 1.6 ms against the gather's 0.6 ms)
template <int D>
__global__ void __launch_bounds__(kGB)
k_cell_scatter_rec(const GridWord<D>* __restrict__ code, const uint32_t* __restrict__ cell,
                   uint32_t r, const uint32_t* __restrict__ seg, uint32_t* __restrict__ cursor,
                   GridWord<D>* __restrict__ scode, uint32_t* __restrict__ sidx,
                   const double* __restrict__ v, const uint32_t* __restrict__ R,
                   double* __restrict__ rec) {
    pdl_wait();
    constexpr int RS = D + 1;  // record stride in doubles
    constexpr int SS = RS | 1;  // staging stride (odd: no bank conflicts either way)
    __shared__ double stage[kGB / 32][32 * SS];
    __shared__ uint32_t spos[kGB / 32][32];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t nround = (r + gridDim.x * blockDim.x - 1) / (gridDim.x * blockDim.x);
    for (uint32_t it = 0; it < nround; ++it) {
        const uint32_t i = (it * gridDim.x + blockIdx.x) * blockDim.x + threadIdx.x;
        uint32_t pos = ~0u;
        if (i < r) {
            const uint32_t cl = cell[i];
            pos = seg[cl] + atomicAdd(&cursor[cl], 1u);
            scode[pos] = code[i];
            sidx[pos] = i;
            const uint64_t p = R ? R[i] : i;
#pragma unroll
            for (int j = 0; j < D; ++j) stage[warp][lane * SS + j] = v[p * D + j];
            stage[warp][lane * SS + D] = 0.0;
        }
        spos[warp][lane] = pos;
        __syncwarp();
        // 32 records x RS doubles, written RS doubles (one record) per RS lanes
        for (uint32_t e = lane; e < 32u * RS; e += 32) {
            const uint32_t t = e / RS, k = e - t * RS;
            const uint32_t q = spos[warp][t];
            if (q != ~0u) rec[(uint64_t)q * RS + k] = stage[warp][t * SS + k];
        }
        __syncwarp();
    }
}

// work items: (row, first sorted position) chunks of <= 128 candidates; a
// sharded call keeps only the rows this shard owns (row % world == rank)
__global__ void k_row_items(const uint32_t* __restrict__ seg, uint32_t nrows, int k0,
                            uint2* __restrict__ items, unsigned* __restrict__ ctr, int rank,
                            int world) {
    pdl_wait();
    for (uint32_t row = blockIdx.x * blockDim.x + threadIdx.x; row < nrows;
         row += gridDim.x * blockDim.x) {
        if ((int)(row % (uint32_t)world) != rank) continue;
        const uint32_t a = seg[row * k0], n = seg[(row + 1) * k0] - a;
        if (!n) continue;
        const uint32_t ch = (n + kItem - 1) / kItem;
        const uint32_t base = atomicAdd(&ctr[0], ch);
        for (uint32_t u = 0; u < ch; ++u) items[base + u] = make_uint2(row, a + u * kItem);
    }
}

// exact test: does the tuple at sorted position qs dominate, and precede,
// the tuple at sorted position qt?
template <int D>
__device__ __noinline__ bool exact_pred(const double* __restrict__ v,
                                        const unsigned long long* __restrict__ key,
                                        const int64_t* __restrict__ ids,
                                        const uint32_t* __restrict__ R,
                                        const uint32_t* __restrict__ sidx, uint32_t qs,
                                        uint32_t qt) {
    const uint32_t is = sidx[qs], it = sidx[qt];
    const uint64_t ps = R ? R[is] : is, pt = R ? R[it] : it;
    double s[D], t[D];
#pragma unroll
    for (int j = 0; j < D; ++j) {
        s[j] = v[ps * D + j];
        t[j] = v[pt * D + j];
    }
    if (!dom_f64<D>(s, t)) return false;
    const unsigned long long ks = key[ps], kt = key[pt];
    if (ks != kt) return ks < kt;  // dominance implies ks <= kt
    if (!ids) return ps < pt;  // (ids in flight: position order, checked later)
    const int64_t is_ = ids[ps], it_ = ids[pt];
    return is_ < it_ || (is_ == it_ && ps < pt);
}

// zero iff every byte of s <= the byte of t, given tg = t | 0x80.. (codes
// <= 127): the guard bits of tg - s that a borrow cleared.  Accumulated
// with min() over a tile, a zero result flags a pass in one instruction.
__device__ __forceinline__ uint32_t code_miss(uint32_t tg, uint32_t s) {
    return ~(tg - s) & 0x80808080u;
}
__device__ __forceinline__ uint32_t code_miss(unsigned long long tg, unsigned long long s) {
    const unsigned long long x = tg - s;
    return ~((uint32_t)x & (uint32_t)(x >> 32)) & 0x80808080u;
}
// a code word that never passes: byte 0 = 0x80 clears guard bit 7 of
// (t0 | 0x80) - 0x80 for every t0
template <class W>
__device__ __forceinline__ W code_never() {
    return (W)0x80;
}

// exact follow-up of the code passes of one staged tile for candidate slot
// u of this lane (skipping comparator `self`, a sorted position or ~0):
// false when a dominating predecessor was found
template <int D, class W>
__device__ __forceinline__ bool tile_exact(const W* st, const uint32_t* sp, W tgu, uint32_t qt,
                                           uint32_t self, const double* __restrict__ v,
                                           const unsigned long long* __restrict__ key,
                                           const int64_t* __restrict__ ids,
                                           const uint32_t* __restrict__ R,
                                           const uint32_t* __restrict__ sidx) {
    uint32_t m = 0;
#pragma unroll 8
    for (int j = 0; j < 32; ++j) m |= (code_miss(tgu, st[j]) == 0u ? 1u : 0u) << j;
    while (m) {
        const int j = __ffs(m) - 1;
        m &= m - 1;
        const uint32_t qs = sp[j];
        if (qs != self && qs != ~0u && exact_pred<D>(v, key, ids, R, sidx, qs, qt)) return false;
    }
    return true;
}

// exact_pred over the cell-ordered records (k_cell_scatter_rec): values and
// key from one record per side; ties of the key fall back to ids/positions
template <int D>
__device__ __forceinline__ bool exact_rec(const double* __restrict__ rec,
                                          const int64_t* __restrict__ ids,
                                          const uint32_t* __restrict__ R,
                                          const uint32_t* __restrict__ sidx, uint32_t qs,
                                          uint32_t qt) {
    const double* a = rec + (uint64_t)qs * (D + 1);
    const double* b = rec + (uint64_t)qt * (D + 1);
    double s[D], t[D];
#pragma unroll
    for (int j = 0; j < D; ++j) {
        s[j] = a[j];
        t[j] = b[j];
    }
    if (!dom_f64<D>(s, t)) return false;
    // the (sum, id) precedence only matters when the float64 sums tie
    // (dominance implies sum(s) <= sum(t)): the sums are recomputed here, for
    // the few confirmed dominances, exactly as K1 computes the keys
    // (left-to-right __dadd_rn from 0.0, ord_bits) — the records carry no key,
    // which spares the gather a random 8-byte read per tuple
    double ss = 0.0, st = 0.0;
#pragma unroll
    for (int j = 0; j < D; ++j) {
        ss = __dadd_rn(ss, s[j]);
        st = __dadd_rn(st, t[j]);
    }
    const unsigned long long ks = ord_bits(ss), kt = ord_bits(st);
    if (ks != kt) return ks < kt;  // dominance implies ks <= kt
    const uint32_t is = sidx[qs], it = sidx[qt];
    const uint64_t ps = R ? R[is] : is, pt = R ? R[it] : it;
    if (!ids) return ps < pt;  // (ids in flight: position order, checked later)
    const int64_t is_ = ids[ps], it_ = ids[pt];
    return is_ < it_ || (is_ == it_ && ps < pt);
}

// code-pass flags of one staged tile for the first KC candidate slots
template <int KC, class W>
__device__ __forceinline__ unsigned tile_hits(const W* st, const W (&tg)[kCand]) {
    uint32_t acc[KC];
#pragma unroll
    for (int u = 0; u < KC; ++u) acc[u] = 0xFFFFFFFFu;
#pragma unroll 8
    for (int j = 0; j < 32; ++j) {
        const W s = st[j];
#pragma unroll
        for (int u = 0; u < KC; ++u) acc[u] = min(acc[u], code_miss(tg[u], s));
    }
    unsigned hm = 0;
#pragma unroll
    for (int u = 0; u < KC; ++u) hm |= (acc[u] == 0u ? 1u : 0u) << u;
    return hm;
}

// K6: persistent warps pull (row, chunk) items; each lane holds up to kCand
// candidate slots.  The chunk is first tested against itself (exact
// follow-up of every pass except the candidate itself); then the comparator
// ranges — one per row <= the item's row, own row first, minus the chunk —
// are streamed 32 codes at a time through shared memory: tiles are filled
// across row boundaries and the next tile's load is issued before the
// current one is tested.  The tile test is 4 integer instructions per
// (candidate, comparator) with no branch (min-accumulated miss bits); a tile
// with a pass (rare: equal codes, near-dominators) gets the exact follow-up.
// Dominated candidates free their slots: when the live ones fit in fewer
// slots the warp repacks them (shared memory) and tests only the occupied
// slots.  Warp exit when every candidate is decided.  keep[R index] = 1 for
// kept tuples.
template <int D>
__global__ void __launch_bounds__(kGB)
k_grid_decide(const double* __restrict__ v, const unsigned long long* __restrict__ key,
              const int64_t* __restrict__ ids, const uint32_t* __restrict__ R,
              const GridWord<D>* __restrict__ scode, const uint32_t* __restrict__ sidx,
              const uint32_t* __restrict__ seg, const uint2* __restrict__ items,
              unsigned* __restrict__ ctr, int k0, int k, uint8_t* __restrict__ keep,
              unsigned long long* __restrict__ tests) {
    pdl_wait();
    using W = GridWord<D>;
    __shared__ W stage[kGB / 32][32];
    __shared__ uint32_t spos[kGB / 32][32];
    __shared__ W pk_tg[kGB / 32][kItem];
    __shared__ uint32_t pk_q[kGB / 32][kItem];
    const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const W H = (W)0x8080808080808080ULL;
    const uint32_t nitems = ctr[0];
    W* st = stage[wib];
    uint32_t* sp = spos[wib];
    uint32_t wj[D];  // row-id weight of attribute j >= 1
    wj[0] = 0;
    if (D > 1) wj[1] = 1;
#pragma unroll
    for (int j = 2; j < D; ++j) wj[j] = wj[j - 1] * (uint32_t)k;
    unsigned long long cnt = 0;
    for (;;) {
        uint32_t it = 0;
        if (lane == 0) it = atomicAdd(&ctr[1], 1u);
        it = __shfl_sync(0xffffffffu, it, 0);
        if (it >= nitems) break;
        const uint2 item = items[it];
        const uint32_t own = item.x, first = item.y;
        const uint32_t end = min(seg[(own + 1) * k0], first + kItem);
        W tg[kCand];
        uint32_t qt[kCand];
        unsigned alive = 0;
#pragma unroll
        for (int u = 0; u < kCand; ++u) {
            qt[u] = first + u * 32 + lane;
            tg[u] = qt[u] < end ? (scode[qt[u]] | H) : (W)0;
            alive |= (qt[u] < end ? 1u : 0u) << u;
        }
        unsigned valid = alive;
        int kc = (int)((end - first + 31) / 32);  // occupied slots (warp-uniform)
        // ---- the chunk against itself
        for (int t = 0; t < kc; ++t) {
            const uint32_t q = first + t * 32 + lane;
            st[lane] = q < end ? scode[q] : code_never<W>();
            sp[lane] = q < end ? q : ~0u;
            __syncwarp();
#pragma unroll
            for (int u = 0; u < kCand; ++u) {
                if ((alive >> u) & 1u) {
                    if (!tile_exact<D>(st, sp, tg[u], qt[u], qt[u], v, key, ids, R, sidx))
                        alive &= ~(1u << u);
                }
            }
            cnt += (unsigned long long)min(32u, end - (first + t * 32)) * __popc(alive);
            __syncwarp();
        }
        // largest attribute-0 bin among the candidates = that of the last one
        const uint32_t od0 = (uint32_t)((((uint32_t)scode[end - 1] & 0xFFu) * (uint32_t)k0) >> 7);
        // the rows <= own in every coarse attribute, in mixed-radix countdown
        // order (attribute 1 fastest): position p -> digit j = od[j] -
        // (p / base[j]) % (od[j] + 1).  Position 0 is the own row.
        uint32_t od[D], base[D];
        uint32_t total = 1;
#pragma unroll
        for (int j = 1; j < D; ++j) {
            od[j] = (own / wj[j]) % (uint32_t)k;
            base[j] = total;
            total *= od[j] + 1;
        }
        auto row_at = [&](uint32_t p) -> uint32_t {
            uint32_t rw = 0;
#pragma unroll
            for (int j = 1; j < D; ++j) rw += (od[j] - (p / base[j]) % (od[j] + 1)) * wj[j];
            return rw;
        };
        // own row: [row start, first) then [end, row end at od0)
        uint32_t cur = seg[own * k0], rend = first;
        uint32_t gap_end = seg[own * k0 + od0 + 1];
        bool rows_left = D > 1 && total > 1, gap = true;
        // the other rows are opened from a window of 32 consecutive countdown
        // positions whose comparator ranges the lanes load in parallel (one
        // row each): empty rows cost nothing, a non-empty one a shuffle
        uint32_t lin = 1, wlo = 0, whi = 0;  // next window start; this lane's range
        unsigned nzmask = 0;                    // window rows not yet opened, non-empty
        // next <= 32 comparator positions across rows (warp-uniform walk)
        auto fill = [&](uint32_t& mypos) -> uint32_t {
            uint32_t filled = 0;
            mypos = ~0u;
            while (filled < 32) {
                if (cur == rend) {
                    if (gap) {
                        gap = false;
                        cur = end;
                        rend = gap_end;
                        continue;
                    }
                    if (!nzmask) {
                        if (!rows_left || lin >= total) {
                            rows_left = false;
                            break;
                        }
                        const uint32_t p = lin + lane;
                        wlo = whi = 0;
                        if (p < total) {
                            const uint32_t rw = row_at(p);
                            wlo = seg[rw * k0];
                            whi = seg[rw * k0 + od0 + 1];
                        }
                        nzmask = __ballot_sync(0xffffffffu, whi > wlo);
                        lin += 32;
                        continue;
                    }
                    const int f = __ffs(nzmask) - 1;
                    nzmask &= nzmask - 1;
                    cur = __shfl_sync(0xffffffffu, wlo, f);
                    rend = __shfl_sync(0xffffffffu, whi, f);
                    continue;
                }
                const uint32_t take = min(32u - filled, rend - cur);
                if (lane >= filled && lane < filled + take) mypos = cur + (lane - filled);
                filled += take;
                cur += take;
            }
            return filled;
        };
        // repack the live candidates into the first slots
        auto repack = [&](int live) {
            unsigned mine = __popc(alive);
            unsigned incl = mine;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
                if ((int)lane >= o) incl += y;
            }
            unsigned at = incl - mine;
#pragma unroll
            for (int u = 0; u < kCand; ++u) {
                if ((alive >> u) & 1u) {
                    pk_tg[wib][at] = tg[u];
                    pk_q[wib][at] = qt[u];
                    ++at;
                } else if ((valid >> u) & 1u) {
                    keep[sidx[qt[u]]] = 0;  // decided: dominated
                }
            }
            __syncwarp();
            alive = 0;
#pragma unroll
            for (int u = 0; u < kCand; ++u) {
                const int i = u * 32 + (int)lane;
                if (i < live) {
                    tg[u] = pk_tg[wib][i];
                    qt[u] = pk_q[wib][i];
                    alive |= 1u << u;
                }
            }
            valid = alive;
            kc = (live + 31) / 32;
            __syncwarp();
        };
        uint32_t pos_next;
        int live = __reduce_add_sync(0xffffffffu, __popc(alive));
        uint32_t npos = live ? fill(pos_next) : 0;
        W code_next = pos_next != ~0u ? scode[pos_next] : code_never<W>();
        while (npos) {
            if (live <= 32 * (kc - 1)) repack(live);
            st[lane] = code_next;
            sp[lane] = pos_next;
            const uint32_t n = npos;
            __syncwarp();
            npos = fill(pos_next);  // prefetch the next tile
            code_next = pos_next != ~0u ? scode[pos_next] : code_never<W>();
            unsigned hm;
            switch (kc) {
                case 1: hm = tile_hits<1>(st, tg); break;
                case 2: hm = tile_hits<2>(st, tg); break;
                case 3: hm = tile_hits<3>(st, tg); break;
                default: hm = tile_hits<4>(st, tg); break;
            }
            cnt += (unsigned long long)n * __popc(alive);
            hm &= alive;
            if (__any_sync(0xffffffffu, hm != 0u)) {  // rare: exact follow-up
#pragma unroll
                for (int u = 0; u < kCand; ++u) {
                    if ((hm >> u) & 1u) {
                        if (!tile_exact<D>(st, sp, tg[u], qt[u], ~0u, v, key, ids, R, sidx))
                            alive &= ~(1u << u);
                    }
                }
            }
            __syncwarp();
            live = __reduce_add_sync(0xffffffffu, __popc(alive));
            if (!live) break;
        }
#pragma unroll
        for (int u = 0; u < kCand; ++u)
            if ((valid >> u) & 1u) keep[sidx[qt[u]]] = (alive >> u) & 1u;
    }
    add_count(tests, cnt);
}

// ---------------------------------------------------------------------------
// K6 (default): the same decision, restructured around two facts of the ALU
// kernel above — (1) a (candidate, comparator) code test costs ~6 issued ALU
// instructions there (3 for the test, the rest the per-lane tile walk), and
// (2) each comparator row is fetched by per-lane loads whose L2 latency the
// warp must hide on its own.
//
//  * Bitset test.  An item's 128 candidates are turned into per-attribute
//    tables in shared memory: tab[j][r] = the 128-bit set of candidates whose
//    rank code on attribute j is >= r (one ballot per (j, r) inside the
//    candidates' code range).  The candidates a comparator s code-dominates
//    are then AND_j tab[j][code_j(s)]: D 16-byte shared loads and ~3D/2 LOP3
//    test s against all 128 candidates at once (bitmap skyline technique),
//    instead of 128 SWAR tests.
//  * TMA bulk staging.  Warp 0 of the CTA is a producer: it walks the same
//    comparator ranges (own chunk, own row, then every row <= the item's
//    row) and streams them with cp.async.bulk into a 3-stage (3 x 384 codes) shared-memory
//    ring (mbarrier complete_tx); warps 1..3 consume stages.  Ranges are
//    copied at 16-byte granularity, so up to one code on either side of a
//    range is an extra comparator — harmless: the predecessor rule may test
//    t against ANY tuple of R (a tuple never dominates itself).
//  * Code passes take the exact float64 + precedence test (exact_pred), as
//    before; a confirmed dominator clears the candidate's bit in the CTA's
//    alive mask, and the item ends as soon as no candidate is alive.
// ---------------------------------------------------------------------------
constexpr int kTB = 128;          // threads: warp 0 producer, warps 1..3 consumers
constexpr int kTCons = kTB / 32 - 1;
// (compile-time knobs: scripts/build_k6_variant.sh NAME -DSKY_K6_...=.. builds a
// variant beside the in-tree library for same-box timing, scripts/gpu_k6_variants.sh.
// Measured on C5, 8 CTAs/SM each: 4 x 256 codes 5.89 ms, 3 x 384 5.51 ms, 2 x 576
// 5.53 ms, 4 x 288 5.64 ms, 6 x 192 5.95 ms, 4 x 320 (7 CTAs/SM) 6.19 ms — long
// stages matter more than many; 384 = 4 full rounds of the 3 consumer warps.)
#ifndef SKY_K6_STAGES
#define SKY_K6_STAGES 3
#endif
#ifndef SKY_K6_STAGE_CAP
#define SKY_K6_STAGE_CAP 384
#endif
#ifndef SKY_K6_MAX_PIECES
#define SKY_K6_MAX_PIECES 24
#endif
constexpr int kStages = SKY_K6_STAGES;
constexpr int kStageCap = SKY_K6_STAGE_CAP;    // codes per stage
constexpr int kMaxPieces = SKY_K6_MAX_PIECES;  // ranges per stage
constexpr int kTabR = 129;        // table entries per attribute: codes 0..127, 128 = never
#ifndef SKY_K6_HIT_CAP
#define SKY_K6_HIT_CAP 128
#endif
constexpr int kHitCap = SKY_K6_HIT_CAP;  // batched exact follow-ups per consumer warp

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(
                     smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity, int site = 0) {
    const uint32_t a = smem_u32(bar);
    uint32_t ok = 0;
#ifdef SKYGPU_K6_WATCHDOG
    unsigned long long spins = 0;
#endif
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(a), "r"(parity)
            : "memory");
#ifdef SKYGPU_K6_WATCHDOG  // debug build: name the wait that never completes, then trap
        if (!ok && ++spins == (1ull << 24) && (threadIdx.x & 31) == 0) {
            unsigned long long st;
            asm volatile("ld.shared.b64 %0, [%1];" : "=l"(st) : "r"(a));
            printf("[K6 watchdog] block %d warp %d site %d bar@%u parity %u state %llx\n",
                   blockIdx.x, threadIdx.x >> 5, site, a, parity, st);
        }
        if (!ok && spins == (1ull << 25)) __trap();
#else
        (void)site;
#endif
    } while (!ok);
}
// global -> shared bulk copy (16-byte aligned, size a multiple of 16),
// completion counted on `bar` in bytes
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// x / b for x < 2^24 from a float reciprocal (one correction step each way):
// the producer's mixed-radix row walk without integer division
__device__ __forceinline__ uint32_t div_rcp(uint32_t x, uint32_t b, float inv) {
    uint32_t q = __float2uint_rz(__uint2float_rn(x) * inv);
    if (q * b > x) --q;
    if ((q + 1) * b <= x) ++q;
    return q;
}

template <int D>
struct alignas(16) DecideSmem {
    using W = GridWord<D>;
    uint4 tab[D * kTabR];                 // candidate bitsets per (attribute, code)
    W ring[kStages][kStageCap];           // staged comparator codes
    uint32_t pslot[kStages][kMaxPieces];  // first slot of each staged range
    uint32_t ppos[kStages][kMaxPieces];   // its sorted position
    uint32_t nslot[kStages], npiece[kStages], nreal[kStages], last[kStages];
    uint64_t full[kStages], empty[kStages];
    uint32_t alive[4];
    uint32_t item;
    uint8_t lo4[4][8], hi4[4][8];         // each warp's candidate code range per attribute
    uint8_t binlo[132];                   // first code of coarse bin b (b <= k), 128 beyond
    uint2 hits[kTCons][kHitCap];          // a consumer warp's code passes, tested in parallel
};

template <int D>
__global__ void __launch_bounds__(kTB, 8)
k_grid_decide_tma(const double* __restrict__ rec, const int64_t* __restrict__ ids,
                  const uint32_t* __restrict__ R,
                  const GridWord<D>* __restrict__ scode, const uint32_t* __restrict__ sidx,
                  const uint32_t* __restrict__ seg, const uint2* __restrict__ items,
                  unsigned* __restrict__ ctr, int k0, int k, uint8_t* __restrict__ keep,
                  unsigned long long* __restrict__ tests) {
    pdl_wait();
    using W = GridWord<D>;
    constexpr uint32_t kAlign = 16 / sizeof(W);  // codes per 16 bytes
    __shared__ DecideSmem<D> sm;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&sm.full[s], 1);
            mbar_init(&sm.empty[s], kTCons);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    // first code of every coarse bin: bin(c) = (c * k) >> 7 (k_rank_codes)
    for (uint32_t b = threadIdx.x; b < 132; b += blockDim.x)
        sm.binlo[b] = (uint8_t)min(128u, (b * 128u + (uint32_t)k - 1u) / (uint32_t)k);
    __syncthreads();
    const uint32_t nitems = ctr[0];
    uint32_t wj[D];
    wj[0] = 0;
    if (D > 1) wj[1] = 1;
#pragma unroll
    for (int j = 2; j < D; ++j) wj[j] = wj[j - 1] * (uint32_t)k;
    uint32_t ps = 0, pphase = 0;  // producer ring position (warp 0)
    uint32_t cs = 0, cphase = 0;  // consumer ring position (warps 1..3)
    unsigned long long cnt = 0, ucnt = 0;  // tests, (comparator, item) units
    for (;;) {
        if (threadIdx.x == 0) sm.item = atomicAdd(&ctr[1], 1u);
        __syncthreads();
        const uint32_t it = sm.item;
        if (it >= nitems) break;
        const uint2 item = items[it];
        const uint32_t own = item.x, first = item.y;
        const uint32_t end = min(seg[(own + 1) * k0], first + kItem);
        // ---- candidate bitset tables: warp w builds word w of every entry
        {
            const uint32_t q = first + threadIdx.x;
            const bool valid = q < end;
            const W cw = valid ? scode[q] : (W)0;
            const unsigned vmask = __ballot_sync(0xffffffffu, valid);
            // the item's candidates share one row: on attributes 1.. their codes
            // lie in ONE coarse bin, and only entries inside the item's code
            // range are ever read (the consumers' predicates) — so a warp fills
            // its word for that bin's codes only (attribute 0, whose fine bins
            // an item spans, and grids of < 4 bins keep the whole range)
            const W c0w = scode[first];
#pragma unroll
            for (int j = 0; j < D; ++j) {
                const uint32_t x = (uint32_t)(cw >> (8 * j)) & 0xFFu;
                const uint32_t lo = __reduce_min_sync(0xffffffffu, valid ? x : 255u);
                const uint32_t hi = __reduce_max_sync(0xffffffffu, valid ? x : 0u);
                uint32_t* T = reinterpret_cast<uint32_t*>(&sm.tab[j * kTabR]) + warp;
                uint32_t flo = 0, fhi = (uint32_t)kTabR - 1u;
                if (j >= 1 && k >= 4) {
                    const uint32_t b = ((((uint32_t)(c0w >> (8 * j)) & 0xFFu)) * (uint32_t)k) >> 7;
                    flo = sm.binlo[b];
                    fhi = sm.binlo[b + 1];
                }
                for (uint32_t r = flo + lane; r <= fhi; r += 32)
                    if (r <= lo || r > hi) T[r * 4] = r <= lo ? vmask : 0u;
                for (uint32_t r = lo + 1; r <= hi; ++r) {
                    const unsigned b = __ballot_sync(0xffffffffu, valid && x >= r);
                    if ((r & 31u) == lane) T[r * 4] = b;
                }
                if (lane == 0) {
                    sm.lo4[warp][j] = (uint8_t)lo;
                    sm.hi4[warp][j] = (uint8_t)hi;
                }
            }
            if (lane == 0) sm.alive[warp] = vmask;
        }
        __syncthreads();
        if (warp == 0) {
            // ================= producer: walk the comparator ranges
            uint32_t used = 0, np = 0, nr = 0;
            bool open = false, stop = false;
            // (the consumers clear alive bits concurrently: ONE lane reads
            // and the warp takes its answer — lanes reading for themselves
            // can disagree and diverge around the warp-level waits below)
            auto all_dead = [&]() {
                uint32_t x = 0;
                if (lane == 0) {
                    const volatile uint32_t* a = sm.alive;
                    x = a[0] | a[1] | a[2] | a[3];
                }
                return __shfl_sync(0xffffffffu, x, 0) == 0u;
            };
            auto close = [&](bool fin) {
                if (lane == 0) {
                    sm.nslot[ps] = used;
                    sm.npiece[ps] = np;
                    sm.nreal[ps] = nr;
                    sm.last[ps] = fin ? 1u : 0u;
                    mbar_arrive(&sm.full[ps]);
                }
                __syncwarp();
                if (++ps == kStages) {
                    ps = 0;
                    pphase ^= 1u;
                }
                open = false;
            };
            auto emit = [&](uint32_t lo, uint32_t hi) {
                while (lo < hi && !stop) {
                    if (!open) {
                        if (all_dead()) {
                            stop = true;
                            break;
                        }
                        mbar_wait(&sm.empty[ps], pphase ^ 1u, 1);
                        used = np = nr = 0;
                        open = true;
                    }
                    const int space = kStageCap - (int)used - 2 * (int)(kAlign - 1);
                    if (space <= 0 || np == (uint32_t)kMaxPieces) {
                        close(false);
                        continue;
                    }
                    const uint32_t take = min(hi - lo, (uint32_t)space);
                    const uint32_t a = lo & ~(kAlign - 1);
                    const uint32_t b = (lo + take + kAlign - 1) & ~(kAlign - 1);
                    if (lane == 0) {
                        const uint32_t bytes = (b - a) * (uint32_t)sizeof(W);
                        mbar_expect_tx(&sm.full[ps], bytes);
                        bulk_g2s(&sm.ring[ps][used], scode + a, bytes, &sm.full[ps]);
                        sm.pslot[ps][np] = used;
                        sm.ppos[ps][np] = a;
                    }
                    used += b - a;
                    ++np;
                    nr += take;
                    lo += take;
                }
            };
            // the chunk itself, then the own row around it
            emit(first, end);
            const uint32_t od0 =
                (uint32_t)((((uint32_t)scode[end - 1] & 0xFFu) * (uint32_t)k0) >> 7);
            emit(seg[own * k0], first);
            emit(end, seg[own * k0 + od0 + 1]);
            // rows <= own in every coarse attribute (mixed-radix countdown,
            // attribute 1 fastest), 32 rows per window (one per lane)
            uint32_t od[D], base[D];
            float ib[D], ir[D];
            uint32_t total = 1;
#pragma unroll
            for (int j = 1; j < D; ++j) {
                od[j] = (own / wj[j]) % (uint32_t)k;
                base[j] = total;
                ib[j] = 1.0f / (float)total;
                ir[j] = 1.0f / (float)(od[j] + 1);
                total *= od[j] + 1;
            }
            for (uint32_t lin = 1; lin < total && !stop; lin += 32) {
                const uint32_t p = lin + lane;
                uint32_t wlo = 0, whi = 0;
                if (p < total) {  // (total <= rows < 2^22: div_rcp is exact)
                    uint32_t rw = 0;
#pragma unroll
                    for (int j = 1; j < D; ++j) {
                        const uint32_t t = div_rcp(p, base[j], ib[j]);
                        const uint32_t dj = t - div_rcp(t, od[j] + 1, ir[j]) * (od[j] + 1);
                        rw += (od[j] - dj) * wj[j];
                    }
                    wlo = seg[rw * k0];
                    whi = seg[rw * k0 + od0 + 1];
                }
                unsigned nz = __ballot_sync(0xffffffffu, whi > wlo);
                while (nz && !stop) {
                    const int f = __ffs(nz) - 1;
                    nz &= nz - 1;
                    emit(__shfl_sync(0xffffffffu, wlo, f), __shfl_sync(0xffffffffu, whi, f));
                }
            }
            if (!open) {  // an empty stage carries the end marker
                mbar_wait(&sm.empty[ps], pphase ^ 1u, 2);
                used = np = nr = 0;
            }
            close(true);
        } else {
            // ================= consumers: test staged comparators
            const uint32_t cw = warp - 1;
            // the item's code range per attribute: a comparator code <= lo
            // passes every candidate on that attribute (the entry would be
            // all-ones: no table read), one above hi passes none (no read,
            // the comparator is out) — only codes inside (lo, hi] are looked
            // up.  Comparators from rows strictly below the item's in an
            // attribute's coarse bin never need that attribute's table.
            uint32_t ilo[D], ihi[D];
#pragma unroll
            for (int j = 0; j < D; ++j) {
                ilo[j] = min(min(sm.lo4[0][j], sm.lo4[1][j]), min(sm.lo4[2][j], sm.lo4[3][j]));
                ihi[j] = max(max(sm.hi4[0][j], sm.hi4[1][j]), max(sm.hi4[2][j], sm.hi4[3][j]));
            }
            for (;;) {
                mbar_wait(&sm.full[cs], cphase, 3);
                const uint32_t n = sm.nslot[cs];
                const bool fin = sm.last[cs] != 0u;
                // the alive masks change under the other consumer warps'
                // atomicAnd while this warp's lanes leave the wait one by one:
                // lane 0 reads them and broadcasts, so that the whole warp
                // takes the same branch around the warp-level votes below
                // (lanes reading for themselves could see "all dead" and
                // "one alive" in the same stage and wait for each other at
                // different warp barriers for ever)
                uint32_t al[4] = {0u, 0u, 0u, 0u};
                __syncwarp();
                if (lane == 0) {
                    const volatile uint32_t* av = sm.alive;
                    al[0] = av[0];
                    al[1] = av[1];
                    al[2] = av[2];
                    al[3] = av[3];
                }
#pragma unroll
                for (int w = 0; w < 4; ++w) al[w] = __shfl_sync(0xffffffffu, al[w], 0);
                if ((al[0] | al[1] | al[2] | al[3]) != 0u) {
                    if (cw == 0 && lane == 0) {
                        cnt += (unsigned long long)sm.nreal[cs] *
                               (__popc(al[0]) + __popc(al[1]) + __popc(al[2]) + __popc(al[3]));
                        ucnt += sm.nreal[cs];
                    }
                    uint2* hb = sm.hits[cw];
                    for (uint32_t s0 = cw * 32; s0 < n; s0 += 32 * kTCons) {
                        const uint32_t s = s0 + lane;
                        uint4 m = make_uint4(0u, 0u, 0u, 0u);
                        if (s < n) {
                            const W c = sm.ring[cs][s];
                            bool out = false;
#pragma unroll
                            for (int j = 0; j < D; ++j)
                                out |= ((uint32_t)(c >> (8 * j)) & 0xFFu) > ihi[j];
                            if (!out) {
                                m = make_uint4(al[0], al[1], al[2], al[3]);
#pragma unroll
                                for (int j = 0; j < D; ++j) {
                                    const uint32_t cj = (uint32_t)(c >> (8 * j)) & 0xFFu;
                                    if (cj > ilo[j]) {
                                        const uint4 e = sm.tab[j * kTabR + cj];
                                        m.x &= e.x;
                                        m.y &= e.y;
                                        m.z &= e.z;
                                        m.w &= e.w;
                                    }
                                }
                            }
                        }
                        const bool hit = (m.x | m.y | m.z | m.w) != 0u;
                        if (!__any_sync(0xffffffffu, hit)) continue;
                        // code passes (rare): the exact float64 + precedence
                        // test, the warp's (comparator, candidate) pairs
                        // gathered and tested one per lane
                        uint32_t qs = 0, nb = 0;
                        if (hit) {
                            uint32_t pi = 0;
                            const uint32_t npc = sm.npiece[cs];
                            while (pi + 1 < npc && sm.pslot[cs][pi + 1] <= s) ++pi;
                            qs = sm.ppos[cs][pi] + (s - sm.pslot[cs][pi]);
                            nb = __popc(m.x) + __popc(m.y) + __popc(m.z) + __popc(m.w);
                        }
                        uint32_t incl = nb;
#pragma unroll
                        for (int o = 1; o < 32; o <<= 1) {
                            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                            if ((int)lane >= o) incl += y;
                        }
                        const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
                        const uint32_t mw[4] = {m.x, m.y, m.z, m.w};
                        if (total <= (uint32_t)kHitCap) {
                            uint32_t at = incl - nb;
#pragma unroll
                            for (int w = 0; w < 4; ++w) {
                                uint32_t b = mw[w];
                                while (b) {
                                    const uint32_t i = (uint32_t)__ffs(b) - 1u;
                                    b &= b - 1;
                                    hb[at++] = make_uint2(qs, 32u * w + i);
                                }
                            }
                            __syncwarp();
                            for (uint32_t h = lane; h < total; h += 32) {
                                const uint2 pr = hb[h];
                                if (exact_rec<D>(rec, ids, R, sidx, pr.x, first + pr.y))
                                    atomicAnd(&sm.alive[pr.y >> 5], ~(1u << (pr.y & 31u)));
                            }
                            __syncwarp();
                        } else {
#pragma unroll
                            for (int w = 0; w < 4; ++w) {
                                uint32_t b = mw[w];
                                while (b) {
                                    const int i = __ffs(b) - 1;
                                    b &= b - 1;
                                    if (exact_rec<D>(rec, ids, R, sidx, qs,
                                                     first + 32 * w + (uint32_t)i))
                                        atomicAnd(&sm.alive[w], ~(1u << i));
                                }
                            }
                        }
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&sm.empty[cs]);
                if (++cs == kStages) {
                    cs = 0;
                    cphase ^= 1u;
                }
                if (fin) break;
            }
        }
        __syncthreads();
        {
            const uint32_t q = first + threadIdx.x;
            if (q < end) keep[sidx[q]] = (uint8_t)((sm.alive[warp] >> lane) & 1u);
        }
    }
    add_count(tests, cnt);
    add_count(tests + (S_UNITS_SKY - S_TESTS_SKY), ucnt);
}

template <int D, class F>
void with_d(int d, F&& f) {
    if (d == D) f(std::integral_constant<int, D>{});
    if constexpr (D < 8) with_d<D + 1>(d, f);
}

double env_or(const char* name, double dflt) {
    const char* e = getenv(name);
    const double x = e ? atof(e) : 0.0;
    return x > 0 ? x : dflt;
}

struct GridShape {
    int k0 = 0, k = 0;
    uint32_t rows = 0, ncells = 0;
};

// bins: k coarse bins on attributes 1..d-1 so that a row holds ~512 tuples
// (SKYGPU_GRID_ROW), k0 fine bins on attribute 0 (SKYGPU_GRID_K0, <= 128)
GridShape grid_shape(uint64_t r, int d) {
    GridShape g;
    if (d < 1 || d > 8) return g;
    static const double per_row = env_or("SKYGPU_GRID_ROW", 512.0);
    static const int k0 = (int)std::min(128.0, env_or("SKYGPU_GRID_K0", 64.0));
    int k = 1;
    if (d > 1) {
        k = (int)std::lround(std::pow(std::max(1.0, (double)r / per_row), 1.0 / (d - 1)));
        k = std::max(2, std::min(k, 128));
        while (k > 2 && std::pow((double)k, d - 1) * k0 > (double)(1u << 22)) --k;
    }
    const double rows = std::pow((double)k, d - 1);
    if (rows * k0 > (double)(1u << 22)) return g;
    g.k0 = k0;
    g.k = k;
    g.rows = (uint32_t)rows;
    g.ncells = g.rows * (uint32_t)k0;
    return g;
}

}  // namespace

int sky_grid_bins(uint64_t r, int d) { return grid_shape(r, d).k0; }

void sky_grid_decide(Ctx& c, const double* d_vals, int d, const unsigned long long* keys,
                     const int64_t* d_ids, const uint32_t* R, uint64_t r, uint8_t* keep,
                     double* kernel_ms, int shard_rank, int shard_world) {
    const GridShape g = grid_shape(r, d);
    if (shard_world > 1)  // tuples of rows other shards own stay 0 until the MAX reduce
        SKY_CUDA(cudaMemsetAsync(keep, 0, r, c.stream));
    if (!g.k0) throw Error(SKYGPU_ERUNTIME, "sky_grid_decide: unsupported shape (internal)");
    const uint32_t ncells = g.ncells;
    double* bounds = c.buf[B_PROJ].as<double>(8 * 128 + (sizeof(RankTable) + 7) / 8);
    RankTable* rtab = reinterpret_cast<RankTable*>(bounds + 8 * 128);
    const uint64_t cwords = 2 * ((uint64_t)ncells + 1) + 2;
    uint32_t* count = c.buf[B_GCNT].as<uint32_t>(cwords);
    uint32_t* seg = count + ncells + 1;
    unsigned* ctr = (unsigned*)(seg + ncells + 1);
    static const bool atomic_bucket = [] {  // see the bucketing below
        const char* e = getenv("SKYGPU_GRID_SORT");
        return !(e && e[0] == '1');
    }();
    if (atomic_bucket)
        SKY_CUDA(cudaMemsetAsync(count, 0, sizeof(uint32_t) * cwords, c.stream));
    else  // (seg is written whole by k_seg_bounds; only the item counters)
        SKY_CUDA(cudaMemsetAsync(ctr, 0, sizeof(unsigned) * 2, c.stream));
    pdl_launch(k_rank_bounds, d, 1024, 0, c.stream, d_vals, d, R, r, bounds, rtab);
    SKY_LAUNCH_CHECK();
    note_launch(c);
    trace_mark(c, "grid: bounds");
    with_d<1>(d, [&](auto DC) {
        constexpr int D = decltype(DC)::value;
        using W = GridWord<D>;
        W* code = c.buf[B_GCODE].as<W>(r);
        uint32_t* cell = c.buf[B_GCELL].as<uint32_t>(r);
        // (+ 16 bytes of never-passing codes: the bulk copies of the TMA
        // decide kernel round the last range up to 16 bytes)
        W* scode = c.buf[B_GSCODE].as<W>(r + 16 / sizeof(W));
        SKY_CUDA(cudaMemsetAsync(scode + r, 0x80, 16, c.stream));
        uint32_t* sidx = c.buf[B_GSIDX].as<uint32_t>(r);
        uint2* items = c.buf[B_GITEMS].as<uint2>(r / kItem + g.rows + 1);
        // bucketing by cell: a histogram + scan + atomic scatter (default),
        // or a stable radix sort of the cell ids (SKYGPU_GRID_SORT=1:
        // deterministic order inside a cell, measured 0.15 ms slower on C5)
        // K6: the TMA-staged bitset kernel (default) or the per-lane ALU
        // kernel (SKYGPU_GRID_KERNEL=alu, kept for A/B measurement)
        static const bool alu = [] {
            const char* e = getenv("SKYGPU_GRID_KERNEL");
            return e && e[0] == 'a';
        }();
        double* rec = alu ? nullptr : c.buf[B_GREC].as<double>(r * (D + 1));
        if (atomic_bucket) {
            pdl_launch(k_rank_codes<D>, grid_for(r, kGB, c.num_sms * 8), kGB, 0, c.stream,
                d_vals, R, (uint32_t)r, (const RankTable*)rtab, g.k0, g.k, code, cell, count,
                (uint32_t*)nullptr);
            SKY_LAUNCH_CHECK();
            size_t tmp = 0;
            SKY_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, count, seg, (int)ncells + 1,
                                                   c.stream));
            void* t = c.buf[B_CUB].get(tmp);
            SKY_CUDA(cub::DeviceScan::ExclusiveSum(t, tmp, count, seg, (int)ncells + 1, c.stream));
            SKY_CUDA(cudaMemsetAsync(count, 0, sizeof(uint32_t) * ncells, c.stream));  // cursors
            // (SKYGPU_GRID_RECSCATTER=0: scatter, then gather the records — C5
            // skyline stage 8.03 ms against 7.85 ms fused)
            static const bool rec_scatter = [] {
                const char* e = getenv("SKYGPU_GRID_RECSCATTER");
                return !(e && e[0] == '0');
            }();
            if (rec && rec_scatter) {
                pdl_launch(k_cell_scatter_rec<D>, grid_for(r, kGB), kGB, 0, c.stream,
                           (const W*)code, (const uint32_t*)cell, (uint32_t)r,
                           (const uint32_t*)seg, count, scode, sidx, d_vals, R, rec);
            } else {
                pdl_launch(k_cell_scatter<W>, grid_for(r, kGB), kGB, 0, c.stream, code, cell,
                           (uint32_t)r, seg, count, scode, sidx);
                if (rec)
                    pdl_launch(k_gather_rec<D>, grid_for(r, kGB), kGB, 0, c.stream, sidx,
                               (uint32_t)r, d_vals, keys, R, rec, (const W*)nullptr, (W*)nullptr);
            }
            SKY_LAUNCH_CHECK();
        } else {
            uint32_t* iota = c.buf[B_GIOTA].as<uint32_t>(r);
            uint32_t* skey = c.buf[B_GSKEY].as<uint32_t>(r);
            pdl_launch(k_rank_codes<D>, grid_for(r, kGB, c.num_sms * 8), kGB, 0, c.stream,
                d_vals, R, (uint32_t)r, (const RankTable*)rtab, g.k0, g.k, code, cell, count, iota);
            SKY_LAUNCH_CHECK();
            cub::DoubleBuffer<uint32_t> kb(cell, skey), vb(iota, sidx);
            const int end_bit = std::max(1, 32 - __builtin_clz(ncells));
            size_t tmp = 0;
            SKY_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, kb, vb, (int64_t)r, 0, end_bit,
                                                     c.stream));
            void* t = c.buf[B_CUB].get(tmp);
            SKY_CUDA(cub::DeviceRadixSort::SortPairs(t, tmp, kb, vb, (int64_t)r, 0, end_bit,
                                                     c.stream));
            if (vb.Current() != sidx)
                SKY_CUDA(cudaMemcpyAsync(sidx, vb.Current(), sizeof(uint32_t) * r,
                                         cudaMemcpyDeviceToDevice, c.stream));
            pdl_launch(k_seg_bounds, grid_for((uint64_t)r + 1, kGB), kGB, 0, c.stream,
                       (const uint32_t*)kb.Current(), (uint32_t)r, ncells, seg);
            if (rec)
                pdl_launch(k_gather_rec<D>, grid_for(r, kGB), kGB, 0, c.stream, sidx, (uint32_t)r,
                           d_vals, keys, R, rec, (const W*)code, scode);
            else
                pdl_launch(k_gather_codes<W>, grid_for(r, kGB), kGB, 0, c.stream, sidx,
                           (uint32_t)r, (const W*)code, scode);
            SKY_LAUNCH_CHECK();
        }
        pdl_launch(k_row_items, grid_for(g.rows, kGB), kGB, 0, c.stream, seg, g.rows, g.k0, items,
                   ctr,
                                                                 shard_rank, shard_world);
        SKY_LAUNCH_CHECK();
        note_launch(c, 5);
        trace_mark(c, "grid: codes + cells + items");
        int per_sm = 0;
        if (alu)
            SKY_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_grid_decide<D>, kGB, 0));
        else
            SKY_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_grid_decide_tma<D>,
                                                                   kTB, 0));
        per_sm = std::max(1, per_sm);
        SKY_CUDA(cudaEventRecord(c.ev[14], c.stream));
        issue_late_ids(c);  // (deferred host ids: their copy overlaps K6)
        if (alu)
            pdl_launch(k_grid_decide<D>, c.num_sms * per_sm, kGB, 0, c.stream,
                d_vals, keys, d_ids, R, scode, sidx, seg, items, ctr, g.k0, g.k, keep,
                c.d_slots + S_TESTS_SKY);
        else
            pdl_launch(k_grid_decide_tma<D>, c.num_sms * per_sm, kTB, 0, c.stream,
                (const double*)rec, d_ids, R, scode, sidx, seg, items, ctr, g.k0, g.k, keep,
                c.d_slots + S_TESTS_SKY);
        SKY_LAUNCH_CHECK();
        SKY_CUDA(cudaEventRecord(c.ev[15], c.stream));
        note_launch(c);
        trace_mark(c, "grid: K6 decide kernel");
    });
    if (kernel_ms) {
        SKY_CUDA(cudaEventSynchronize(c.ev[15]));
        float ms = 0;
        SKY_CUDA(cudaEventElapsedTime(&ms, c.ev[14], c.ev[15]));
        *kernel_ms += ms;
    }
}

}  // namespace skygpu
