// skyline.cu — the skyline stage on sm_100a (north_star (a)).
//
// Reference: parallel_skyline (proj/src/parallel.cpp:22-101) runs a local
// sort-filter skyline per partition and one SFS merge (core.cpp:48-73).  Its
// result is the PREDECESSOR RULE: tuple t is kept iff no tuple strictly
// before t in (sum, id) order dominates it (sum = left-to-right float64
// accumulate from 0.0, core.cpp:21-23).  Proof: an SFS window
// only holds kept tuples, and a dropped dominator is itself dominated by an
// earlier kept one (transitivity), for every plan and every partition order.
// This equals the skyline except in the FP-tie case of SURVEY.md §7.4 item 1,
// where it reproduces parallel_skyline (not skyline_bruteforce) exactly.
//
// GPU algorithm — prefix rounds, no sort of the relation:
//   K1 score     left-to-right __dadd_rn sum -> order-preserving key bits,
//                contract checks (one HBM pass over the relation)
//   K2 sample    one CTA sorts a strided sample of the undecided keys ->
//                threshold T with about k keys below it.  {key < T} is a
//                PREFIX of the (sum, id) order: every predecessor of a prefix
//                member is in the prefix, so the prefix can be decided alone.
//   K3 select    the prefix (order-preserving compaction)
//   K3b sort     the prefix by (sum, id): key-bucket counting sort + in-bucket
//                rank (two short launches, k <= 16384)
//   K4 intra     warp-per-candidate: each prefix member against its
//                predecessors in sum order (strongest first), warp-ballot
//                exit at the first dominator -> new skyline tuples A', already
//                in the reference's output order
//   K5 filter    every other undecided tuple against A' regrouped by
//                direction cell (own cell first, coalesced float64 SoA loads,
//                ballot exit); survivors are the next round's undecided set.
// The lowest-sum tuples are the strongest dominators: one round of k ~ 12k
// leaves ~10^3 survivors out of 10^6 on the benchmark data; large skylines
// (ANT d=7) grow k up to 65536 per round.  The direction cells are the GPU
// recast of the paper's angular partitioning: they only decide the SCAN
// ORDER (how fast a dominator is met), never the result.
#include <cub/cub.cuh>

#include "sky_common.cuh"

namespace skygpu {

namespace {

constexpr int kBlock = 256;
constexpr int kCTAItems = 16;
constexpr uint32_t kCTACap = 1024 * kCTAItems;  // single-CTA helpers up to 16384 items
constexpr uint32_t kMaxCells = 4096;

// in-place exclusive scan of a 4096-entry shared-memory table by a
// 1024-thread block (4 entries per thread); returns the total
__device__ __forceinline__ uint32_t block_exclusive_scan_4096(uint32_t* tab) {
    using Scan = cub::BlockScan<uint32_t, 1024>;
    __shared__ typename Scan::TempStorage tmp;
    uint32_t x[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) x[j] = tab[threadIdx.x * 4 + j];
    uint32_t total = 0;
    Scan(tmp).ExclusiveSum(x, x, total);
#pragma unroll
    for (int j = 0; j < 4; ++j) tab[threadIdx.x * 4 + j] = x[j];
    __syncthreads();
    return total;
}

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

// K1 (core.cpp:21-23): sum with __dadd_rn from +0.0, key = ord bits (sums
// are never -0.0: 0.0 + -0.0 = +0.0), value contract (Relation::add), key
// range, and (D in 1..8) the per-attribute maxima that scale the 16-bit
// quantised codes of the dominance prefilter.
template <int D>
__global__ void k_score(const double* __restrict__ v, uint64_t n, int d,
                        unsigned long long* __restrict__ key,
                        unsigned long long* __restrict__ slots,
                        unsigned long long* __restrict__ amax, uint64_t base = 0,
                        const int64_t* __restrict__ ids = nullptr,
                        uint32_t* __restrict__ prefix = nullptr) {
    pdl_wait();
    constexpr int DA = D > 0 ? D : 1;
    unsigned long long mn = ~0ULL, mx = 0;
    unsigned long long am[DA];
#pragma unroll
    for (int k = 0; k < DA; ++k) am[k] = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        bool bad = false;
        if (D > 0) {
#pragma unroll
            for (int k = 0; k < DA; ++k) {
                const double x = v[i * DA + k];
                bad |= !(x >= 0.0);  // negative or NaN
                s = __dadd_rn(s, x);
                const unsigned long long xb = ord_bits(x);
                am[k] = xb > am[k] ? xb : am[k];
            }
        } else {
            for (int k = 0; k < d; ++k) {
                const double x = v[i * d + k];
                bad |= !(x >= 0.0);
                s = __dadd_rn(s, x);
            }
        }
        const unsigned long long b = ord_bits(s);
        key[i] = b;
        if (prefix) {  // the first round's prefix {key < T} appended (unordered:
            // the prefix sort orders it fully by (sum, id, position))
            const bool in = b < slots[S_THR];
            const unsigned am_ = __activemask();
            const unsigned bal = __ballot_sync(am_, in);
            if (bal) {
                const int lane = threadIdx.x & 31, leader = __ffs(bal) - 1;
                unsigned long long at = 0;
                if (lane == leader) at = atomicAdd(&slots[S_C1], (unsigned long long)__popc(bal));
                at = __shfl_sync(am_, at, leader);
                if (in) prefix[at + __popc(bal & ((1u << lane) - 1u))] = (uint32_t)i;
            }
        }
        mn = b < mn && b > 0 ? b : mn;  // min POSITIVE key (zero sums: bucket 0 below)
        mx = b > mx ? b : mx;
        if (bad) atomicMin(&slots[S_BAD], static_cast<unsigned long long>(base + i));
        if (ids && i + 1 < n && ids[i] >= ids[i + 1]) atomicOr(&slots[S_FLAG], 1ULL);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long x = __shfl_down_sync(0xffffffffu, mn, o);
        const unsigned long long y = __shfl_down_sync(0xffffffffu, mx, o);
        mn = x < mn ? x : mn;
        mx = y > mx ? y : mx;
#pragma unroll
        for (int k = 0; k < DA; ++k) {
            const unsigned long long z = __shfl_down_sync(0xffffffffu, am[k], o);
            am[k] = z > am[k] ? z : am[k];
        }
    }
    // block-level combine first: one set of atomics per block, not per warp
    __shared__ unsigned long long s_mn[32], s_mx[32], s_am[32][DA];
    const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        s_mn[warp] = mn;
        s_mx[warp] = mx;
#pragma unroll
        for (int k = 0; k < DA; ++k) s_am[warp][k] = am[k];
    }
    __syncthreads();
    if (threadIdx.x == 0) {  // key range of the relation, per-attribute maxima
        for (int w = 1; w < nw; ++w) {
            mn = s_mn[w] < mn ? s_mn[w] : mn;
            mx = s_mx[w] > mx ? s_mx[w] : mx;
#pragma unroll
            for (int k = 0; k < DA; ++k) am[k] = s_am[w][k] > am[k] ? s_am[w][k] : am[k];
        }
        atomicMin(&slots[S_SMIN], mn);
        atomicMax(&slots[S_SMAX], mx);
        if (D > 0)
#pragma unroll
            for (int k = 0; k < DA; ++k) atomicMax(&amax[k], am[k]);
    }
}

// ---- 16-bit quantised codes: an exact-safe prefilter for float64 dominance.
// q_j(x) = min(floor(x * 32767 / max_j), 32767) is monotone in x, so
// s_j <= t_j implies q_j(s) <= q_j(t): if any q_j(s) > q_j(t), s cannot
// dominate t (exact reject).  Only pairs that pass (true dominators and rare
// near-ties) take the float64 test.  Four 16-bit fields per u64 word (bit 15
// of each field is the SWAR guard): ((qt | H) - qs) & H == H  <=>  all
// fields qs <= qt.  D <= 4: one word, D <= 8: two.
constexpr unsigned long long kH16 = 0x8000800080008000ULL;

template <int D>
struct QW {
    static constexpr int W = D <= 4 ? 1 : 2;
};

template <int D>
__device__ __forceinline__ void load_scales(const unsigned long long* __restrict__ amax,
                                            double (&sc)[D]) {
#pragma unroll
    for (int k = 0; k < D; ++k) {
        const double m = __longlong_as_double((long long)amax[k]);
        sc[k] = m > 0.0 ? __ddiv_rn(32767.0, m) : 0.0;
    }
}

template <int D>
__device__ __forceinline__ void encode16(const double (&t)[D], const double (&sc)[D],
                                         unsigned long long (&w)[QW<D>::W]) {
#pragma unroll
    for (int k = 0; k < QW<D>::W; ++k) w[k] = 0;
#pragma unroll
    for (int k = 0; k < D; ++k) {
        double q = floor(__dmul_rn(t[k], sc[k]));
        q = q < 32767.0 ? q : 32767.0;
        w[k / 4] |= (unsigned long long)(unsigned)q << (16 * (k % 4));
    }
}

template <int D>
__device__ __forceinline__ bool le16(const unsigned long long* __restrict__ cs,
                                     const unsigned long long (&tg)[QW<D>::W]) {
    bool ok = true;
#pragma unroll
    for (int k = 0; k < QW<D>::W; ++k) ok &= ((tg[k] - cs[k]) & kH16) == kH16;
    return ok;
}

// compact SoA float64 copy [D][cap] plus quantised codes [cap][W] of the
// tuples list[0..count) (count from device when given), one thread per tuple
template <int D>
__global__ void k_gather_q(const double* __restrict__ v, const uint32_t* __restrict__ list,
                           uint64_t cap, const unsigned long long* __restrict__ count,
                           const unsigned long long* __restrict__ amax, double* __restrict__ out,
                           unsigned long long* __restrict__ qout) {
    pdl_wait();
    const uint64_t mm = count ? *count : cap;
    if (mm > cap) return;  // (a speculative count above the capacity: no-op)
    double sc[D];
    load_scales<D>(amax, sc);
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < mm;
         k += (uint64_t)gridDim.x * blockDim.x) {
        double t[D];
        const uint64_t p = list[k];
#pragma unroll
        for (int a = 0; a < D; ++a) {
            t[a] = v[p * D + a];
            out[(uint64_t)a * cap + k] = t[a];
        }
        unsigned long long w[QW<D>::W];
        encode16<D>(t, sc, w);
#pragma unroll
        for (int a = 0; a < QW<D>::W; ++a) qout[k * QW<D>::W + a] = w[a];
    }
}

__global__ void k_ids_check(const int64_t* __restrict__ ids, uint64_t n,
                            unsigned long long* __restrict__ slots, int slot = S_FLAG) {
    pdl_wait();
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i + 1 < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        if (ids[i] >= ids[i + 1]) atomicOr(&slots[slot], 1ULL);
}

// Grid strategy contract (partition.cpp:88-95): values must lie in [0,1];
// the first offending (tuple, attribute) in input order is reported.
__global__ void k_grid_range(const double* __restrict__ v, uint64_t total,
                             unsigned long long* __restrict__ slots) {
    pdl_wait();
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
         i += (uint64_t)gridDim.x * blockDim.x) {
        double x = v[i];
        if (x < 0.0 || x > 1.0) atomicMin(&slots[S_GRIDBAD], static_cast<unsigned long long>(i));
    }
}

// K2: threshold key T with about `want` undecided keys below it.  One block
// sorts a strided sample of 4096 keys; T = (q-th sample) + 1 for
// q = want * 4096 / r, so at least that sample is selected (progress).  The
// keys are order-preserving bits of the sums, so {key < T} is a prefix of
// the (sum, id) order.  want >= r takes everything.
constexpr int kSampleItems = 4;
__global__ void __launch_bounds__(1024)
k_sample_threshold(const unsigned long long* __restrict__ key, const uint32_t* __restrict__ R,
                   uint64_t r, uint64_t want, unsigned long long* __restrict__ slots,
                   const double* __restrict__ v, int d) {
    pdl_wait();
    // An approximate quantile suffices (T is exact once chosen): the samples
    // are bucketed linearly between their min and max sum and the bucket
    // holding the q-th sample gives T — one histogram, no sort.
    using Scan = cub::BlockScan<uint32_t, 1024>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ uint32_t hist[1024];
    __shared__ unsigned long long smin, smax;
    constexpr uint64_t NS = 1024 * kSampleItems;
    if (want >= r) {
        if (threadIdx.x == 0) slots[S_THR] = ~0ULL;
        return;
    }
    hist[threadIdx.x] = 0;
    if (threadIdx.x == 0) smin = ~0ULL, smax = 0;
    __syncthreads();
    unsigned long long items[kSampleItems];
    unsigned long long mn = ~0ULL, mx = 0;
#pragma unroll
    for (int j = 0; j < kSampleItems; ++j) {
        const uint64_t s = threadIdx.x * kSampleItems + j;
        const uint64_t pos = s * r / NS;
        const uint32_t t = R ? R[pos] : (uint32_t)pos;
        if (v) {  // (before the keys exist: the sampled tuple's sum, K1's order)
            double sum = 0.0;
            for (int a = 0; a < d; ++a) sum = __dadd_rn(sum, v[(uint64_t)t * d + a]);
            items[j] = ord_bits(sum);
        } else {
            items[j] = key[t];
        }
        mn = items[j] < mn ? items[j] : mn;
        mx = items[j] > mx ? items[j] : mx;
    }
    atomicMin(&smin, mn);
    atomicMax(&smax, mx);
    __syncthreads();
    const double lo = __longlong_as_double((long long)smin);
    const double hi = __longlong_as_double((long long)smax);
    const double scale = hi > lo ? 1024.0 / (hi - lo) : 0.0;
#pragma unroll
    for (int j = 0; j < kSampleItems; ++j) {
        int b = (int)((__longlong_as_double((long long)items[j]) - lo) * scale);
        b = b < 0 ? 0 : (b > 1023 ? 1023 : b);
        atomicAdd(&hist[b], 1u);
    }
    __syncthreads();
    uint32_t incl = 0;
    Scan(tmp).InclusiveSum(hist[threadIdx.x], incl);
    const uint64_t q = want * NS / r + 1;  // samples wanted below T
    const uint32_t prev = incl - hist[threadIdx.x];
    if (prev < q && incl >= q) {  // exactly one thread: the bucket holding the q-th sample
        const double bound = lo + (double)(threadIdx.x + 1) / scale;
        unsigned long long T = threadIdx.x == 1023 || !(scale > 0.0) ? smax + 1 : ord_bits(bound);
        if (T <= smin) T = smin + 1;  // progress: the smallest sample is always selected
        slots[S_THR] = T;
    }
}

// K3 predicate: the prefix {key < T} of the undecided set
struct BelowThreshold {
    const unsigned long long* key;
    const unsigned long long* thr;
    __device__ __forceinline__ bool operator()(uint32_t t) const { return key[t] < *thr; }
};

// Scan-order cells.  The reference partitions the relation (grid, angular,
// sliced — partition.cpp:85-213) so that each local SFS sees nearby tuples;
// here the plan's partition of a tuple decides which comparators its scan
// visits FIRST (own partition, then the rest), never the result.  A cell
// spec packs (kind << 16 | m):
//   kind 0  direction cells: grid over u_j = t_j / sum(t), j < d-1, m bins
//   kind 1  Grid plan: the reference's grid cell (partition.cpp:85-109), m slices
//   kind 2  Angular plan: the reference's hyperspherical angles
//           (partition.cpp:139-174), m slices per angle
//   kind 3  Sliced plan: m slices of attribute 0 (equi-width over its range;
//           the reference's exact equi-depth ranks only change the order)
enum CellKind {
    kCellDirection = 0,
    kCellGrid = 1,
    kCellAngular = 2,
    kCellSliced = 3,
    kCellQuantile = 4  // quantile grid over the raw attributes (qgrid_cell)
};

// Direction cell of a tuple: a grid over its first d-1 normalised
// coordinates u_j = t_j / sum(t).  A dominator s of t lies in the orthant
// below t; on large-skyline data (tuples near a hyperplane) that means a
// nearby direction, so scanning t's own cell first finds it early.
template <int DM>
__device__ __forceinline__ uint32_t direction_cell(const double* t, int dd, int m) {
    if (dd < 2 || m <= 1) return 0;
    double s = 0.0;
    for (int k = 0; k < DM; ++k)
        if (k < dd) s += t[k];
    if (!(s > 0.0)) return 0;
    const float inv = (float)m / (float)s;  // (scan order only: float32 suffices)
    uint32_t cell = 0;
    for (int k = DM - 2; k >= 0; --k) {
        if (k >= dd - 1) continue;
        int b = (int)((float)t[k] * inv);
        b = b < 0 ? 0 : (b >= m ? m - 1 : b);
        cell = cell * (uint32_t)m + (uint32_t)b;
    }
    return cell;
}

// grid cell index, partition.cpp:85-109 (values validated in [0,1])
template <int DM>
__device__ __forceinline__ uint32_t grid_cell_id(const double* t, int dd, int m) {
    uint32_t id = 0, w = 1;
    for (int k = 0; k < DM; ++k) {
        if (k >= dd) break;
        int b = (int)(t[k] * m);
        b = b < 0 ? 0 : (b >= m ? m - 1 : b);
        id += (uint32_t)b * w;
        w *= (uint32_t)m;
    }
    return id;
}

// angular partition id, partition.cpp:139-174 (all-zero tuple -> 0)
template <int DM>
__device__ __forceinline__ uint32_t angular_cell_id(const double* t, int dd, int m) {
    // (K5 scan order only — never a partition id the results depend on — so
    // float32 and the SFU: atan2/sqrt in float64 cost ~100 instructions per
    // candidate)
    bool zero = true;
    for (int k = 0; k < DM; ++k)
        if (k < dd) zero &= (t[k] == 0.0);
    if (zero || dd < 2) return 0;
    float tail[DM + 1];
    tail[dd] = 0.0f;
    for (int k = DM - 1; k >= 0; --k)
        if (k < dd) {
            const float x = (float)t[k];
            tail[k] = tail[k + 1] + x * x;
        }
    uint32_t id = 0, w = 1;
    for (int k = 0; k < DM - 1; ++k) {
        if (k >= dd - 1) break;
        const float angle = atan2f(sqrtf(tail[k + 1]), (float)t[k]);
        int b = (int)(angle * (0.63661977236758134f * (float)m));
        b = b < 0 ? 0 : (b >= m ? m - 1 : b);
        id += (uint32_t)b * w;
        w *= (uint32_t)m;
    }
    return id;
}

// Quantile grid over the raw attributes (kind 4, the default scan index of
// the filter): k bins per attribute, bounds = quantiles of the round's new
// skyline tuples A', held in constant memory.  bin_j(t) = #bounds <= t_j is
// monotone, so a tuple in a cell with bin_j above t's has its attribute j at
// or above a bound that exceeds t_j.
constexpr int kQMaxBins = 16;
__constant__ double c_qbounds[kMaxDims * kQMaxBins];

template <int DM>
__device__ __forceinline__ uint32_t qgrid_cell(const double* t, int dd, int k) {
    uint32_t id = 0, w = 1;
    for (int j = 0; j < DM; ++j) {
        if (j >= dd) break;
        uint32_t b = 0;
        for (int i = 0; i < k - 1; ++i) b += t[j] >= c_qbounds[j * kQMaxBins + i] ? 1u : 0u;
        id += b * w;
        w *= (uint32_t)k;
    }
    return id;
}

// bounds[j][i] = the (i+1)/k quantile of attribute j over list[0..*count)
// (4096 strided samples, one CTA per attribute)
__global__ void __launch_bounds__(1024)
k_qgrid_bounds(const double* __restrict__ v, int d, const uint32_t* __restrict__ list,
               const unsigned long long* __restrict__ count, int k, double* __restrict__ bounds) {
    pdl_wait();
    using Sort = cub::BlockRadixSort<unsigned long long, 1024, 4>;
    __shared__ typename Sort::TempStorage tmp;
    const int j = blockIdx.x;
    const uint64_t m = *count;
    unsigned long long items[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const uint64_t s = threadIdx.x * 4 + u;
        items[u] = m ? ord_bits(v[(uint64_t)list[s * m / 4096] * d + j]) : 0ULL;
    }
    Sort(tmp).Sort(items);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const uint32_t rank = threadIdx.x * 4 + u;
        for (int i = 1; i < k; ++i)
            if (rank == (uint32_t)(i * 4096 / k))
                bounds[j * kQMaxBins + i - 1] = __longlong_as_double((long long)items[u]);
    }
}

template <int DM>
__device__ __forceinline__ uint32_t plan_cell(const double* t, int dd, int spec,
                                              const unsigned long long* __restrict__ amax) {
    const int kind = spec >> 16, m = spec & 0xFFFF;
    switch (kind) {
        case kCellGrid: return grid_cell_id<DM>(t, dd, m);
        case kCellQuantile: return qgrid_cell<DM>(t, dd, m);
        case kCellAngular: return angular_cell_id<DM>(t, dd, m);
        case kCellSliced: {
            const double mx = amax ? __longlong_as_double((long long)amax[0]) : 1.0;
            int b = mx > 0.0 ? (int)(t[0] / mx * m) : 0;
            return (uint32_t)(b < 0 ? 0 : (b >= m ? m - 1 : b));
        }
        default: return direction_cell<DM>(t, dd, m);
    }
}

// Grid plan pre-merge pruning (parallel.cpp:32-42, partition.cpp:115-137): a
// cell strictly above a non-empty cell in every dimension holds no skyline
// tuple (each of its tuples is strictly dominated by — and so preceded by —
// any tuple of the lower cell).  Occupancy over the m^d cells, an inclusive
// prefix-OR along every dimension, then cell c is pruned iff the prefix-OR at
// c - (1,..,1) is set.
__global__ void k_grid_occ(const double* __restrict__ v, uint64_t n, int d, int m,
                           uint8_t* __restrict__ occ) {
    pdl_wait();
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        occ[grid_cell_id<kMaxDims>(v + i * d, d, m)] = 1;
}

__global__ void k_prefix_or_dim(uint8_t* __restrict__ occ, uint32_t ncells, int m,
                                uint32_t stride) {
    pdl_wait();
    const uint32_t lines = ncells / m;
    for (uint32_t l = blockIdx.x * blockDim.x + threadIdx.x; l < lines; l += gridDim.x * blockDim.x) {
        const uint32_t lo = l % stride, hi = l / stride;
        const uint32_t base = hi * stride * m + lo;
        uint8_t acc = 0;
        for (int k = 0; k < m; ++k) {
            acc |= occ[base + (uint32_t)k * stride];
            occ[base + (uint32_t)k * stride] = acc;
        }
    }
}

__global__ void k_grid_keep(const double* __restrict__ v, uint64_t n, int d, int m,
                            const uint8_t* __restrict__ P, uint8_t* __restrict__ keep) {
    pdl_wait();
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const double* t = v + i * d;
        uint32_t low = 0, w = 1;
        bool inner = true;
        for (int k = 0; k < d; ++k) {
            int b = (int)(t[k] * m);
            b = b < 0 ? 0 : (b >= m ? m - 1 : b);
            inner &= b >= 1;
            low += (uint32_t)(b - 1) * w;
            w *= (uint32_t)m;
        }
        keep[i] = !(inner && P[low]);
    }
}

// K3b: cell of every prefix member, then a one-CTA counting sort by cell
// (m <= 16384): cell-ordered list + cell keys.  Order inside a cell is free.
template <int D>
__global__ void __launch_bounds__(1024)
k_cell_order(const double* __restrict__ v, int d, const uint32_t* __restrict__ in, uint32_t mcap,
             const unsigned long long* __restrict__ count, int mcell, uint32_t ncells,
             const unsigned long long* __restrict__ amax,
             uint32_t* __restrict__ out, uint32_t* __restrict__ out_cell,
             uint32_t* __restrict__ seg) {
    pdl_wait();
    constexpr int DM = D > 0 ? D : kMaxDims;
    const int dd = D > 0 ? D : d;
    const uint32_t m = count ? (uint32_t)*count : mcap;
    __shared__ uint32_t cnt[kMaxCells];
    for (uint32_t c = threadIdx.x; c < kMaxCells; c += 1024) cnt[c] = 0;
    __syncthreads();
    uint32_t cl[kCTAItems];
#pragma unroll
    for (int j = 0; j < kCTAItems; ++j) {
        const uint32_t i = threadIdx.x + j * 1024;
        cl[j] = 0;
        if (i < m) {
            double t[DM];
            const uint64_t p = in[i];
#pragma unroll
            for (int k = 0; k < DM; ++k)
                if (k < dd) t[k] = v[p * dd + k];
            cl[j] = plan_cell<DM>(t, dd, mcell, amax);
            atomicAdd(&cnt[cl[j]], 1u);
        }
    }
    __syncthreads();
    block_exclusive_scan_4096(cnt);
    if (seg) {  // segment table: seg[c] = first position of cell c, seg[ncells] = m
        for (uint32_t c = threadIdx.x; c < ncells; c += 1024) seg[c] = cnt[c];
        if (threadIdx.x == 0) seg[ncells] = m;
        __syncthreads();  // read cnt before the scatter below bumps it
    }
#pragma unroll
    for (int j = 0; j < kCTAItems; ++j) {
        const uint32_t i = threadIdx.x + j * 1024;
        if (i < m) {
            const uint32_t pos = atomicAdd(&cnt[cl[j]], 1u);
            out[pos] = in[i];
            out_cell[pos] = cl[j];
        }
    }
}

// The same regrouping over many CTAs (A' of a few thousand tuples: one CTA
// walking it serially was a latency chain): cell ids + a global histogram,
// one CTA's exclusive scan into the segment table (and the scatter cursors),
// an atomic scatter.  The order inside a cell is immaterial (K5's scan order
// only), so the scatter needs no stability.
template <int D>
__global__ void k_cell_hist(const double* __restrict__ v, int d, const uint32_t* __restrict__ in,
                            uint32_t mcap, const unsigned long long* __restrict__ count,
                            int mcell, const unsigned long long* __restrict__ amax,
                            uint32_t* __restrict__ cell_of, uint32_t* __restrict__ hist) {
    pdl_wait();
    constexpr int DM = D > 0 ? D : kMaxDims;
    const int dd = D > 0 ? D : d;
    const uint32_t m = count ? min((uint32_t)*count, mcap) : mcap;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
        double t[DM];
        const uint64_t p = in[i];
#pragma unroll
        for (int k = 0; k < DM; ++k)
            if (k < dd) t[k] = v[p * dd + k];
        const uint32_t cl = plan_cell<DM>(t, dd, mcell, amax);
        cell_of[i] = cl;
        atomicAdd(&hist[cl], 1u);
    }
}

__global__ void __launch_bounds__(1024)
k_cell_seg(uint32_t* __restrict__ hist, uint32_t ncells, const unsigned long long* __restrict__ count,
           uint32_t mcap, uint32_t* __restrict__ seg, uint32_t* __restrict__ cursor) {
    pdl_wait();
    __shared__ uint32_t cnt[kMaxCells];
    for (uint32_t c = threadIdx.x; c < kMaxCells; c += 1024) cnt[c] = c < ncells ? hist[c] : 0u;
    __syncthreads();
    block_exclusive_scan_4096(cnt);
    for (uint32_t c = threadIdx.x; c < ncells; c += 1024) {
        seg[c] = cnt[c];
        cursor[c] = cnt[c];
        hist[c] = 0;  // (ready for the next round)
    }
    if (threadIdx.x == 0) seg[ncells] = count ? min((uint32_t)*count, mcap) : mcap;
}

__global__ void k_cell_scatter_a(const uint32_t* __restrict__ in, uint32_t mcap,
                                 const unsigned long long* __restrict__ count,
                                 const uint32_t* __restrict__ cell_of, uint32_t* __restrict__ cursor,
                                 uint32_t* __restrict__ out) {
    pdl_wait();
    const uint32_t m = count ? min((uint32_t)*count, mcap) : mcap;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x)
        out[atomicAdd(&cursor[cell_of[i]], 1u)] = in[i];
}

// compact SoA copy [d][cap] of the tuples list[0..m) from the AoS input; the
// count is read from device memory when `count` is given (no host sync)
__global__ void k_gather_aos(const double* __restrict__ v, int d, const uint32_t* __restrict__ list,
                             uint64_t cap, const unsigned long long* __restrict__ count,
                             double* __restrict__ out) {
    pdl_wait();
    const uint64_t mm = count ? *count : cap;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < mm * d;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t k = i / d;
        const int a = (int)(i - k * d);
        out[(uint64_t)a * cap + k] = v[(uint64_t)list[k] * d + a];
    }
}

// Representative filter (partition.cpp:287-302): a tuple dominated by any
// representative never enters the local skylines.  reps: AoS [n_reps][d].
template <int D>
__global__ void k_rep_filter(const double* __restrict__ v, uint64_t n, int d,
                             const double* __restrict__ reps, uint32_t n_reps,
                             uint8_t* __restrict__ keep, unsigned long long* __restrict__ tests,
                             int and_mode) {
    pdl_wait();
    constexpr int DM = D > 0 ? D : kMaxDims;
    const int dd = D > 0 ? D : d;
    unsigned long long cnt = 0;
    for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < n;
         p += (uint64_t)gridDim.x * blockDim.x) {
        double t[DM];
#pragma unroll
        for (int k = 0; k < DM; ++k)
            if (k < dd) t[k] = v[p * dd + k];
        bool alive = true;
        for (uint32_t r = 0; r < n_reps && alive; ++r) {
            ++cnt;
            alive = !dom_f64_dyn(reps + (uint64_t)r * dd, t, dd);
        }
        keep[p] = and_mode ? (uint8_t)(keep[p] && alive) : (uint8_t)alive;
    }
    add_count(tests, cnt);
}

// (key, id) order of the predecessor rule; ids are unique
__device__ __forceinline__ bool precedes(unsigned long long ka, int64_t ia,
                                         unsigned long long kb, int64_t ib) {
    return ka < kb || (ka == kb && ia < ib);
}

// Exact sort of the prefix (m <= 16384) by (key, id, position) in two short
// launches, no device radix sort:
//  1. one CTA buckets the prefix by the high bits of (key - kmin) into 4096
//     monotone key buckets (shared-memory counting sort), so every bucket
//     precedes the next in (sum, id) order;
//  2. every element ranks itself inside its (small) bucket and scatters to
//     bucket_start + rank.
constexpr uint32_t kKeyBuckets = 4096;

// bucket parameters of the prefix sort computed on the device from the
// round's slots (a round sized on the device: the host has not read them):
// kmin = min key; keys up to the threshold - 1 (or the max key) spread over
// 4096 buckets — the host's formula in decide_prefix
// monotone key -> bucket map: keys below kmin (the zero sums; kmin is the
// smallest POSITIVE key) share bucket 0, the rest spread linearly over the
// raw bits from kmin — a zero sum no longer stretches the span (C3: 149 zero
// tuples once crowded the whole prefix into a couple of buckets)
__device__ __forceinline__ uint32_t key_bucket(unsigned long long key, unsigned long long kmin,
                                               int shift) {
    if (key < kmin) return 0;
    const unsigned long long x = ((key - kmin) >> shift) + 1;
    return x < kKeyBuckets ? (uint32_t)x : kKeyBuckets - 1;
}

__device__ __forceinline__ void bucket_params_dev(const unsigned long long* __restrict__ slots,
                                                  int use_thr, unsigned long long& kmin,
                                                  int& shift) {
    const unsigned long long gmin = slots[S_SMIN] == ~0ULL ? 0 : slots[S_SMIN];
    const unsigned long long thr = use_thr ? slots[S_THR] : ~0ULL, gmax = slots[S_SMAX];
    const unsigned long long top = thr == ~0ULL || thr - 1 > gmax ? gmax : thr - 1;
    const unsigned long long span = top > gmin ? top - gmin : 0;
    const int bits = span ? 64 - __clzll((long long)span) : 0;
    kmin = gmin;
    shift = bits > 12 ? bits - 12 : 0;
}

// device-sized launch (the speculative final round): the item count lives in
// *mdev; a count above the launch's capacity m means the launch does not
// apply and every kernel returns at once
__device__ __forceinline__ bool dev_count(const unsigned long long* mdev, uint32_t& m) {
    if (!mdev) return true;
    const unsigned long long x = *mdev;
    if (x > m) return false;
    m = (uint32_t)x;
    return true;
}

__global__ void __launch_bounds__(1024)
k_bucket_order(const uint32_t* __restrict__ in, uint32_t m, const unsigned long long* __restrict__ key,
               unsigned long long kmin, int shift, uint32_t* __restrict__ out,
               uint32_t* __restrict__ bstart, const unsigned long long* __restrict__ mdev,
               const unsigned long long* __restrict__ pslots = nullptr, int use_thr = 1) {
    pdl_wait();
    if (!dev_count(mdev, m)) return;
    if (pslots) bucket_params_dev(pslots, use_thr, kmin, shift);
    __shared__ uint32_t cnt[kKeyBuckets];
    for (uint32_t b = threadIdx.x; b < kKeyBuckets; b += 1024) cnt[b] = 0;
    __syncthreads();
    uint32_t bk[kCTAItems];
#pragma unroll
    for (int j = 0; j < kCTAItems; ++j) {
        const uint32_t i = threadIdx.x + j * 1024;
        bk[j] = 0;
        if (i < m) {
            bk[j] = key_bucket(key[in[i]], kmin, shift);
            atomicAdd(&cnt[bk[j]], 1u);
        }
    }
    __syncthreads();
    const uint32_t total = block_exclusive_scan_4096(cnt);
    for (uint32_t b = threadIdx.x; b < kKeyBuckets; b += 1024) bstart[b] = cnt[b];
    if (threadIdx.x == 0) bstart[kKeyBuckets] = total;
    __syncthreads();  // bstart read cnt before the scatter below bumps it
#pragma unroll
    for (int j = 0; j < kCTAItems; ++j) {
        const uint32_t i = threadIdx.x + j * 1024;
        if (i < m) out[atomicAdd(&cnt[bk[j]], 1u)] = in[i];
    }
}

__global__ void k_bucket_rank(const uint32_t* __restrict__ in, uint32_t m,
                              const unsigned long long* __restrict__ key,
                              const int64_t* __restrict__ ids, unsigned long long kmin, int shift,
                              const uint32_t* __restrict__ bstart, uint32_t* __restrict__ out,
                              const unsigned long long* __restrict__ mdev,
                              const unsigned long long* __restrict__ pslots = nullptr,
                              int use_thr = 1) {
    pdl_wait();
    if (!dev_count(mdev, m)) return;
    if (pslots) bucket_params_dev(pslots, use_thr, kmin, shift);
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
        const uint32_t p = in[i];
        const unsigned long long kp = key[p];
        const long long ip = ids ? ids[p] : (long long)p;  // (no ids: position order)
        const uint32_t b = key_bucket(kp, kmin, shift);
        const uint32_t s0 = bstart[b], s1 = bstart[b + 1];
        uint32_t rank = 0;
        for (uint32_t j = s0; j < s1; ++j) {
            const uint32_t q = in[j];
            const unsigned long long kq = key[q];
            const long long iq = ids ? ids[q] : (long long)q;
            rank += (kq < kp) | ((kq == kp) & ((iq < ip) | ((iq == ip) & (q < p))));
        }
        out[s0 + rank] = p;
    }
}

// K4: warp-per-candidate SFS inside the (sum, id)-sorted prefix Av[d][m]:
// candidate i tests its predecessors 0..i-1 in sum order (strongest
// dominators first), 32 per iteration, leaving at the first non-zero ballot
// (north_star (a): warp-ballot early exit).
template <int D>
__global__ void __launch_bounds__(kBlock)
k_sfs_intra_sorted(const double* __restrict__ Av, uint32_t m, int d, uint8_t* __restrict__ keep,
                   unsigned long long* __restrict__ tests) {
    pdl_wait();
    constexpr int DM = D > 0 ? D : kMaxDims;
    const int dd = D > 0 ? D : d;
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    unsigned long long cnt = 0;
    for (uint32_t i = warp; i < m; i += nwarps) {
        double t[DM];
#pragma unroll
        for (int k = 0; k < DM; ++k)
            if (k < dd) t[k] = Av[(uint64_t)k * m + i];
        bool dominated = false;
        for (uint32_t j0 = 0; j0 < i; j0 += 32) {
            const uint32_t j = j0 + lane;
            bool hit = false;
            if (j < i) {
                double s[DM];
#pragma unroll
                for (int k = 0; k < DM; ++k)
                    if (k < dd) s[k] = Av[(uint64_t)k * m + j];
                hit = D > 0 ? dom_f64<(D > 0 ? D : 1)>(s, t) : dom_f64_dyn(s, t, dd);
                ++cnt;
            }
            if (__any_sync(0xffffffffu, hit)) {
                dominated = true;
                break;
            }
        }
        if (lane == 0) keep[i] = dominated ? 0 : 1;
    }
    add_count(tests, cnt);
}

// K5: 32 candidates are loaded per warp at once (lane-parallel, coalesced),
// then decided one after another with the whole warp scanning the new
// skyline tuples Pv[d][pcap] (np = slots[S_C2], all preceding the candidate
// in (sum, id) order) 32 at a time, starting in the candidate's own cell and
// wrapping around; ballot exit at the first dominator.  keep[i] = 1 marks
// survivors (compacted in order by the caller).
template <int D>
__global__ void __launch_bounds__(kBlock)
k_sfs_filter_cells(const double* __restrict__ v, int d, const unsigned long long* __restrict__ key,
                   const uint32_t* __restrict__ R, uint32_t r, const double* __restrict__ Pv,
                   uint32_t pcap, const uint32_t* __restrict__ seg, int m,
                   const unsigned long long* __restrict__ slots, uint8_t* __restrict__ keep,
                   unsigned long long* __restrict__ tests, uint32_t bs) {
    pdl_wait();
    constexpr int DM = D > 0 ? D : kMaxDims;
    const int dd = D > 0 ? D : d;
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    const unsigned long long T = slots[S_THR];
    const uint32_t np = (uint32_t)slots[S_C2];
    unsigned long long cnt = 0;
    for (uint32_t base = warp * bs; base < r; base += nwarps * bs) {
        const uint32_t idx = base + lane;
        const bool valid = lane < bs && idx < r;
        const uint32_t p = valid ? (R ? R[idx] : idx) : 0;
        double t[DM];
#pragma unroll
        for (int k = 0; k < DM; ++k)
            if (k < dd) t[k] = valid ? v[(uint64_t)p * dd + k] : 0.0;
        const bool need = valid && !(key[p] < T);  // not in the (decided) prefix
        const uint32_t start = (need && seg) ? seg[direction_cell<DM>(t, dd, m)] : 0;
        bool mykeep = need;
        unsigned todo = __ballot_sync(0xffffffffu, need);
        while (todo) {
            const int j = __ffs(todo) - 1;
            todo &= todo - 1;
            double tj[DM];
#pragma unroll
            for (int k = 0; k < DM; ++k)
                if (k < dd) tj[k] = __shfl_sync(0xffffffffu, t[k], j);
            uint32_t q = __shfl_sync(0xffffffffu, start, j) + lane;
            if (q >= np) q -= np;
            bool dominated = false;
            for (uint32_t done = 0; done < np; done += 32) {
                bool hit = false;
                if (done + lane < np) {
                    double s[DM];
#pragma unroll
                    for (int k = 0; k < DM; ++k)
                        if (k < dd) s[k] = Pv[(uint64_t)k * pcap + q];
                    hit = D > 0 ? dom_f64<(D > 0 ? D : 1)>(s, tj) : dom_f64_dyn(s, tj, dd);
                    ++cnt;
                }
                if (__any_sync(0xffffffffu, hit)) {
                    dominated = true;
                    break;
                }
                q += 32;
                if (q >= np) q -= np;
            }
            if ((int)lane == j) mykeep = !dominated;
        }
        if (valid) keep[idx] = mykeep ? 1 : 0;
    }
    add_count(tests, cnt);
}

// K4 with the quantised prefilter (D in 1..8): candidate i against its
// predecessors in sum order, 64 per ballot (two per lane); a comparator
// whose 16-bit codes are not all <= the candidate's is rejected with one
// SWAR test per code word, the rest take the exact float64 test.
template <int D>
__global__ void __launch_bounds__(kBlock)
k_sfs_intra_q(const double* __restrict__ Av, const unsigned long long* __restrict__ Aq,
              uint32_t m, uint8_t* __restrict__ keep, unsigned long long* __restrict__ tests) {
    pdl_wait();
    constexpr int W = QW<D>::W;
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    unsigned long long cnt = 0;
    for (uint32_t i = warp; i < m; i += nwarps) {
        double t[D];
#pragma unroll
        for (int k = 0; k < D; ++k) t[k] = Av[(uint64_t)k * m + i];
        unsigned long long tg[W];
#pragma unroll
        for (int k = 0; k < W; ++k) tg[k] = Aq[(uint64_t)i * W + k] | kH16;
        bool dominated = false;
        for (uint32_t j0 = 0; j0 < i; j0 += 64) {
            bool hit = false;
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const uint32_t j = j0 + u * 32 + lane;
                if (j < i) {
                    ++cnt;
                    if (le16<D>(Aq + (uint64_t)j * W, tg)) {
                        double s[D];
#pragma unroll
                        for (int k = 0; k < D; ++k) s[k] = Av[(uint64_t)k * m + j];
                        hit |= dom_f64<D>(s, t);
                    }
                }
            }
            if (__any_sync(0xffffffffu, hit)) {
                dominated = true;
                break;
            }
        }
        if (lane == 0) keep[i] = dominated ? 0 : 1;
    }
    add_count(tests, cnt);
}

// K4, chunked: the predecessor scan of a prefix member is split into chunks
// of kIntraChunk comparators, one warp per (chunk, candidate) item, so the
// long scans of late skyline members no longer serialise the kernel on one
// warp's load-latency chain.  Items run chunk-major (chunk 0 of every
// candidate first); a warp that finds a dominator clears keep[i] (pre-set to
// 1), and the other chunks of that candidate poll it and stop.  128
// comparators per ballot (four per lane, loads in flight together).
constexpr uint32_t kIntraChunk = 1024;

template <int D>
__global__ void __launch_bounds__(kBlock)
k_sfs_intra_chunked(const double* __restrict__ Av, const unsigned long long* __restrict__ Aq,
                    uint32_t m, volatile uint8_t* keep, unsigned long long* __restrict__ tests,
                    uint32_t astride, const unsigned long long* __restrict__ mdev) {
    pdl_wait();
    if (!dev_count(mdev, m)) return;
    constexpr int W = QW<D>::W;
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    const uint32_t nch = (m + kIntraChunk - 1) / kIntraChunk;
    uint64_t total = 0;
    for (uint32_t c = 0; c < nch; ++c)
        if ((uint64_t)c * kIntraChunk + 1 < m) total += m - c * kIntraChunk - 1;
    unsigned long long cnt = 0;
    for (uint64_t it = warp; it < total; it += nwarps) {
        uint64_t rem = it;
        uint32_t c = 0;
        for (;;) {
            const uint64_t nc = m - c * kIntraChunk - 1;
            if (rem < nc) break;
            rem -= nc;
            ++c;
        }
        const uint32_t i = c * kIntraChunk + 1 + (uint32_t)rem;
        // another chunk already found a dominator (keep[i] moves under other
        // warps: the warp takes lane 0's reading, so no lane skips the votes
        // below that the others wait at)
        if (__shfl_sync(0xffffffffu, (unsigned)(keep[i] == 0), 0)) continue;
        const uint32_t j1 = min(i, (c + 1) * kIntraChunk);
        double t[D];
#pragma unroll
        for (int k = 0; k < D; ++k) t[k] = Av[(uint64_t)k * astride + i];
        unsigned long long tg[W];
#pragma unroll
        for (int k = 0; k < W; ++k) tg[k] = Aq[(uint64_t)i * W + k] | kH16;
        bool dominated = false;
        for (uint32_t j0 = c * kIntraChunk; j0 < j1; j0 += 128) {
            bool hit = false;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint32_t j = j0 + u * 32 + lane;
                if (j < j1) {
                    ++cnt;
                    if (le16<D>(Aq + (uint64_t)j * W, tg)) {
                        double s[D];
#pragma unroll
                        for (int k = 0; k < D; ++k) s[k] = Av[(uint64_t)k * astride + j];
                        hit |= dom_f64<D>(s, t);
                    }
                }
            }
            if (__any_sync(0xffffffffu, hit)) {
                dominated = true;
                break;
            }
            if (__shfl_sync(0xffffffffu, (unsigned)(keep[i] == 0), 0)) break;
        }
        if (dominated && lane == 0) keep[i] = 0;
    }
    add_count(tests, cnt);
}

// K4 with the prefix's codes resident in shared memory (one u64 code word
// per tuple for d <= 4, two for d <= 8; <= 16384 words = 128 KB): one CTA per SM loads the
// codes once, then each warp takes a candidate (longest first: candidate i
// has i predecessors) and scans its predecessors in sum order, 64 per vote
// (two per lane), shared-memory latency instead of L2 latency per step; the
// exact float64 test runs only on a code pass.  keep[i] is written for
// every i < m.
constexpr uint32_t kIntraSmemMax = 16384;

template <int D>
__global__ void __launch_bounds__(1024, 1)
k_sfs_intra_smem(const double* __restrict__ Av, const unsigned long long* __restrict__ Aq,
                 uint32_t m, uint8_t* __restrict__ keep, unsigned long long* __restrict__ tests,
                 uint32_t astride, const unsigned long long* __restrict__ mdev,
                 uint32_t scap) {
    pdl_wait();
    constexpr int W = QW<D>::W;  // code words per tuple (1: d <= 4, 2: d <= 8)
    if (!dev_count(mdev, m)) return;
    // the codes in shared memory when they fit the launch's allocation
    // (scap words), else read through L1 (a device-sized round larger than
    // expected): same results either way
    extern __shared__ unsigned long long sq_sm[];
    const bool in_smem = (uint64_t)m * W <= scap;
    if (in_smem)
        for (uint32_t j = threadIdx.x; j < m * W; j += blockDim.x) sq_sm[j] = Aq[j];
    __syncthreads();
    // (two instantiations of the scan so the shared-memory one keeps LDS)
    unsigned long long cnt = 0;
    auto scan = [&](const unsigned long long* __restrict__ sq) {
        const uint32_t lane = threadIdx.x & 31;
        // consecutive candidates (similar cost) on different SMs
        const uint32_t warp = (threadIdx.x >> 5) * gridDim.x + blockIdx.x;
        const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
        for (uint32_t k = warp; k < m; k += nwarps) {
            const uint32_t i = m - 1 - k;
            unsigned long long tg[W];
#pragma unroll
            for (int w = 0; w < W; ++w) tg[w] = sq[(uint64_t)i * W + w] | kH16;
            double t[D];
#pragma unroll
            for (int a = 0; a < D; ++a) t[a] = Av[(uint64_t)a * astride + i];
            bool dominated = false;
            // 128 comparators per step, the code tests branch-free; only a step
            // with a code pass somewhere in the warp takes the exact tests.
            // Full steps carry no bounds checks; the partial last one does.
            auto step = [&](uint32_t j0, bool full) -> bool {
                unsigned pm = 0;
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const uint32_t j = j0 + u * 32 + lane;
                    const bool in = full || j < i;
                    bool ok = in;
#pragma unroll
                    for (int w = 0; w < W; ++w) {
                        const unsigned long long cq = in ? sq[(uint64_t)j * W + w] : 0ULL;
                        ok &= ((tg[w] - cq) & kH16) == kH16;
                    }
                    pm |= (unsigned)ok << u;
                }
                if (!__any_sync(0xffffffffu, pm != 0)) return false;
                bool hit = false;
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    if ((pm >> u) & 1u) {
                        const uint32_t j = j0 + u * 32 + lane;
                        double sv[D];
#pragma unroll
                        for (int a = 0; a < D; ++a) sv[a] = Av[(uint64_t)a * astride + j];
                        hit |= dom_f64<D>(sv, t);
                    }
                }
                return __any_sync(0xffffffffu, hit);
            };
            uint32_t j0 = 0;
            for (; j0 + 128 <= i && !dominated; j0 += 128) dominated = step(j0, true);
            if (!dominated && j0 < i) {
                dominated = step(j0, false);
                j0 += 128;
            }
            if (lane == 0) {
                cnt += j0 < i ? j0 : i;  // comparators examined (whole steps)
                keep[i] = dominated ? 0 : 1;
            }
        }
    };
    if (in_smem)
        scan(sq_sm);
    else
        scan(Aq);
    add_count(tests, cnt);
}

// K5 with the quantised prefilter (D in 1..8).  Two scan modes:
//  qk > 0  quantile grid (the default): the new skyline tuples A' are grouped
//          by a k^d grid whose bin bounds are quantiles of A' itself; a
//          comparator in a cell with any bin above the candidate's cannot
//          dominate it (its value there is >= a bound > the candidate's), so
//          only the cells <= the candidate's own cell are visited, own cell
//          first, then descending — an EXACT pruning of the comparator set
//          (the GPU recast of the paper's partition-level pruning).
//  qk == 0 plan cells (grid / angular / sliced / direction): own partition
//          first, then all others (scan order only).
// Phase A: every lane alone tests the first kSolo (16) comparators of its own cell
// (most candidates are dominated there — no shuffles, no votes); phase B:
// warp-cooperative, 32 comparators per ballot, for the still-undecided ones.
template <int D>
__global__ void __launch_bounds__(kBlock)
k_sfs_filter_q(const double* __restrict__ v, const unsigned long long* __restrict__ key,
               const uint32_t* __restrict__ R, uint32_t r, const double* __restrict__ Pv,
               const unsigned long long* __restrict__ Pq, uint32_t pcap,
               const uint32_t* __restrict__ seg, int m, int qk,
               const unsigned long long* __restrict__ amax,
               const unsigned long long* __restrict__ slots, uint8_t* __restrict__ keep,
               unsigned long long* __restrict__ tests, uint32_t bs,
               const uint32_t* __restrict__ Ppos, const int64_t* __restrict__ ids,
               uint32_t kSolo) {
    pdl_wait();
    // Ppos != nullptr: A' is a seed that need not precede every candidate
    // (host-overlapped first part, skygpu_pipeline); a dominating comparator
    // then also has to precede the candidate in (sum, id, position) order
    auto precedes_pos = [&](uint32_t ps, uint32_t pt) {
        const unsigned long long ks = key[ps], kt = key[pt];
        if (ks != kt) return ks < kt;
        if (!ids) return ps < pt;  // (ids in flight: position order, checked later)
        const int64_t is = ids[ps], it = ids[pt];
        return is < it || (is == it && ps < pt);
    };
    constexpr int W = QW<D>::W;
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    if (slots[S_GATE]) {  // the host switches to the rank-grid engine: keep all
        for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < r; i += gridDim.x * blockDim.x)
            keep[i] = 1;
        return;
    }
    const unsigned long long T = slots[S_THR];
    const uint32_t np = (uint32_t)slots[S_C2];
    double sc[D];
    load_scales<D>(amax, sc);
    unsigned long long cnt = 0;
    for (uint32_t base = warp * bs; base < r; base += nwarps * bs) {
        const uint32_t idx = base + lane;
        const bool valid = lane < bs && idx < r;
        const uint32_t p = valid ? (R ? R[idx] : idx) : 0;
        double t[D];
#pragma unroll
        for (int k = 0; k < D; ++k) t[k] = valid ? v[(uint64_t)p * D + k] : 0.0;
        unsigned long long tq[W];
        encode16<D>(t, sc, tq);
        const bool need = valid && !(key[p] < T) && np > 0;  // not in the (decided) prefix
        uint32_t mycell = 0, start = 0, lim = 0;
        if (need && seg) {
            mycell = qk > 0 ? qgrid_cell<D>(t, D, qk) : plan_cell<D>(t, D, m, amax);
            start = seg[mycell];
        }
        if (need) {
            if (qk > 0) {
                const uint32_t own = seg[mycell + 1] - start;
                lim = own < kSolo ? own : kSolo;
            } else {
                lim = np < kSolo ? np : kSolo;
            }
        }
        bool mykeep = need, undecided = need;
        if (need) {  // phase A
            unsigned long long tgl[W];
#pragma unroll
            for (int k = 0; k < W; ++k) tgl[k] = tq[k] | kH16;
            uint32_t q = start >= np ? 0 : start;
            for (uint32_t s = 0; s < lim; ++s) {
                ++cnt;
                if (le16<D>(Pq + (uint64_t)q * W, tgl)) {
                    double sv[D];
#pragma unroll
                    for (int k = 0; k < D; ++k) sv[k] = Pv[(uint64_t)k * pcap + q];
                    if (dom_f64<D>(sv, t) && (!Ppos || precedes_pos(Ppos[q], p))) {
                        mykeep = false;
                        undecided = false;
                        break;
                    }
                }
                if (++q >= np) q = 0;
            }
            if (qk == 0 && lim == np) undecided = false;  // every comparator tested
        }
        unsigned todo = __ballot_sync(0xffffffffu, undecided);
        while (todo) {  // phase B
            const int j = __ffs(todo) - 1;
            todo &= todo - 1;
            double tj[D];
#pragma unroll
            for (int k = 0; k < D; ++k) tj[k] = __shfl_sync(0xffffffffu, t[k], j);
            unsigned long long tg[W];
#pragma unroll
            for (int k = 0; k < W; ++k) tg[k] = __shfl_sync(0xffffffffu, tq[k], j) | kH16;
            const uint32_t pj = __shfl_sync(0xffffffffu, p, j);
            bool dominated = false;
            if (qk > 0) {
                // cells <= own, own first then descending (mixed-radix counter)
                const uint32_t own = __shfl_sync(0xffffffffu, mycell, j);
                const uint32_t skip = __shfl_sync(0xffffffffu, lim, j);
                int od[D], dig[D];
                uint32_t tmp = own;
#pragma unroll
                for (int k = 0; k < D; ++k) {
                    od[k] = (int)(tmp % (uint32_t)qk);
                    tmp /= (uint32_t)qk;
                    dig[k] = od[k];
                }
                uint32_t cell = own;
                while (true) {
                    const uint32_t s1 = seg[cell + 1];
                    for (uint32_t q0 = seg[cell] + (cell == own ? skip : 0); q0 < s1; q0 += 32) {
                        const uint32_t q = q0 + lane;
                        bool hit = false;
                        if (q < s1) {
                            ++cnt;
                            if (le16<D>(Pq + (uint64_t)q * W, tg)) {
                                double s[D];
#pragma unroll
                                for (int k = 0; k < D; ++k) s[k] = Pv[(uint64_t)k * pcap + q];
                                hit = dom_f64<D>(s, tj) && (!Ppos || precedes_pos(Ppos[q], pj));
                            }
                        }
                        if (__any_sync(0xffffffffu, hit)) {
                            dominated = true;
                            break;
                        }
                    }
                    if (dominated) break;
                    int k = 0;
                    uint32_t w = 1;
                    for (; k < D; ++k, w *= (uint32_t)qk) {
                        if (dig[k] > 0) {
                            --dig[k];
                            cell -= w;
                            break;
                        }
                        dig[k] = od[k];
                        cell += (uint32_t)od[k] * w;
                    }
                    if (k == D) break;  // every cell <= own visited
                }
            } else {
                uint32_t q = __shfl_sync(0xffffffffu, start, j) + kSolo + lane;
                while (q >= np) q -= np;
                uint32_t done = kSolo;
                for (; done < np; done += 32) {
                    bool hit = false;
                    if (done + lane < np) {
                        if (le16<D>(Pq + (uint64_t)q * W, tg)) {
                            double s[D];
#pragma unroll
                            for (int k = 0; k < D; ++k) s[k] = Pv[(uint64_t)k * pcap + q];
                            hit = dom_f64<D>(s, tj) && (!Ppos || precedes_pos(Ppos[q], pj));
                        }
                    }
                    q += 32;
                    while (q >= np) q -= np;
                    if (__any_sync(0xffffffffu, hit)) {
                        dominated = true;
                        done += 32;
                        break;
                    }
                }
                // comparators examined, counted once (not per lane and step)
                if ((int)lane == j && np > kSolo) cnt += min(done, np) - kSolo;
            }
            if ((int)lane == j) mykeep = !dominated;
        }
        if (valid) keep[idx] = mykeep ? 1 : 0;
    }
    add_count(tests, cnt);
}

// One-CTA order-preserving compaction of up to 16384 flagged items (and
// their cell keys); the count lands in *count.
__global__ void __launch_bounds__(1024)
k_cta_select(const uint32_t* __restrict__ in, const uint32_t* __restrict__ in_cell,
             const uint8_t* __restrict__ flags, uint32_t m, uint32_t* __restrict__ out,
             uint32_t* __restrict__ out_cell, unsigned long long* __restrict__ count,
             const unsigned long long* __restrict__ mdev = nullptr,
             const unsigned long long* __restrict__ out_off = nullptr) {
    pdl_wait();
    if (!dev_count(mdev, m)) return;
    if (out_off) out += *out_off;
    using Scan = cub::BlockScan<uint32_t, 1024>;
    __shared__ typename Scan::TempStorage tmp;
    uint32_t f[kCTAItems];
    uint32_t local = 0;
#pragma unroll
    for (int j = 0; j < kCTAItems; ++j) {
        const uint32_t i = threadIdx.x * kCTAItems + j;
        f[j] = (i < m && flags[i]) ? 1u : 0u;
        local += f[j];
    }
    uint32_t offset = 0, total = 0;
    Scan(tmp).ExclusiveSum(local, offset, total);
#pragma unroll
    for (int j = 0; j < kCTAItems; ++j) {
        const uint32_t i = threadIdx.x * kCTAItems + j;
        if (f[j]) {
            out[offset] = in[i];
            if (out_cell) out_cell[offset] = in_cell[i];
            ++offset;
        }
    }
    if (threadIdx.x == 0) *count = total;
}

__global__ void k_keys_of(const unsigned long long* __restrict__ key,
                          const uint32_t* __restrict__ list, uint64_t m,
                          unsigned long long* __restrict__ out) {
    pdl_wait();
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
         i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = key[list[i]];
}

__global__ void k_id_keys(const int64_t* __restrict__ ids, const uint32_t* __restrict__ list,
                          uint64_t m, unsigned long long* __restrict__ out) {
    pdl_wait();
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
         i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = static_cast<unsigned long long>(ids[list[i]]) ^ 0x8000000000000000ULL;
}

// (D > 0: the tuple's D values loaded together, then stored per attribute)
template <int D>
__global__ void k_emit_skyline(const uint32_t* __restrict__ K, uint64_t S,
                               const double* __restrict__ v, int d,
                               const int64_t* __restrict__ ids, int64_t* __restrict__ oid,
                               double* __restrict__ skyv, uint64_t* __restrict__ pos64) {
    pdl_wait();
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < S;
         k += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t p = K[k];
        if (ids) oid[k] = ids[p];
        pos64[k] = p;  // (the output's u64 positions, no separate widening pass)
        if constexpr (D > 0) {
            double t[D];
#pragma unroll
            for (int a = 0; a < D; ++a) t[a] = v[(uint64_t)p * D + a];
#pragma unroll
            for (int a = 0; a < D; ++a) skyv[a * S + k] = t[a];
        } else {
            for (int a = 0; a < d; ++a) skyv[a * S + k] = v[(uint64_t)p * d + a];
        }
    }
}

template <class KT>
void sort_pairs(Ctx& c, KT* k0, KT* k1, uint32_t* v0, uint32_t* v1, uint64_t n, int end_bit,
                KT** kout, uint32_t** vout) {
    cub::DoubleBuffer<KT> kb(k0, k1);
    cub::DoubleBuffer<uint32_t> vb(v0, v1);
    size_t tmp = 0;
    SKY_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, kb, vb, (int64_t)n, 0, end_bit,
                                             c.stream));
    void* t = c.buf[B_CUB].get(tmp);
    SKY_CUDA(cub::DeviceRadixSort::SortPairs(t, tmp, kb, vb, (int64_t)n, 0, end_bit, c.stream));
    note_launch(c, 4);
    *kout = kb.Current();
    *vout = vb.Current();
}

// order-preserving compactions (CUB DeviceSelect); counts stay on the device
template <class Op>
void select_if(Ctx& c, const uint32_t* R, uint64_t r, Op op, uint32_t* out,
               unsigned long long* d_count) {
    size_t tmp = 0;
    if (R) {
        SKY_CUDA(cub::DeviceSelect::If(nullptr, tmp, R, out, d_count, (int64_t)r, op, c.stream));
        void* t = c.buf[B_CUB].get(tmp);
        SKY_CUDA(cub::DeviceSelect::If(t, tmp, R, out, d_count, (int64_t)r, op, c.stream));
    } else {
        cub::CountingInputIterator<uint32_t> it(0);
        SKY_CUDA(cub::DeviceSelect::If(nullptr, tmp, it, out, d_count, (int64_t)r, op, c.stream));
        void* t = c.buf[B_CUB].get(tmp);
        SKY_CUDA(cub::DeviceSelect::If(t, tmp, it, out, d_count, (int64_t)r, op, c.stream));
    }
    note_launch(c, 2);
}

template <class T>
void select_flags(Ctx& c, const T* R, uint64_t r, const uint8_t* flags, T* out,
                  unsigned long long* d_count) {
    size_t tmp = 0;
    if (R) {
        SKY_CUDA(cub::DeviceSelect::Flagged(nullptr, tmp, R, flags, out, d_count, (int64_t)r,
                                             c.stream));
        void* t = c.buf[B_CUB].get(tmp);
        SKY_CUDA(cub::DeviceSelect::Flagged(t, tmp, R, flags, out, d_count, (int64_t)r,
                                             c.stream));
    } else {
        cub::CountingInputIterator<T> it(0);
        SKY_CUDA(cub::DeviceSelect::Flagged(nullptr, tmp, it, flags, out, d_count, (int64_t)r,
                                             c.stream));
        void* t = c.buf[B_CUB].get(tmp);
        SKY_CUDA(cub::DeviceSelect::Flagged(t, tmp, it, flags, out, d_count, (int64_t)r,
                                             c.stream));
    }
    note_launch(c, 2);
}

// candidates per warp batch: 32 (one coalesced load per lane) when there
// are enough candidates to keep ~48 warps per SM busy, fewer otherwise
uint32_t batch_size(const Ctx& c, uint64_t count) {
    const uint64_t target_warps = (uint64_t)c.num_sms * 48;
    uint64_t bs = (count + target_warps - 1) / target_warps;
    return (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(32, bs));
}

int cells_per_dim(uint64_t m, int d, uint32_t* ncells);

// The scan-order cell spec (see plan_cell): direction cells sized for ~128
// tuples each — measured faster than the plan's own partition (C2 -4%, C1
// -3%, C4/C3 even: one float division per candidate instead of the angular
// plan's arctangents); SKYGPU_SCAN_CELLS=plan scans in the plan's partition
// when it has at most kMaxCells parts (and d <= 8 for the attribute-scaled
// kinds).  Scan order only: the results never depend on it.
int scan_cell_spec(const skygpu_plan& plan, uint64_t m, int d, bool qpre, uint32_t* ncells) {
    static const bool dir_only = [] {
        const char* e = getenv("SKYGPU_SCAN_CELLS");
        return !(e && e[0] == 'p');
    }();
    if (dir_only) {
        const int mc = cells_per_dim(m, d, ncells);
        return mc > 1 ? mc : 0;
    }
    auto ipow = [](uint64_t b, int e) {
        uint64_t v = 1;
        for (int i = 0; i < e; ++i) {
            v *= b;
            if (v > kMaxCells) return (uint64_t)kMaxCells + 1;
        }
        return v;
    };
    if (qpre && plan.strategy == SKYGPU_GRID && plan.slices >= 1) {
        const uint64_t nc = ipow((uint64_t)plan.slices, d);
        if (nc > 1 && nc <= kMaxCells) {
            *ncells = (uint32_t)nc;
            return (kCellGrid << 16) | plan.slices;
        }
    }
    if (qpre && plan.strategy == SKYGPU_ANGULAR && plan.slices >= 1 && d >= 2) {
        const uint64_t nc = ipow((uint64_t)plan.slices, d - 1);
        if (nc > 1 && nc <= kMaxCells) {
            *ncells = (uint32_t)nc;
            return (kCellAngular << 16) | plan.slices;
        }
    }
    if (qpre && plan.strategy == SKYGPU_SLICED && plan.partitions > 1) {
        const uint32_t nc = (uint32_t)std::min<long long>(plan.partitions, kMaxCells);
        *ncells = nc;
        return (kCellSliced << 16) | (int)nc;
    }
    const int mc = cells_per_dim(m, d, ncells);
    return mc > 1 ? mc : 0;
}

// bins per normalised coordinate so that the cells hold ~128 tuples each
int cells_per_dim(uint64_t m, int d, uint32_t* ncells) {
    int mcell = 1;
    if (d >= 2) {
        static const double per_cell = [] {
            const char* e = getenv("SKYGPU_DIR_PER_CELL");
            const double x = e ? atof(e) : 0.0;
            return x > 0 ? x : 128.0;
        }();
        const double target = std::max(1.0, (double)m / per_cell);
        mcell = (int)std::floor(std::pow(target, 1.0 / (d - 1)) + 1e-9);
        mcell = std::max(1, std::min(mcell, 64));
    }
    uint32_t nc = 1;
    for (int k = 0; k < d - 1; ++k) nc *= (uint32_t)mcell;
    if (nc > kMaxCells) mcell = 1, nc = 1;
    *ncells = nc;
    return mcell;
}

}  // namespace

namespace {
// first-round engine gate: most of the prefix survived -> rank-grid engine
__global__ void k_grid_gate(unsigned long long* slots, uint64_t m) {
    pdl_wait();
    if (m == 0) m = slots[S_C1];  // (a device-sized round: the prefix count)
    if (threadIdx.x == 0) slots[S_GATE] = slots[S_C2] * 4 > m * 3 ? 1ULL : 0ULL;
}
// streamed input: seeded K5 state (no decided prefix, |A'| = the seed)
__global__ void k_seed_slots(unsigned long long* slots, uint64_t nseed) {
    pdl_wait();
    if (threadIdx.x == 0) {
        slots[S_THR] = 0;
        slots[S_C2] = nseed;
    }
}
__global__ void k_iota(uint32_t* __restrict__ a, uint64_t n) {
    pdl_wait();
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        a[i] = (uint32_t)i;
}
}  // namespace

SkylineOut skyline_device(Ctx& c, const double* d_vals, const int64_t* d_ids, uint64_t n, int d,
                          const skygpu_plan& plan, const double* d_reps, uint64_t n_reps,
                          unsigned sky_engine, const TailFeed* feed) {
    SkylineOut out;
    skygpu_stats& st = *c.st;
    if (n == 0) return out;
    if (n >= 0xFFFFFFFFull) invalid("parallel_skyline: more than 2^32-1 tuples");
    const unsigned gb = grid_for(n, kBlock);
    // ---- streamed input: seed from the head while the rest is still in flight
    uint32_t* seed = nullptr;
    uint64_t nseed = 0;
    bool head_grid = false;
    unsigned long long* scale_snap = nullptr;
    if (feed) {
        SKY_CUDA(cudaStreamWaitEvent(c.stream, feed->ready[0], 0));
        const bool eligible = d >= 1 && d <= 8 && plan.strategy != SKYGPU_GRID && n_reps == 0 &&
                              sky_engine != SKYGPU_SKY_GRID && feed->nchunks >= 2;
        if (eligible) {
            try {
                const SkylineOut h =
                    skyline_device(c, d_vals, d_ids, feed->bound[1], d, plan, nullptr, 0,
                                   kSkyAbortIfLarge | kSkyFirstPrefix, nullptr);
                head_grid = h.aborted;  // the head's first prefix asked for the rank grid
                if (!h.aborted && h.S > 0 && h.S <= kCTACap) {
                    seed = c.buf[B_SEED].as<uint32_t>(h.S);
                    scale_snap = c.buf[B_AMAX2].as<unsigned long long>(kMaxDims);
                    SKY_CUDA(cudaMemcpyAsync(seed, h.d_inpos, h.S * sizeof(uint32_t),
                                             cudaMemcpyDeviceToDevice, c.stream));
                    SKY_CUDA(cudaMemcpyAsync(scale_snap, c.buf[B_AMAX].p,
                                             sizeof(unsigned long long) * kMaxDims,
                                             cudaMemcpyDeviceToDevice, c.stream));
                    nseed = h.S;
                }
            } catch (const Error&) {
                // the full pass below reports the reference's error
            }
        }
        // deferred ids: straight behind the values (the tail work after the
        // last chunk is short), unless the rank grid comes next — then at its
        // compute-bound kernel, clear of the HBM-bound code passes
        if (!head_grid) issue_late_ids(c);
        if (!nseed) {
            for (int ch = 1; ch < feed->nchunks; ++ch)
                SKY_CUDA(cudaStreamWaitEvent(c.stream, feed->ready[ch], 0));
            feed = nullptr;
        }
        trace_mark(c, "sky: streamed head seed");
    }
    st.tuples_in = n;
    // ids still in flight (host-pointer pipeline): ties by position until the
    // ids are needed (rank grid, output); their strict order is checked then
    const bool ids_late = c.ids_ready != nullptr || c.ids_host != nullptr;
    const int64_t* tie_ids = ids_late ? nullptr : d_ids;
    bool ids_waited = false;
    auto ensure_ids = [&]() {
        // (the streamed head's seed never waits: its ids are not an output)
        if (!ids_late || ids_waited || (sky_engine & kSkyFirstPrefix)) return;
        ids_waited = true;
        issue_late_ids(c);  // (if K5 never ran)
        SKY_CUDA(cudaStreamWaitEvent(c.stream, c.ids_ready, 0));
        pdl_launch(k_ids_check, grid_for(n, kBlock), kBlock, 0, c.stream, d_ids, n, c.d_slots,
                   S_IDSBAD);
        SKY_LAUNCH_CHECK();
        note_launch(c);
    };

    zero_slots(c);
    auto* keys = c.buf[B_KEY0].as<unsigned long long>(n);
    trace_mark(c, "sky: start");
    // quantised prefilter for 1 <= d <= 8 (per-attribute maxima from K1)
    const bool qpre = d >= 1 && d <= 8;
    unsigned long long* amax = c.buf[B_AMAX].as<unsigned long long>(kMaxDims);
    SKY_CUDA(cudaMemsetAsync(amax, 0, sizeof(unsigned long long) * kMaxDims, c.stream));
    // prefix size per round: stays below the one-CTA capacity despite
    // sampling noise (SKYGPU_PREFIX overrides, for tuning)
    static const uint64_t kWant = [] {
        const char* e = getenv("SKYGPU_PREFIX");
        const long long v = e ? atoll(e) : 0;
        return v > 0 ? (uint64_t)v : (uint64_t)8000;
    }();
    static const bool fused_sel_on = [] {  // SKYGPU_FUSED_SELECT=0: CUB selection
        const char* e = getenv("SKYGPU_FUSED_SELECT");
        return !(e && e[0] == '0');
    }();
    // the first round's threshold sampled from the values and its prefix
    // appended by K1 itself (no separate selection pass) — plain rounds only
    // local-skyline pruning per plan partition before the merge (partition.cu)
    const bool lprune = c.local_prune && local_prune_applies(plan, d) && n > 1 &&
                        !(sky_engine & (kSkyAbortIfLarge | kSkyFirstPrefix));
    bool fused_first = !feed && sky_engine == 0 && !(plan.strategy == SKYGPU_GRID) &&
                       n_reps == 0 && qpre && n > kCTACap && fused_sel_on && !lprune;
    if (fused_first) {
        pdl_launch(k_sample_threshold, 1, 1024, 0, c.stream, (const unsigned long long*)nullptr,
                   (const uint32_t*)nullptr, n, kWant, c.d_slots, d_vals, d);
        SKY_LAUNCH_CHECK();
        note_launch(c);
    }
    if (!feed) {  // (streamed input: per chunk, below)
        uint32_t* pre = fused_first ? c.buf[B_IDX0].as<uint32_t>(n) : nullptr;
        dispatch_d(d, [&](auto DC) {
            constexpr int D = decltype(DC)::value;
            pdl_launch(k_score<D>, grid_for(n, kBlock, c.num_sms * 8), kBlock, 0, c.stream,
                       d_vals, n, d, keys, c.d_slots, amax, 0, tie_ids, pre);  // + ids order
        });
        SKY_LAUNCH_CHECK();
        note_launch(c, 1);
    }
    if (plan.strategy == SKYGPU_GRID) {
        pdl_launch(k_grid_range, grid_for(n * d, kBlock), kBlock, 0, c.stream, d_vals, n * d,
                   c.d_slots);
        SKY_LAUNCH_CHECK();
        note_launch(c);
    }

    uint32_t* R = nullptr;  // nullptr = all tuples
    uint64_t r = n;
    uint32_t* Rbuf0 = c.buf[B_R0].as<uint32_t>(n);
    uint32_t* Rbuf1 = c.buf[B_R1].as<uint32_t>(n);
    uint32_t* K = c.buf[B_KLIST].as<uint32_t>(n);
    uint32_t* seg_table = c.buf[B_ORDER].as<uint32_t>(kMaxCells + 1 + kKeyBuckets + 1);
    bool checked = false;
    // pre-merge pruning: the Grid plan's dominated cells (parallel.cpp:32-42)
    // and the representative filter (partition.cpp:287-302)
    uint64_t grid_cells = 0;
    if (plan.strategy == SKYGPU_GRID && plan.slices >= 2) {
        grid_cells = 1;
        for (int k = 0; k < d && grid_cells <= (1u << 22); ++k) grid_cells *= (uint64_t)plan.slices;
        if (grid_cells > (1u << 22)) grid_cells = 0;  // too fine to tabulate: skip pruning
    }
    uint64_t into_final = ~0ULL;  // survivors of the local pruning (the merge's input)
    if (grid_cells || n_reps > 0 || lprune) {
        uint8_t* pre = c.buf[B_FLAGS].as<uint8_t>(n);
        if (grid_cells) {
            const int m = plan.slices;
            uint8_t* occ = c.buf[B_CELLS].as<uint8_t>(grid_cells);
            SKY_CUDA(cudaMemsetAsync(occ, 0, grid_cells, c.stream));
            pdl_launch(k_grid_occ, gb, kBlock, 0, c.stream, d_vals, n, d, m, occ);
            SKY_LAUNCH_CHECK();
            uint32_t stride = 1;
            for (int k = 0; k < d; ++k, stride *= (uint32_t)m) {
                pdl_launch(k_prefix_or_dim, grid_for(grid_cells / m, kBlock), kBlock, 0, c.stream,
                    occ, (uint32_t)grid_cells, m, stride);
                SKY_LAUNCH_CHECK();
            }
            pdl_launch(k_grid_keep, gb, kBlock, 0, c.stream, d_vals, n, d, m, occ, pre);
            SKY_LAUNCH_CHECK();
            note_launch(c, 2 + d);
        }
        if (n_reps > 0) {
            dispatch_d(d, [&](auto DC) {
                constexpr int D = decltype(DC)::value;
                pdl_launch(k_rep_filter<D>, gb, kBlock, 0, c.stream, d_vals, n, d, d_reps,
                                                              (uint32_t)n_reps, pre,
                                                              c.d_slots + S_TESTS_SKY,
                                                              grid_cells ? 1 : 0);
            });
            SKY_LAUNCH_CHECK();
            note_launch(c);
        }
        uint64_t into_parallel = 0;
        if (lprune) {
            if (grid_cells || n_reps > 0) {  // the tuples entering the partitions
                select_flags<uint32_t>(c, nullptr, n, pre, Rbuf1, c.d_slots + S_C2);
            }
            uint8_t* lk = c.buf[B_PFLAGS].as<uint8_t>(n);
            local_prune_device(c, d_vals, keys, tie_ids, n, d, plan,
                               (grid_cells || n_reps > 0) ? pre : nullptr, lk, nullptr);
            pre = lk;
            trace_mark(c, "sky: local pruning");
        }
        select_flags<uint32_t>(c, nullptr, n, pre, Rbuf0, c.d_slots + S_C3);
        read_slots(c, S_BAD, 11);  // S_BAD .. S_C3 (checks + survivors)
        R = Rbuf0;
        r = c.h_slots[S_C3];
        into_parallel = lprune ? ((grid_cells || n_reps > 0) ? c.h_slots[S_C2] : n) : r;
        if (lprune) into_final = r;
        st.tuples_into_parallel = into_parallel;
    } else {
        st.tuples_into_parallel = r;
    }

    uint64_t kc = 0;
    static const uint64_t kSeedWant = [] {  // the streamed head's seed prefix
        const char* e = getenv("SKYGPU_SEED_PREFIX");
        const long long v = e ? atoll(e) : 0;
        return v > 0 ? (uint64_t)v : (uint64_t)8000;
    }();
    uint64_t want = (sky_engine & kSkyFirstPrefix) ? kSeedWant : kWant;
    const uint64_t kMaxPrefix = 65536, kFinal = kCTACap;
    const uint64_t kGridMin = 1u << 16;  // auto rank-grid engine from this many tuples
    int rounds = 0;
    cudaEvent_t e0 = c.ev[8], e1 = c.ev[9], e2 = c.ev[14], e3 = c.ev[15];
    double kernel_ms = 0;
    uint64_t kernel_launches = 0;
    uint32_t* Rnext = Rbuf1;
    bool ids_sorted = true;
    // device radix sort of a position list (in position order) by (sum, id,
    // position); returns the buffer holding the sorted list (Pfull or B_IDX1)
    auto radix_order = [&](uint32_t* Pfull, uint64_t m) -> uint32_t* {
        uint32_t* Ps = c.buf[B_IDX1].as<uint32_t>(m);
        uint32_t* order = Ps;
        unsigned long long* Pkey = c.buf[B_KEY1].as<unsigned long long>(m);
        unsigned long long* Pkey2 = c.buf[B_GTMP0].as<unsigned long long>(m);
        unsigned long long* kcur;
        if (ids_sorted) {
            pdl_launch(k_keys_of, grid_for(m, kBlock), kBlock, 0, c.stream, keys, Pfull, m, Pkey);
            SKY_LAUNCH_CHECK();
            sort_pairs<unsigned long long>(c, Pkey, Pkey2, Pfull, Ps, m, 64, &kcur, &order);
        } else {  // stable LSD: by id first, then by sum
            unsigned long long* ik0 = c.buf[B_GTMP1].as<unsigned long long>(m);
            pdl_launch(k_id_keys, grid_for(m, kBlock), kBlock, 0, c.stream, d_ids, Pfull, m, ik0);
            SKY_LAUNCH_CHECK();
            unsigned long long* ikc;
            uint32_t* by_id;
            sort_pairs<unsigned long long>(c, ik0, Pkey2, Pfull, Ps, m, 64, &ikc, &by_id);
            uint32_t* other = by_id == Pfull ? Ps : Pfull;
            pdl_launch(k_keys_of, grid_for(m, kBlock), kBlock, 0, c.stream, keys, by_id, m, Pkey);
            SKY_LAUNCH_CHECK();
            sort_pairs<unsigned long long>(c, Pkey, Pkey2, by_id, other, m, 64, &kcur, &order);
        }
        note_launch(c, 2);
        return order;
    };
    // value contract / Grid range checks of K1, read back with the first sync
    auto validate = [&]() {
        if (!checked) {
            checked = true;
            if (c.h_slots[S_BAD] != ~0ULL)
                invalid("parallel_skyline: tuple at position " + std::to_string(c.h_slots[S_BAD]) +
                        " has a negative or NaN value (Relation::add contract, core.cpp:14-17)");
            if (c.h_slots[S_GRIDBAD] != ~0ULL) {
                const uint64_t flat = c.h_slots[S_GRIDBAD];
                double v = 0;
                SKY_CUDA(cudaMemcpyAsync(&v, d_vals + flat, sizeof(double),
                                         cudaMemcpyDeviceToHost, c.stream));
                SKY_CUDA(cudaStreamSynchronize(c.stream));
                invalid("grid_cell: value " + std::to_string(v) + " in attribute " +
                        std::to_string(flat % d + 1) +
                        " outside [0,1]; normalize the data first");
            }
        }
        ids_sorted = (c.h_slots[S_FLAG] & 1ULL) == 0;
    };
    // the one-pass rank-grid engine over the whole undecided set (R, r)
    bool grid_used = false;
    auto run_grid = [&]() {
        uint8_t* gkeep = c.buf[B_SV].as<uint8_t>(r);
        double kms = 0;
        sky_grid_decide(c, d_vals, d, keys, tie_ids, R, r, gkeep, &kms, c.shard_rank,
                        c.shard_world);
        if (c.shard_world > 1) shard_allreduce_max(c, gkeep, r, 1);  // every row decided somewhere
        kernel_ms += kms;
        kernel_launches += 1;
        uint32_t* surv = c.buf[B_IDX0].as<uint32_t>(r);
        select_flags<uint32_t>(c, R, r, gkeep, surv, c.d_slots + S_C2);
        read_slots(c, S_C2, 1);
        const uint64_t m = c.h_slots[S_C2];
        if (m) {
            uint32_t* order = radix_order(surv, m);
            SKY_CUDA(cudaMemcpyAsync(K, order, m * sizeof(uint32_t), cudaMemcpyDeviceToDevice,
                                     c.stream));
        }
        kc = m;
        ++rounds;
        grid_used = true;
        trace_mark(c, "grid: survivors sorted");
    };
    // sort a prefix by (sum, id), decide it (K4) and append its skyline tuples
    // to K; true when the whole undecided set was this prefix
    // capacity of a device-sized round (one CTA's 16384; SKYGPU_DEV_CAP lowers
    // it so tests can drive the redo paths)
    const uint64_t dev_cap = [] {
        const char* e = getenv("SKYGPU_DEV_CAP");
        const long long v = e ? atoll(e) : 0;
        return v > 0 && v < (long long)kCTACap ? (uint64_t)v : (uint64_t)kCTACap;
    }();
    static const bool intra_chunked = [] {
        const char* e = getenv("SKYGPU_INTRA");
        return !(e && e[0] == '1');  // SKYGPU_INTRA=1: one warp per candidate
    }();
    static const bool intra_smem = [] {  // SKYGPU_INTRA=2: chunked K4 even for d <= 4
        const char* e = getenv("SKYGPU_INTRA");
        return !(e && e[0] == '2');
    }();
    // mdev (speculative final round): the prefix count lives in *mdev, m is
    // the capacity (kCTACap); nothing is read back — the caller checks the
    // count and the appended A' count (slot S_SEL2, appended after the
    // round's A' at K + kc + slots[S_C2])
    auto decide_prefix = [&](uint32_t* Pfull, uint64_t m, bool final_round,
                             const unsigned long long* mdev = nullptr) -> bool {
            // ---- sort the prefix by (sum, id)
            uint32_t* Ps = c.buf[B_IDX1].as<uint32_t>(m);
            uint32_t* order = Ps;
            if (m <= kCTACap) {
                const unsigned long long gmin = c.h_slots[S_SMIN] == ~0ULL ? 0 : c.h_slots[S_SMIN];
                const unsigned long long thr = c.h_slots[S_THR];
                const unsigned long long gmax = c.h_slots[S_SMAX];
                const unsigned long long top = thr == ~0ULL || thr - 1 > gmax ? gmax : thr - 1;
                const unsigned long long span = top > gmin ? top - gmin : 0;
                int bits = span ? 64 - __builtin_clzll(span) : 0;
                const int shift = bits > 12 ? bits - 12 : 0;  // 4096 buckets
                uint32_t* Pb = c.buf[B_GTMP1].as<uint32_t>(m);
                uint32_t* bst = c.buf[B_ORDER].as<uint32_t>(kMaxCells + 1 + kKeyBuckets + 1) +
                                (kMaxCells + 1);
                // (the in-bucket rank stays a many-CTA kernel: a bucket of
                // equal sums — C3's zero tuples — would serialise one CTA)
                // (a device-sized round: the host may not have seen the key
                // range or the threshold yet, the kernels derive the bucket
                // parameters from the slots; a final round has no threshold)
                const unsigned long long* ps = mdev ? c.d_slots : nullptr;
                const int use_thr = final_round ? 0 : 1;
                pdl_launch(k_bucket_order, 1, 1024, 0, c.stream, Pfull, (uint32_t)m, keys, gmin,
                           shift, Pb,
                                                         bst, mdev, ps, use_thr);
                SKY_LAUNCH_CHECK();
                pdl_launch(k_bucket_rank, grid_for(m, kBlock), kBlock, 0, c.stream, Pb, (uint32_t)m,
                           keys,
                                                                             tie_ids, gmin, shift, bst,
                                                                             Ps, mdev, ps, use_thr);
                SKY_LAUNCH_CHECK();
                note_launch(c, 2);
            } else {
                order = radix_order(Pfull, m);
            }
            double* Av = c.buf[B_MISC].as<double>(m * d);
            unsigned long long* Aq = qpre ? c.buf[B_AQ].as<unsigned long long>(m * 2) : nullptr;
            dispatch_d(d, [&](auto DC) {
                constexpr int D = decltype(DC)::value;
                if constexpr (D > 0)
                    pdl_launch(k_gather_q<D>, grid_for(m, kBlock), kBlock, 0, c.stream,
                        d_vals, order, m, mdev, amax, Av, Aq);
                else
                    pdl_launch(k_gather_aos, grid_for(m * d, kBlock), kBlock, 0, c.stream,
                        d_vals, d, order, m, nullptr, Av);
            });
            SKY_LAUNCH_CHECK();
            note_launch(c);
            trace_mark(c, "sky: (sync) + sort prefix + gather");

            // ---- K4: SFS inside the prefix, predecessors in sum order
            uint8_t* keep = c.buf[B_FLAGS].as<uint8_t>(m);
            const uint64_t wi = std::min<uint64_t>(m, (uint64_t)c.num_sms * 64);
            if (qpre && intra_chunked)
                SKY_CUDA(cudaMemsetAsync(keep, 1, m, c.stream));
            cudaEvent_t k0 = (mdev && final_round) ? c.ev[16] : e0;
            cudaEvent_t k1 = (mdev && final_round) ? c.ev[17] : e1;
            SKY_CUDA(cudaEventRecord(k0, c.stream));
            dispatch_d(d, [&](auto DC) {
                constexpr int D = decltype(DC)::value;
                const unsigned grid = (unsigned)((wi * 32 + kBlock - 1) / kBlock);
                if constexpr (D > 0 && D <= 8) {
                    constexpr uint32_t kWq = QW<D>::W;
                    if (intra_chunked && intra_smem && m <= kIntraSmemMax) {
                        const uint32_t scap =
                            (uint32_t)std::min<uint64_t>(m * kWq, kIntraSmemMax);
                        static bool attr = false;
                        if (!attr) {
                            SKY_CUDA(cudaFuncSetAttribute(
                                k_sfs_intra_smem<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)(kIntraSmemMax * sizeof(unsigned long long))));
                            attr = true;
                        }
                        pdl_launch(k_sfs_intra_smem<D>, c.num_sms, 1024,
                                   scap * sizeof(unsigned long long), c.stream, Av, Aq,
                                   (uint32_t)m, keep, c.d_slots + S_TESTS_SKY, (uint32_t)m, mdev,
                                   scap);
                        return;
                    }
                }
                if constexpr (D > 0) {
                    if (intra_chunked)
                        pdl_launch(k_sfs_intra_chunked<D>, c.num_sms * 8, kBlock, 0, c.stream,
                            Av, Aq, (uint32_t)m, keep, c.d_slots + S_TESTS_SKY, (uint32_t)m, mdev);
                    else
                        pdl_launch(k_sfs_intra_q<D>, grid, kBlock, 0, c.stream, Av, Aq, (uint32_t)m,
                                   keep,
                                                                        c.d_slots + S_TESTS_SKY);
                } else
                    pdl_launch(k_sfs_intra_sorted<D>, grid, kBlock, 0, c.stream,
                        Av, (uint32_t)m, d, keep, c.d_slots + S_TESTS_SKY);
            });
            SKY_CUDA(cudaEventRecord(k1, c.stream));
            SKY_LAUNCH_CHECK();
            note_launch(c);
            trace_mark(c, "sky: K4 intra kernel");
            // A' in (sum, id) order appended to K; its count lands in S_C2
            if (mdev) {  // final: count in S_SEL2, after the round's A' (S_C2)
                pdl_launch(k_cta_select, 1, 1024, 0, c.stream,
                    order, nullptr, keep, (uint32_t)m, K + kc, nullptr,
                    c.d_slots + (final_round ? S_SEL2 : S_C2), mdev,
                    final_round ? c.d_slots + S_C2 : nullptr);
                SKY_LAUNCH_CHECK();
                note_launch(c);
                return false;
            }
            if (m <= kCTACap) {
                pdl_launch(k_cta_select, 1, 1024, 0, c.stream, order, nullptr, keep, (uint32_t)m,
                           K + kc,
                           nullptr, c.d_slots + S_C2, nullptr, nullptr);
                SKY_LAUNCH_CHECK();
                note_launch(c);
            } else {
                select_flags<uint32_t>(c, order, m, keep, K + kc, c.d_slots + S_C2);
            }
            ++rounds;
            kernel_launches += 1;
            if (final_round || m == r) {
                read_slots(c, S_C2, 1);
                float ms = 0;
                SKY_CUDA(cudaEventElapsedTime(&ms, e0, e1));
                kernel_ms += ms;
                kc += c.h_slots[S_C2];
                return true;
            }
            return false;
    };
    // K5 over the undecided list (R, r) against A' = alist[0..m) (positions in
    // (sum, id) order, count also in slot S_C2); seeded: A' need not precede
    // the candidates (precedence checked per hit).  Survivors replace (R, r);
    // returns |A'|.
    struct AScan {
        uint32_t* seg = nullptr;
        int mcell = 0, qk = 0;
        const uint32_t* psrc = nullptr;
        double* Pv = nullptr;
        unsigned long long* Pq = nullptr;
        uint64_t m = 0;
    };
    // A' = alist[0..m) (count also in slot S_C2) regrouped by cells, values
    // and quantised codes gathered (codes scaled by `scale`, the per-attribute
    // maxima every candidate code of the same K5 must use)
    auto prep_aprime = [&](const uint32_t* alist, uint64_t m,
                           const unsigned long long* scale) -> AScan {
        // ---- K5: filter the rest against A', A' regrouped (one-CTA counting
        // sort) by the quantile grid (exact cell pruning, default) or by the
        // plan's partition (scan order only, SKYGPU_PLAN_CELLS=1)
        // (the quantile grid is opt-in, SKYGPU_QGRID=1: its exact pruning pays
        // only when candidates survive; measured slower on C2/C4)
        static const bool qgrid_env = [] {
            const char* e = getenv("SKYGPU_QGRID");
            return e && e[0] == '1';
        }();
        AScan A;
        A.m = m;
        uint32_t ncells = 1;
        int mcell = 0, qk = 0;
        if (m <= kCTACap && qpre && qgrid_env) {
            // k bins per attribute: ~32 tuples per cell, k^d <= kMaxCells
            int k = (int)std::floor(std::pow(std::max(1.0, (double)m / 32.0), 1.0 / d) + 1e-9);
            k = std::max(2, std::min(k, kQMaxBins));
            while (k > 2 && std::pow((double)k, d) > kMaxCells) --k;
            if (std::pow((double)k, d) <= kMaxCells) {
                qk = k;
                ncells = 1;
                for (int j = 0; j < d; ++j) ncells *= (uint32_t)k;
                mcell = (kCellQuantile << 16) | k;
                double* bounds = c.buf[B_PROJ].as<double>(kMaxDims * kQMaxBins);
                pdl_launch(k_qgrid_bounds, d, 1024, 0, c.stream, d_vals, d, alist, c.d_slots + S_C2,
                           k,
                                                         bounds);
                SKY_LAUNCH_CHECK();
                SKY_CUDA(cudaMemcpyToSymbolAsync(c_qbounds, bounds,
                                                 sizeof(double) * kMaxDims * kQMaxBins, 0,
                                                 cudaMemcpyDeviceToDevice, c.stream));
                note_launch(c);
            }
        }
        if (!qk && m <= kCTACap) mcell = scan_cell_spec(plan, m, d, qpre, &ncells);
        uint32_t* seg = nullptr;
        const uint32_t* psrc = alist;
        if (ncells > 1) {
            uint32_t* Alist = c.buf[B_GTMP1].as<uint32_t>(m);
            uint32_t* Akey = c.buf[B_GTMP0].as<uint32_t>(m);
            static const bool one_cta = [] {  // SKYGPU_CELL_ORDER=1: the one-CTA kernel
                const char* e = getenv("SKYGPU_CELL_ORDER");
                return e && e[0] == '1';
            }();
            if (one_cta) {
                dispatch_d(d, [&](auto DC) {
                    constexpr int D = decltype(DC)::value;
                    pdl_launch(k_cell_order<D>, 1, 1024, 0, c.stream, d_vals, d, alist,
                               (uint32_t)m, c.d_slots + S_C2, mcell, ncells,
                               qpre ? scale : nullptr, Alist, Akey, seg_table);
                });
                note_launch(c, 1);
            } else {
                // the histogram is zeroed once per call, then kept zeroed
                // between rounds by k_cell_seg
                uint32_t* hist = c.buf[B_CHIST].as<uint32_t>(kMaxCells);
                uint32_t* curs = c.buf[B_CCUR].as<uint32_t>(kMaxCells);
                if (!c.chist_zeroed) {
                    SKY_CUDA(cudaMemsetAsync(hist, 0, kMaxCells * sizeof(uint32_t), c.stream));
                    c.chist_zeroed = true;
                }
                const unsigned gm = grid_for(m, kBlock);
                dispatch_d(d, [&](auto DC) {
                    constexpr int D = decltype(DC)::value;
                    pdl_launch(k_cell_hist<D>, gm, kBlock, 0, c.stream, d_vals, d, alist,
                               (uint32_t)m, c.d_slots + S_C2, mcell, qpre ? scale : nullptr,
                               Akey, hist);
                });
                pdl_launch(k_cell_seg, 1, 1024, 0, c.stream, hist, ncells, c.d_slots + S_C2,
                           (uint32_t)m, seg_table, curs);
                pdl_launch(k_cell_scatter_a, gm, kBlock, 0, c.stream, alist, (uint32_t)m,
                           c.d_slots + S_C2, Akey, curs, Alist);
                note_launch(c, 3);
            }
            SKY_LAUNCH_CHECK();
            seg = seg_table;
            psrc = Alist;
        }
        double* Pv = c.buf[B_CSUM].as<double>(m * d);
        unsigned long long* Pq = qpre ? c.buf[B_PQ].as<unsigned long long>(m * 2) : nullptr;
        dispatch_d(d, [&](auto DC) {
            constexpr int D = decltype(DC)::value;
            if constexpr (D > 0)
                pdl_launch(k_gather_q<D>, grid_for(m, kBlock), kBlock, 0, c.stream,
                    d_vals, psrc, m, c.d_slots + S_C2, scale, Pv, Pq);
            else
                pdl_launch(k_gather_aos, grid_for(m * d, kBlock), kBlock, 0, c.stream,
                    d_vals, d, psrc, m, c.d_slots + S_C2, Pv);
        });
        SKY_LAUNCH_CHECK();
        note_launch(c);
        A.seg = seg;
        A.mcell = mcell;
        A.qk = qk;
        A.psrc = psrc;
        A.Pv = Pv;
        A.Pq = Pq;
        return A;
    };
    // K5 launch: candidates Rl[0..rl) (nullptr: positions 0..rl), keep flags
    // into fkeep[0..rl); seeded = A' need not precede them (checked per hit)
    auto launch_k5 = [&](const AScan& A, const uint32_t* Rl, uint64_t rl, uint8_t* fkeep,
                         bool seeded, const unsigned long long* scale) {
        // comparators each lane tests alone (phase A) before the warp-wide scan
        static const uint32_t solo = [] {
            const char* e = getenv("SKYGPU_SOLO");
            const int v = e ? atoi(e) : 0;
            return v > 0 ? (uint32_t)v : 16u;
        }();
        const uint32_t bsf = batch_size(c, rl);
        const uint64_t wf = std::min<uint64_t>((rl + bsf - 1) / bsf, (uint64_t)c.num_sms * 64);
        dispatch_d(d, [&](auto DC) {
            constexpr int D = decltype(DC)::value;
            const unsigned grid = (unsigned)((wf * 32 + kBlock - 1) / kBlock);
            if constexpr (D > 0)
                pdl_launch(k_sfs_filter_q<D>, grid, kBlock, 0, c.stream,
                    d_vals, keys, Rl, (uint32_t)rl, A.Pv, A.Pq, (uint32_t)A.m, A.seg, A.mcell,
                    A.qk, scale, c.d_slots, fkeep, c.d_slots + S_TESTS_SKY, bsf,
                    seeded ? A.psrc : nullptr, tie_ids, solo);
            else
                pdl_launch(k_sfs_filter_cells<D>, grid, kBlock, 0, c.stream,
                    d_vals, d, keys, Rl, (uint32_t)rl, A.Pv, (uint32_t)A.m, A.seg, A.mcell,
                    c.d_slots, fkeep, c.d_slots + S_TESTS_SKY, bsf);
        });
        SKY_LAUNCH_CHECK();
        note_launch(c);
    };
    // spec_final: the final round over the survivors is queued at once,
    // sized on the device (decide_prefix with mdev = slots[S_C3]); *spec_done
    // tells whether it applied (survivors <= kCTACap) — one host round trip
    // for the round and the final round instead of two
    auto filter_against = [&](const uint32_t* alist, uint64_t m, bool seeded,
                              bool spec_final = false, bool* spec_done = nullptr) -> uint64_t {
        const AScan A = prep_aprime(alist, m, amax);
        uint8_t* fkeep = c.buf[B_SV].as<uint8_t>(r);
        trace_mark(c, "sky: select A' + segments + gather Pv");
        SKY_CUDA(cudaEventRecord(e2, c.stream));
        issue_late_ids(c);  // the deferred ids copy overlaps K5
        launch_k5(A, R, r, fkeep, seeded, amax);
        SKY_CUDA(cudaEventRecord(e3, c.stream));
        trace_mark(c, "sky: K5 filter kernel");
        select_flags<uint32_t>(c, R, r, fkeep, Rnext, c.d_slots + S_C3);
        trace_mark(c, "sky: select survivors");
        kernel_launches += 1;
        if (spec_final) {
            c.h_slots[S_THR] = ~0ULL;  // the final round: no threshold
            decide_prefix(Rnext, dev_cap, true, c.d_slots + S_C3);
            trace_mark(c, "sky: speculative final round queued");
            read_slots(c, S_BAD, 12);  // S_BAD .. S_GATE (a device-sized round validates here)
            const uint64_t sv = c.h_slots[S_C3];
            *spec_done = sv > 0 && sv <= dev_cap && !c.h_slots[S_GATE];
        } else {
            read_slots(c, S_C2, 3);  // S_C2 (A'), S_C3 (survivors), S_GATE
        }
        float ms = 0;
        SKY_CUDA(cudaEventElapsedTime(&ms, e2, e3));
        kernel_ms += ms;
        r = c.h_slots[S_C3];
        R = Rnext;
        Rnext = (Rnext == Rbuf1) ? Rbuf0 : Rbuf1;
        return (uint64_t)c.h_slots[S_C2];
    };
    if (feed) {
        // every chunk (the head included) scored as it lands and filtered
        // against the seed — the skyline of the head's first prefix — by the
        // seeded K5 (precedence checked per hit: a dominating predecessor
        // rules a tuple out whether or not it is a skyline tuple itself).
        // Survivors (the seed included) form the undecided list of the rounds.
        pdl_launch(k_seed_slots, 1, 32, 0, c.stream, c.d_slots, nseed);
        SKY_LAUNCH_CHECK();
        const AScan A = prep_aprime(seed, nseed, scale_snap);
        uint8_t* flags = c.buf[B_FLAGS].as<uint8_t>(n);
        uint32_t* iota = c.buf[B_IOTA].as<uint32_t>(n);
        pdl_launch(k_iota, grid_for(n, kBlock), kBlock, 0, c.stream, iota, n);
        SKY_LAUNCH_CHECK();
        note_launch(c, 1);
        for (int ch = 0; ch < feed->nchunks; ++ch) {
            const uint64_t lo = feed->bound[ch], hi = feed->bound[ch + 1];
            if (ch > 0) SKY_CUDA(cudaStreamWaitEvent(c.stream, feed->ready[ch], 0));
            dispatch_d(d, [&](auto DC) {
                constexpr int D = decltype(DC)::value;
                pdl_launch(k_score<D>, grid_for(hi - lo, kBlock, c.num_sms * 8), kBlock, 0,
                           c.stream,
                    d_vals + lo * d, hi - lo, d, keys + lo, c.d_slots, amax, lo, nullptr, nullptr);
            });
            if (!ids_late) {  // (late ids: checked whole, once they are in)
                const uint64_t c0 = ch ? lo - 1 : 0;  // pair (lo-1, lo) spans the boundary
                pdl_launch(k_ids_check, grid_for(hi - c0, kBlock), kBlock, 0, c.stream,
                    d_ids + c0, hi - c0, c.d_slots, (int)S_FLAG);
                note_launch(c);
            }
            SKY_LAUNCH_CHECK();
            note_launch(c);
            launch_k5(A, iota + lo, hi - lo, flags + lo, true, scale_snap);
        }
        trace_mark(c, "sky: streamed chunks filtered");
        select_flags<uint32_t>(c, nullptr, n, flags, Rbuf0, c.d_slots + S_C3);
        read_slots(c, S_BAD, 11);
        validate();
        R = Rbuf0;
        r = c.h_slots[S_C3];
        st.tuples_into_parallel = r;
        if (c.trace)
            fprintf(stderr, "[skygpu trace] streamed: seed %llu, survivors %llu of %llu\n",
                    (unsigned long long)nseed, (unsigned long long)r, (unsigned long long)n);
    }
    // the rank grid at once: asked for, or the streamed head's first prefix
    // already showed a large skyline (no first round to repeat on all n)
    if ((sky_engine == SKYGPU_SKY_GRID || (head_grid && sky_engine == 0)) && r > 0 &&
        sky_grid_bins(r, d)) {
        read_slots(c, S_BAD, 11);
        validate();
        run_grid();
        r = 0;
    }
    while (r > 0) {
        // final round: the whole (already ordered) undecided list is the
        // prefix — no threshold, no selection, no host synchronisation
        if (checked && R && r <= kFinal) {
            const uint64_t m = r;
            c.h_slots[S_THR] = ~0ULL;
            trace_mark(c, "sky: final round");
            decide_prefix(R, m, /*final_round=*/true);
            break;
        }
        // ---- K2: sampled threshold, K3: ordered prefix selection
        const uint64_t w = r <= kFinal ? r : want;
        if (!fused_first)
            pdl_launch(k_sample_threshold, 1, 1024, 0, c.stream, keys, R, r, w, c.d_slots,
                       (const double*)nullptr, 0);
        SKY_LAUNCH_CHECK();
        uint32_t* Pfull = c.buf[B_IDX0].as<uint32_t>(r);
        if (!fused_first) {
            reset_counts(c);
            trace_mark(c, "sky: score + sample threshold");
            select_if(c, R, r, BelowThreshold{keys, c.d_slots + S_THR}, Pfull, c.d_slots + S_C1);
            note_launch(c, 1);
            trace_mark(c, "sky: select prefix");
        }
        const bool unordered_prefix = fused_first;
        fused_first = false;
        // the round sized on the device — no host round trip before K5: the
        // prefix sort, K4, K5, the survivor selection and the ride-along final
        // round read the prefix count from its slot; the host checks it with
        // the round's one read-back and, in the rare case the prefix did not
        // fit one CTA (every sized kernel then returned at once), redoes the
        // round the synchronous way
        const bool gate_cond = rounds == 0 && (sky_engine & ~kSkyAbortIfLarge) == 0 &&
                               r >= kGridMin && sky_grid_bins(r, d);
        const bool spec_ok = qpre && intra_chunked && !getenv("SKYGPU_NO_SPEC_FINAL");
        if (spec_ok && !(sky_engine & kSkyFirstPrefix) && w <= kCTACap / 2 && r > w &&
            !getenv("SKYGPU_NO_DEV_ROUND")) {
            uint32_t* const Rin = R;
            const uint64_t rin = r;
            decide_prefix(Pfull, dev_cap, false, c.d_slots + S_C1);
            if (gate_cond) {
                pdl_launch(k_grid_gate, 1, 32, 0, c.stream, c.d_slots, 0);
                SKY_LAUNCH_CHECK();
                note_launch(c);
            }
            bool spec_done = false;
            const uint64_t a = filter_against(K + kc, dev_cap, false, true, &spec_done);
            validate();
            const uint64_t m = c.h_slots[S_C1];
            if (m == 0) throw Error(SKYGPU_ERUNTIME, "skyline: empty prefix (internal)");
            if (m <= dev_cap) {
                ++rounds;  // (decide_prefix's own count: the round ran)
                kernel_launches += 1;
                if (c.trace)
                    fprintf(stderr, "[skygpu trace] round %d (device-sized): prefix %llu, A' %llu, "
                            "survivors %llu\n", rounds, (unsigned long long)m,
                            (unsigned long long)a, (unsigned long long)r);
                if (gate_cond && c.h_slots[S_GATE]) {
                    if (sky_engine & kSkyAbortIfLarge) {
                        out.aborted = true;
                        return out;
                    }
                    run_grid();
                    break;
                }
                float ms4 = 0;
                SKY_CUDA(cudaEventElapsedTime(&ms4, e0, e1));
                kernel_ms += ms4;
                kc += a;
                if (spec_done) {
                    SKY_CUDA(cudaEventElapsedTime(&ms4, c.ev[16], c.ev[17]));
                    kernel_ms += ms4;
                    kc += c.h_slots[S_SEL2];
                    ++rounds;
                    kernel_launches += 1;
                    break;
                }
                if (a * 2 > m) want = std::min(want * 4, kMaxPrefix);
                continue;
            }
            // the prefix did not fit: back to the round's input, synchronous
            R = Rin;
            r = rin;
            Rnext = (Rin == Rbuf1) ? Rbuf0 : Rbuf1;
            trace_mark(c, "sky: device-sized round missed, synchronous redo");
        } else {
            read_slots(c, S_BAD, 11);
            validate();
        }
        if (unordered_prefix) {  // the synchronous path sorts stably: re-select in order
            reset_counts(c);
            select_if(c, R, r, BelowThreshold{keys, c.d_slots + S_THR}, Pfull, c.d_slots + S_C1);
            note_launch(c, 1);
            read_slots(c, S_BAD, 11);
        }
        const uint64_t m = c.h_slots[S_C1];
        if (m == 0) throw Error(SKYGPU_ERUNTIME, "skyline: empty prefix (internal)");

        if (decide_prefix(Pfull, m, false)) break;
        if (sky_engine & kSkyFirstPrefix) {  // the streamed head's seed
            read_slots(c, S_C2, 1);
            const uint64_t a = c.h_slots[S_C2];
            if ((sky_engine & kSkyAbortIfLarge) && r >= kGridMin && a * 4 > m * 3 &&
                sky_grid_bins(r, d)) {
                out.aborted = true;
                return out;
            }
            kc += a;
            break;
        }
        // large skyline ahead (most of the first prefix survived): decide
        // everything at once with the rank-grid engine instead of filtering.
        // Decided on the device (no extra host round trip): the gate makes
        // K5 keep every candidate, the host switches after K5's sync.
        const bool gate = rounds == 1 && gate_cond;
        if (gate) {
            pdl_launch(k_grid_gate, 1, 32, 0, c.stream, c.d_slots, m);
            SKY_LAUNCH_CHECK();
            note_launch(c);
        }

        // the final round rides along when the survivors fit one CTA
        // (checked on the device; the host only sees the outcome)
        bool spec_done = false;
        const uint64_t a = filter_against(K + kc, m, false, spec_ok, &spec_done);  // synchronises
        if (c.trace)
            fprintf(stderr, "[skygpu trace] round %d: prefix %llu, A' %llu, survivors %llu\n",
                    rounds, (unsigned long long)m, (unsigned long long)a, (unsigned long long)r);
        if (gate && c.h_slots[S_GATE]) {
            if (sky_engine & kSkyAbortIfLarge) {
                out.aborted = true;
                return out;
            }
            run_grid();
            break;
        }
        float ms4 = 0;
        SKY_CUDA(cudaEventElapsedTime(&ms4, e0, e1));
        kernel_ms += ms4;
        kc += a;
        if (spec_done) {  // the survivors' final round already ran
            SKY_CUDA(cudaEventElapsedTime(&ms4, c.ev[16], c.ev[17]));
            kernel_ms += ms4;
            kc += c.h_slots[S_SEL2];
            ++rounds;
            kernel_launches += 1;
            break;
        }
        if (a * 2 > m) want = std::min(want * 4, kMaxPrefix);
    }
    st.sfs_rounds = rounds;
    st.sky_engine = grid_used ? SKYGPU_SKY_GRID : SKYGPU_SKY_ROUNDS;
    st.tuples_into_final = into_final != ~0ULL ? into_final : kc;
    st.ms_sky_kernel += kernel_ms;
    st.sky_kernel_launches += kernel_launches;

    // K holds the skyline in the reference's output order, (sum, id): each
    // round's A' is in that order and rounds advance through the order
    out.S = kc;
    out.d_inpos = K;
    out.d_ids = c.buf[B_SKYID].as<int64_t>(kc);
    out.d_skyv = c.buf[B_SKYV].as<double>(kc * d);
    out.d_pos64 = c.buf[B_OUTPOS].as<uint64_t>(kc ? kc : 1);
    ensure_ids();
    if (kc) {
        trace_mark(c, "sky: rounds done (sync)");
        dispatch_d(d, [&](auto DC) {
            constexpr int D = decltype(DC)::value;
            pdl_launch(k_emit_skyline<D>, grid_for(kc, kBlock), kBlock, 0, c.stream, K, kc,
                       d_vals, d, (ids_late && !ids_waited) ? nullptr : d_ids, out.d_ids,
                       out.d_skyv, out.d_pos64);
        });
        SKY_LAUNCH_CHECK();
        note_launch(c);
    }
    st.skyline_size = kc;
    return out;
}

}  // namespace skygpu
