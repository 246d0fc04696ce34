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
// GPU algorithm — prefix rounds (no full sort of the relation):
//   K1 score     left-to-right __dadd_rn sum -> key bits, min/max sum, contract
//                checks (one HBM pass over the relation)
//   K2 histogram of the undecided tuples' sums -> threshold T such that about
//                k tuples have sum < T.  {sum < T} is a PREFIX of the (sum, id)
//                order, so it can be decided on its own:
//   K3 select    the prefix (warp-aggregated compaction)
//   -- CUB radix sort of the prefix by (sum, id)  (k items, not n)
//   K4 intra     warp-per-candidate SFS inside the prefix (warp-ballot exit)
//                -> new skyline tuples A' (appended to the output in order)
//   K5 filter    every other undecided tuple against A' (warp-per-candidate,
//                coalesced float64 SoA comparator loads, ballot exit); the
//                survivors become the next round's undecided set.
// Because the lowest-sum tuples are the strongest dominators, one round of
// k = 16384 leaves ~10^3 survivors out of 10^6 on the benchmark data; large
// skylines (ANT d=7) grow k up to 65536 per round.
#include <cub/cub.cuh>

#include "sky_common.cuh"

namespace skygpu {

namespace {

constexpr int kBlock = 256;
constexpr int kHistBins = 4096;

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

__device__ __forceinline__ double slot_double(const unsigned long long* slots, int i) {
    return __longlong_as_double((long long)slots[i]);
}

// K1 (core.cpp:21-23): sum with __dadd_rn from +0.0, key = ord bits (sums
// are never -0.0: 0.0 + -0.0 = +0.0), min/max of the sums, value contract.
__global__ void k_score(const double* __restrict__ v, uint64_t n, int d,
                        unsigned long long* __restrict__ key,
                        unsigned long long* __restrict__ slots) {
    unsigned long long mn = ~0ULL, mx = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        bool bad = false;
        for (int k = 0; k < d; ++k) {
            double x = v[i * d + k];
            bad |= !(x >= 0.0);  // negative or NaN
            s = __dadd_rn(s, x);
        }
        const unsigned long long b = ord_bits(s);
        key[i] = b;
        mn = b < mn ? b : mn;
        mx = b > mx ? b : mx;
        if (bad) atomicMin(&slots[S_BAD], static_cast<unsigned long long>(i));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        unsigned long long a = __shfl_down_sync(0xffffffffu, mn, o);
        unsigned long long b = __shfl_down_sync(0xffffffffu, mx, o);
        mn = a < mn ? a : mn;
        mx = b > mx ? b : mx;
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(&slots[S_SMIN], mn);
        atomicMax(&slots[S_SMAX], mx);
    }
}

__global__ void k_ids_check(const int64_t* __restrict__ ids, uint64_t n,
                            unsigned long long* __restrict__ slots) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i + 1 < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        if (ids[i] >= ids[i + 1]) atomicOr(&slots[S_FLAG], 1ULL);
}

// Grid strategy contract (partition.cpp:88-95): values must lie in [0,1];
// the first offending (tuple, attribute) in input order is reported.
__global__ void k_grid_range(const double* __restrict__ v, uint64_t total,
                             unsigned long long* __restrict__ slots) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
         i += (uint64_t)gridDim.x * blockDim.x) {
        double x = v[i];
        if (x < 0.0 || x > 1.0) atomicMin(&slots[S_GRIDBAD], static_cast<unsigned long long>(i));
    }
}

// min / max sum of the undecided set (rounds >= 2)
__global__ void k_range(const unsigned long long* __restrict__ key, const uint32_t* __restrict__ R,
                        uint64_t r, unsigned long long* __restrict__ slots) {
    unsigned long long mn = ~0ULL, mx = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < r;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const unsigned long long b = key[R[i]];
        mn = b < mn ? b : mn;
        mx = b > mx ? b : mx;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        unsigned long long a = __shfl_down_sync(0xffffffffu, mn, o);
        unsigned long long b = __shfl_down_sync(0xffffffffu, mx, o);
        mn = a < mn ? a : mn;
        mx = b > mx ? b : mx;
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(&slots[S_SMIN], mn);
        atomicMax(&slots[S_SMAX], mx);
    }
}

// K2a: histogram of the undecided tuples' sums over [min, max]
__global__ void k_hist(const unsigned long long* __restrict__ key, const uint32_t* __restrict__ R,
                       uint64_t r, const unsigned long long* __restrict__ slots,
                       unsigned* __restrict__ hist) {
    __shared__ unsigned h[kHistBins];
    for (int b = threadIdx.x; b < kHistBins; b += blockDim.x) h[b] = 0;
    __syncthreads();
    const double lo = slot_double(slots, S_SMIN), hi = slot_double(slots, S_SMAX);
    const double scale = hi > lo ? (double)kHistBins / (hi - lo) : 0.0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < r;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t t = R ? R[i] : (uint32_t)i;
        const double s = __longlong_as_double((long long)key[t]);
        int b = (int)((s - lo) * scale);
        b = b < 0 ? 0 : (b >= kHistBins ? kHistBins - 1 : b);
        atomicAdd(&h[b], 1u);
    }
    __syncthreads();
    for (int b = threadIdx.x; b < kHistBins; b += blockDim.x)
        if (h[b]) atomicAdd(&hist[b], h[b]);
}

// K2b: threshold T with about `want` undecided sums below it (one block).
// Progress is guaranteed: T > min sum.  want >= r selects everything.
__global__ void k_threshold(const unsigned* __restrict__ hist, uint64_t r, uint64_t want,
                            unsigned long long* __restrict__ slots) {
    __shared__ unsigned long long part[1024];
    const int per = kHistBins / 1024;
    unsigned long long local = 0;
    for (int k = 0; k < per; ++k) local += hist[threadIdx.x * per + k];
    part[threadIdx.x] = local;
    __syncthreads();
    if (threadIdx.x == 0) {
        const double lo = slot_double(slots, S_SMIN), hi = slot_double(slots, S_SMAX);
        double T = __longlong_as_double(0x7FF0000000000000LL);  // +inf: take all
        if (want < r && hi > lo) {
            unsigned long long cum = 0;
            int bin = kHistBins - 1;
            for (int t = 0; t < 1024; ++t) {
                if (cum + part[t] >= want) {
                    for (int k = 0; k < per; ++k) {
                        cum += hist[t * per + k];
                        if (cum >= want) {
                            bin = t * per + k;
                            break;
                        }
                    }
                    break;
                }
                cum += part[t];
            }
            T = lo + (double)(bin + 1) * ((hi - lo) / (double)kHistBins);
            const double nxt = __longlong_as_double((long long)(slots[S_SMIN] + 1));
            if (T < nxt) T = nxt;  // at least the minimum is selected
            if (bin == kHistBins - 1) T = __longlong_as_double(0x7FF0000000000000LL);
        }
        slots[S_THR] = (unsigned long long)__double_as_longlong(T);
    }
}

// warp-aggregated append of `pred` items; returns this lane's slot
__device__ __forceinline__ uint32_t warp_append(bool pred, unsigned long long* counter) {
    const unsigned mask = __ballot_sync(0xffffffffu, pred);
    const uint32_t lane = threadIdx.x & 31;
    unsigned long long base = 0;
    if (mask) {
        const int leader = __ffs(mask) - 1;
        if ((int)lane == leader) base = atomicAdd(counter, (unsigned long long)__popc(mask));
        base = __shfl_sync(0xffffffffu, base, leader);
    }
    return (uint32_t)(base + __popc(mask & ((1u << lane) - 1)));
}

// K3 predicate: the prefix {sum < T} of the undecided set (selected with an
// order-preserving CUB DeviceSelect so ties in the sum keep index order)
struct BelowThreshold {
    const unsigned long long* key;
    const unsigned long long* thr;
    __device__ __forceinline__ bool operator()(uint32_t t) const {
        return __longlong_as_double((long long)key[t]) < __longlong_as_double((long long)*thr);
    }
};

__global__ void k_id_keys(const int64_t* __restrict__ ids, const uint32_t* __restrict__ list,
                          uint64_t m, unsigned long long* __restrict__ out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
         i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = static_cast<unsigned long long>(ids[list[i]]) ^ 0x8000000000000000ULL;
}

__global__ void k_keys_of(const unsigned long long* __restrict__ key,
                          const uint32_t* __restrict__ list, uint64_t m,
                          unsigned long long* __restrict__ out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
         i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = key[list[i]];
}

// compact SoA copy [d][m] of the tuples list[0..m) from the AoS input; the
// count is read from device memory when `count` is given (no host sync)
__global__ void k_gather_aos(const double* __restrict__ v, int d, const uint32_t* __restrict__ list,
                             uint64_t m, const unsigned long long* __restrict__ count,
                             double* __restrict__ out) {
    const uint64_t mm = count ? *count : m;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < mm * d;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t k = i / d;
        const int a = (int)(i - k * d);
        out[(uint64_t)a * m + k] = v[(uint64_t)list[k] * d + a];
    }
}

// Representative filter (partition.cpp:287-302): a tuple dominated by any
// representative never enters the local skylines.  reps: AoS [n_reps][d].
template <int D>
__global__ void k_rep_filter(const double* __restrict__ v, uint64_t n, int d,
                             const double* __restrict__ reps, uint32_t n_reps,
                             uint8_t* __restrict__ keep, unsigned long long* __restrict__ tests) {
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
        keep[p] = alive;
    }
    add_count(tests, cnt);
}

// K4: warp-per-candidate SFS inside the sorted prefix Av[d][m]: candidate i
// tests its predecessors 0..i-1, 32 per iteration, leaving at the first
// non-zero ballot (north_star (a): warp-ballot early exit).
template <int D>
__global__ void __launch_bounds__(kBlock)
k_sfs_intra_warp(const double* __restrict__ Av, uint32_t m, int d, uint8_t* __restrict__ keep,
                 unsigned long long* __restrict__ tests) {
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

// K5: every undecided tuple outside the prefix against the new skyline
// tuples Pv[d][cap] (np = *np_dev, all of which precede it in (sum, id)
// order); keep[i] = 1 for survivors (compacted in order by the caller).
template <int D>
__global__ void __launch_bounds__(kBlock)
k_sfs_filter_warp(const double* __restrict__ v, int d, const unsigned long long* __restrict__ key,
                  const uint32_t* __restrict__ R, uint64_t r, const double* __restrict__ Pv,
                  uint64_t pcap, unsigned long long* __restrict__ slots,
                  uint8_t* __restrict__ keep, unsigned long long* __restrict__ tests) {
    constexpr int DM = D > 0 ? D : kMaxDims;
    const int dd = D > 0 ? D : d;
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const double T = slot_double(slots, S_THR);
    const uint32_t np = (uint32_t)slots[S_C2];
    unsigned long long cnt = 0;
    for (uint64_t i = warp; i < r; i += nwarps) {
        const uint32_t p = R ? R[i] : (uint32_t)i;
        if (__longlong_as_double((long long)key[p]) < T) {  // in the prefix: decided
            if (lane == 0) keep[i] = 0;
            continue;
        }
        double t[DM];
#pragma unroll
        for (int k = 0; k < DM; ++k)
            if (k < dd) t[k] = v[(uint64_t)p * dd + k];
        bool dominated = false;
        for (uint32_t j0 = 0; j0 < np; j0 += 32) {
            const uint32_t j = j0 + lane;
            bool hit = false;
            if (j < np) {
                double s[DM];
#pragma unroll
                for (int k = 0; k < DM; ++k)
                    if (k < dd) s[k] = Pv[(uint64_t)k * pcap + j];
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

// Direction cell of a tuple: a grid over its first d-1 normalised
// coordinates u_j = t_j / sum(t) (a cheap stand-in for the paper's angular
// coordinates, partition.cpp:139-174).  A dominator s of t lies in the
// orthant below t; on large-skyline data (tuples near a hyperplane) that
// means a nearby direction, so scanning t's own cell first finds it early.
// Only the scan ORDER depends on cells — results never do.
template <int DM>
__device__ __forceinline__ uint32_t direction_cell(const double* t, int dd, int m) {
    if (dd < 2 || m <= 1) return 0;
    double s = 0.0;
    for (int k = 0; k < DM; ++k)
        if (k < dd) s += t[k];
    if (!(s > 0.0)) return 0;
    const double inv = (double)m / s;
    uint32_t cell = 0;
    for (int k = DM - 2; k >= 0; --k) {
        if (k >= dd - 1) continue;
        int b = (int)(t[k] * inv);
        b = b < 0 ? 0 : (b >= m ? m - 1 : b);
        cell = cell * (uint32_t)m + (uint32_t)b;
    }
    return cell;
}

// cell keys of the prefix in sorted order; non-skyline entries sort last
template <int D>
__global__ void k_prefix_cells(const double* __restrict__ Av, uint32_t mcount, int d,
                               const uint8_t* __restrict__ keep, int m,
                               uint32_t* __restrict__ ckey) {
    constexpr int DM = D > 0 ? D : kMaxDims;
    const int dd = D > 0 ? D : d;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < mcount;
         i += gridDim.x * blockDim.x) {
        double t[DM];
#pragma unroll
        for (int k = 0; k < DM; ++k)
            if (k < dd) t[k] = Av[(uint64_t)k * mcount + i];
        ckey[i] = keep[i] ? direction_cell<DM>(t, dd, m) : 0xFFFFFFFFu;
    }
}

// seg[c] = first position of cell >= c in the cell-sorted comparator list
__global__ void k_cell_segments(const uint32_t* __restrict__ ckey, uint32_t mcount,
                                uint32_t ncells, uint32_t* __restrict__ seg) {
    for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c <= ncells;
         c += gridDim.x * blockDim.x) {
        uint32_t lo = 0, hi = mcount;
        while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (ckey[mid] < c) lo = mid + 1;
            else hi = mid;
        }
        seg[c] = lo;
    }
}

// K5 (v2): 32 candidates are loaded per warp at once (lane-parallel,
// coalesced), then decided one after another with the whole warp scanning
// the comparators 32 at a time, starting in the candidate's own direction
// cell and wrapping around; ballot exit at the first dominator.
template <int D>
__global__ void __launch_bounds__(kBlock)
k_sfs_filter_cells(const double* __restrict__ v, int d, const unsigned long long* __restrict__ key,
                   const uint32_t* __restrict__ R, uint32_t r, const double* __restrict__ Pv,
                   uint32_t pcap, const uint32_t* __restrict__ seg, int m,
                   const unsigned long long* __restrict__ slots, uint8_t* __restrict__ keep,
                   unsigned long long* __restrict__ tests) {
    constexpr int DM = D > 0 ? D : kMaxDims;
    const int dd = D > 0 ? D : d;
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    const double T = slot_double(slots, S_THR);
    const uint32_t np = (uint32_t)slots[S_C2];
    unsigned long long cnt = 0;
    for (uint32_t base = warp * 32; base < r; base += nwarps * 32) {
        const uint32_t idx = base + lane;
        const bool valid = idx < r;
        const uint32_t p = valid ? (R ? R[idx] : idx) : 0;
        double t[DM];
#pragma unroll
        for (int k = 0; k < DM; ++k)
            if (k < dd) t[k] = valid ? v[(uint64_t)p * dd + k] : 0.0;
        const bool need = valid && !(__longlong_as_double((long long)key[p]) < T);
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

__global__ void k_emit_skyline(const uint32_t* __restrict__ K, uint64_t S,
                               const double* __restrict__ v, int d,
                               const int64_t* __restrict__ ids, int64_t* __restrict__ oid,
                               double* __restrict__ skyv) {
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < S;
         k += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t p = K[k];
        oid[k] = ids[p];
        for (int a = 0; a < d; ++a) skyv[a * S + k] = v[(uint64_t)p * d + a];
    }
}

void sort_pairs(Ctx& c, unsigned long long* k0, unsigned long long* k1, uint32_t* v0,
                uint32_t* v1, uint64_t n, unsigned long long** kout, uint32_t** vout) {
    cub::DoubleBuffer<unsigned long long> kb(k0, k1);
    cub::DoubleBuffer<uint32_t> vb(v0, v1);
    size_t tmp = 0;
    SKY_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, kb, vb, (int64_t)n, 0, 64, c.stream));
    void* t = c.buf[B_CUB].get(tmp);
    SKY_CUDA(cub::DeviceRadixSort::SortPairs(t, tmp, kb, vb, (int64_t)n, 0, 64, c.stream));
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

void select_flags(Ctx& c, const uint32_t* R, uint64_t r, const uint8_t* flags, uint32_t* out,
                  unsigned long long* d_count) {
    size_t tmp = 0;
    if (R) {
        SKY_CUDA(cub::DeviceSelect::Flagged(nullptr, tmp, R, flags, out, d_count, (int64_t)r,
                                             c.stream));
        void* t = c.buf[B_CUB].get(tmp);
        SKY_CUDA(cub::DeviceSelect::Flagged(t, tmp, R, flags, out, d_count, (int64_t)r,
                                             c.stream));
    } else {
        cub::CountingInputIterator<uint32_t> it(0);
        SKY_CUDA(cub::DeviceSelect::Flagged(nullptr, tmp, it, flags, out, d_count, (int64_t)r,
                                             c.stream));
        void* t = c.buf[B_CUB].get(tmp);
        SKY_CUDA(cub::DeviceSelect::Flagged(t, tmp, it, flags, out, d_count, (int64_t)r,
                                             c.stream));
    }
    note_launch(c, 2);
}

}  // namespace

SkylineOut skyline_device(Ctx& c, const double* d_vals, const int64_t* d_ids, uint64_t n, int d,
                          const skygpu_plan& plan, const double* d_reps, uint64_t n_reps) {
    SkylineOut out;
    skygpu_stats& st = *c.st;
    st.tuples_in = n;
    if (n == 0) return out;
    if (n >= 0xFFFFFFFFull) invalid("parallel_skyline: more than 2^32-1 tuples");
    const unsigned gb = grid_for(n, kBlock);

    zero_slots(c);
    auto* keys = c.buf[B_KEY0].as<unsigned long long>(n);
    trace_mark(c, "sky: start");
    k_score<<<gb, kBlock, 0, c.stream>>>(d_vals, n, d, keys, c.d_slots);
    SKY_LAUNCH_CHECK();
    k_ids_check<<<gb, kBlock, 0, c.stream>>>(d_ids, n, c.d_slots);
    SKY_LAUNCH_CHECK();
    note_launch(c, 2);
    if (plan.strategy == SKYGPU_GRID) {
        k_grid_range<<<grid_for(n * d, kBlock), kBlock, 0, c.stream>>>(d_vals, n * d, c.d_slots);
        SKY_LAUNCH_CHECK();
        note_launch(c);
    }

    uint32_t* R = nullptr;  // nullptr = all tuples
    uint64_t r = n;
    uint32_t* Rbuf0 = c.buf[B_R0].as<uint32_t>(n);
    uint32_t* Rbuf1 = c.buf[B_R1].as<uint32_t>(n);
    uint32_t* K = c.buf[B_KLIST].as<uint32_t>(n);
    // histogram bins + direction-cell segment table (ncells <= m/128 + 1 <= 4096)
    unsigned* hist = c.buf[B_ORDER].as<unsigned>(kHistBins + 4096 + 1);
    bool checked = false;
    if (n_reps > 0) {
        uint8_t* rflags = c.buf[B_FLAGS].as<uint8_t>(n);
        dispatch_d(d, [&](auto DC) {
            constexpr int D = decltype(DC)::value;
            k_rep_filter<D><<<gb, kBlock, 0, c.stream>>>(d_vals, n, d, d_reps, (uint32_t)n_reps,
                                                          rflags, c.d_slots + S_TESTS_SKY);
        });
        SKY_LAUNCH_CHECK();
        note_launch(c);
        select_flags(c, nullptr, n, rflags, Rbuf0, c.d_slots + S_C3);
        read_slots(c, S_BAD, 11);  // S_BAD .. S_C3 (checks + survivors)
        checked = true;
        R = Rbuf0;
        r = c.h_slots[S_C3];
    }
    st.tuples_into_parallel = r;

    uint64_t kc = 0;
    uint64_t want = 16384;
    const uint64_t kMaxPrefix = 65536, kFinal = 32768;
    int rounds = 0;
    cudaEvent_t e0 = c.ev[8], e1 = c.ev[9], e2 = c.ev[14], e3 = c.ev[15];
    double kernel_ms = 0;
    uint64_t kernel_launches = 0;
    uint32_t* Rnext = Rbuf1;
    while (r > 0) {
        // ---- K2: threshold, K3: prefix selection
        SKY_CUDA(cudaMemsetAsync(hist, 0, sizeof(unsigned) * kHistBins, c.stream));
        const uint64_t w = r <= kFinal ? r : want;
        if (R) {  // sum range of the undecided set
            reset_range(c);
            k_range<<<grid_for(r, kBlock, c.num_sms * 4), kBlock, 0, c.stream>>>(keys, R, r,
                                                                                 c.d_slots);
            SKY_LAUNCH_CHECK();
            note_launch(c);
        }
        k_hist<<<grid_for(r, kBlock, c.num_sms * 4), kBlock, 0, c.stream>>>(keys, R, r, c.d_slots,
                                                                            hist);
        SKY_LAUNCH_CHECK();
        k_threshold<<<1, 1024, 0, c.stream>>>(hist, r, w, c.d_slots);
        SKY_LAUNCH_CHECK();
        reset_counts(c);
        uint32_t* Pfull = c.buf[B_IDX0].as<uint32_t>(r);
        unsigned long long* Pkey = c.buf[B_KEY1].as<unsigned long long>(r);
        trace_mark(c, "sky: range/hist/threshold");
        select_if(c, R, r, BelowThreshold{keys, c.d_slots + S_THR}, Pfull, c.d_slots + S_C1);
        trace_mark(c, "sky: select prefix");
        note_launch(c, 2);
        read_slots(c, S_BAD, 11);
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
        const bool ids_sorted = (c.h_slots[S_FLAG] & 1ULL) == 0;
        const uint64_t m = c.h_slots[S_C1];
        k_keys_of<<<grid_for(m, kBlock), kBlock, 0, c.stream>>>(keys, Pfull, m, Pkey);
        SKY_LAUNCH_CHECK();
        note_launch(c);

        // ---- sort the prefix by (sum, id)
        uint32_t* P2 = c.buf[B_IDX1].as<uint32_t>(m);
        unsigned long long* Pkey2 = c.buf[B_GTMP0].as<unsigned long long>(m);
        unsigned long long* kcur;
        uint32_t* order;
        if (ids_sorted) {
            sort_pairs(c, Pkey, Pkey2, Pfull, P2, m, &kcur, &order);
        } else {
            // stable LSD: by id first, then by sum
            unsigned long long* ik0 = c.buf[B_GTMP1].as<unsigned long long>(m);
            k_id_keys<<<grid_for(m, kBlock), kBlock, 0, c.stream>>>(d_ids, Pfull, m, ik0);
            SKY_LAUNCH_CHECK();
            unsigned long long* ikc;
            uint32_t* by_id;
            sort_pairs(c, ik0, Pkey2, Pfull, P2, m, &ikc, &by_id);
            uint32_t* other = by_id == Pfull ? P2 : Pfull;
            unsigned long long* sk0 = c.buf[B_GTMP1].as<unsigned long long>(m);
            k_keys_of<<<grid_for(m, kBlock), kBlock, 0, c.stream>>>(keys, by_id, m, sk0);
            SKY_LAUNCH_CHECK();
            note_launch(c, 2);
            sort_pairs(c, sk0, Pkey2, by_id, other, m, &kcur, &order);
        }

        // ---- K4: SFS inside the prefix
        double* Av = c.buf[B_MISC].as<double>(m * d);
        trace_mark(c, "sky: (sync) + sort prefix");
        k_gather_aos<<<grid_for(m * d, kBlock), kBlock, 0, c.stream>>>(d_vals, d, order, m,
                                                                        nullptr, Av);
        SKY_LAUNCH_CHECK();
        uint8_t* keep = c.buf[B_FLAGS].as<uint8_t>(m);
        const uint64_t wi = std::min<uint64_t>(m, (uint64_t)c.num_sms * 64);
        SKY_CUDA(cudaEventRecord(e0, c.stream));
        dispatch_d(d, [&](auto DC) {
            constexpr int D = decltype(DC)::value;
            trace_mark(c, "sky: gather prefix");
            k_sfs_intra_warp<D><<<(unsigned)((wi * 32 + kBlock - 1) / kBlock), kBlock, 0,
                                  c.stream>>>(Av, (uint32_t)m, d, keep, c.d_slots + S_TESTS_SKY);
        });
        SKY_CUDA(cudaEventRecord(e1, c.stream));
        SKY_LAUNCH_CHECK();
        note_launch(c, 2);
        // A' (order-preserving) appended to K; its count lands in S_C2
        {
            size_t tmp = 0;
            SKY_CUDA(cub::DeviceSelect::Flagged(nullptr, tmp, order, keep, K + kc,
                                                 c.d_slots + S_C2, (int64_t)m, c.stream));
            void* t = c.buf[B_CUB].get(tmp);
            SKY_CUDA(cub::DeviceSelect::Flagged(t, tmp, order, keep, K + kc, c.d_slots + S_C2,
                                                 (int64_t)m, c.stream));
            note_launch(c, 2);
        }
        ++rounds;
        kernel_launches += 1;
        if (m == r) {
            read_slots(c, S_C2, 1);
            float ms = 0;
            SKY_CUDA(cudaEventElapsedTime(&ms, e0, e1));
            kernel_ms += ms;
            kc += c.h_slots[S_C2];
            break;
        }
        // ---- K5: filter the rest against A', comparators in direction-cell
        // order (own cell first) so dominators are met early
        int mcell = 1;
        if (d >= 2) {
            const double target = std::max(1.0, (double)m / 128.0);
            mcell = (int)std::floor(std::pow(target, 1.0 / (d - 1)) + 1e-9);
            mcell = std::max(1, std::min(mcell, 32));
        }
        uint32_t ncells = 1;
        for (int k = 0; k < d - 1; ++k) ncells *= (uint32_t)mcell;
        double* Pv = c.buf[B_CSUM].as<double>(m * d);
        uint32_t* seg = nullptr;
        const uint32_t* psrc = K + kc;
        if (mcell > 1) {
            uint32_t* ck0 = c.buf[B_GTMP1].as<uint32_t>(m);
            uint32_t* ck1 = reinterpret_cast<uint32_t*>(Pkey);  // free after the sort
            uint32_t* ov = order;
            uint32_t* oalt = order == Pfull ? P2 : Pfull;
            dispatch_d(d, [&](auto DC) {
                constexpr int D = decltype(DC)::value;
                k_prefix_cells<D><<<grid_for(m, kBlock), kBlock, 0, c.stream>>>(Av, (uint32_t)m, d,
                                                                                 keep, mcell, ck0);
            });
            SKY_LAUNCH_CHECK();
            cub::DoubleBuffer<uint32_t> kb(ck0, ck1), vb(ov, oalt);
            size_t tmp = 0;
            SKY_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, kb, vb, (int64_t)m, 0, 32,
                                                     c.stream));
            void* tp = c.buf[B_CUB].get(tmp);
            SKY_CUDA(cub::DeviceRadixSort::SortPairs(tp, tmp, kb, vb, (int64_t)m, 0, 32,
                                                     c.stream));
            seg = reinterpret_cast<uint32_t*>(hist) + kHistBins;
            k_cell_segments<<<grid_for(ncells + 1, kBlock), kBlock, 0, c.stream>>>(
                kb.Current(), (uint32_t)m, ncells, seg);
            SKY_LAUNCH_CHECK();
            note_launch(c, 6);
            psrc = vb.Current();
        }
        k_gather_aos<<<grid_for(m * d, kBlock), kBlock, 0, c.stream>>>(d_vals, d, psrc, m,
                                                                        c.d_slots + S_C2, Pv);
        SKY_LAUNCH_CHECK();
        const uint64_t wf = std::min<uint64_t>((r + 31) / 32, (uint64_t)c.num_sms * 64);
        uint8_t* fkeep = c.buf[B_SV].as<uint8_t>(r);
        SKY_CUDA(cudaEventRecord(e2, c.stream));
        dispatch_d(d, [&](auto DC) {
            constexpr int D = decltype(DC)::value;
            trace_mark(c, "sky: select A' + cells + gather Pv");
            k_sfs_filter_cells<D><<<(unsigned)((wf * 32 + kBlock - 1) / kBlock), kBlock, 0,
                                    c.stream>>>(d_vals, d, keys, R, (uint32_t)r, Pv, (uint32_t)m,
                                                seg, mcell, c.d_slots, fkeep,
                                                c.d_slots + S_TESTS_SKY);
        });
        SKY_CUDA(cudaEventRecord(e3, c.stream));
        SKY_LAUNCH_CHECK();
        note_launch(c, 2);
        trace_mark(c, "sky: K5 filter kernel");
        select_flags(c, R, r, fkeep, Rnext, c.d_slots + S_C3);
        trace_mark(c, "sky: select survivors");
        kernel_launches += 1;
        read_slots(c, S_C2, 2);  // S_C2 (A'), S_C3 (survivors)
        float ms = 0;
        SKY_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        kernel_ms += ms;
        SKY_CUDA(cudaEventElapsedTime(&ms, e2, e3));
        kernel_ms += ms;
        const uint64_t a = c.h_slots[S_C2];
        kc += a;
        r = c.h_slots[S_C3];
        R = Rnext;
        Rnext = (Rnext == Rbuf1) ? Rbuf0 : Rbuf1;
        if (a * 2 > m) want = std::min(want * 4, kMaxPrefix);
    }
    st.sfs_rounds = rounds;
    st.tuples_into_final = kc;
    st.ms_sky_kernel += kernel_ms;
    st.sky_kernel_launches += kernel_launches;

    out.S = kc;
    out.d_inpos = K;
    out.d_ids = c.buf[B_SKYID].as<int64_t>(kc);
    out.d_skyv = c.buf[B_SKYV].as<double>(kc * d);
    if (kc) {
        trace_mark(c, "sky: rounds done (sync)");
        k_emit_skyline<<<grid_for(kc, kBlock), kBlock, 0, c.stream>>>(K, kc, d_vals, d, d_ids,
                                                                      out.d_ids, out.d_skyv);
        SKY_LAUNCH_CHECK();
        note_launch(c);
    }
    st.skyline_size = kc;
    return out;
}

}  // namespace skygpu
