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
// GPU algorithm (block-SFS with filter passes):
//   K1  score: left-to-right __dadd_rn sum, key = bits(sum)   (HBM-bound)
//   --  CUB radix sort of (key, index) [pre-sorted by id when ids are not
//       ascending], giving the reference's (sum, id) order
//   K2  gather into SoA sorted arrays (coalesced tiles for K3/K4)
//   loop over rounds, R = undecided sorted positions (ascending):
//     K3  intra: the first m of R test all their predecessors in that
//         prefix (smem-tiled, block-level early exit) -> new skyline A'
//     K4  filter: the rest of R is tested against A' (smem-tiled, block
//         early exit) and compacted.  Everything left in R has been tested
//         against every confirmed skyline tuple, so K3's verdict is final.
// Dominated tuples are discarded the first time any earlier skyline tuple
// dominates them; the prefix size m grows when rounds confirm mostly
// skyline tuples (large-skyline data), bounding the number of rounds.
#include <cub/cub.cuh>

#include "sky_common.cuh"

namespace skygpu {

namespace {

constexpr int kBlock = 256;

__global__ void k_score(const double* __restrict__ v, uint64_t n, int d,
                        unsigned long long* __restrict__ key, uint32_t* __restrict__ idx,
                        unsigned long long* __restrict__ slots) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        bool bad = false;
        for (int k = 0; k < d; ++k) {
            double x = v[i * d + k];
            bad |= !(x >= 0.0);  // negative or NaN
            s = __dadd_rn(s, x);
        }
        key[i] = ord_bits(s);
        idx[i] = static_cast<uint32_t>(i);
        if (bad) atomicMin(&slots[S_BAD], static_cast<unsigned long long>(i));
    }
}

__global__ void k_ids_check(const int64_t* __restrict__ ids, uint64_t n,
                            unsigned long long* __restrict__ slots) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i + 1 < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        if (ids[i] >= ids[i + 1]) atomicOr(&slots[S_FLAG], 1ULL);
}

__global__ void k_id_keys(const int64_t* __restrict__ ids, uint64_t n,
                          unsigned long long* __restrict__ key, uint32_t* __restrict__ idx) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        key[i] = static_cast<unsigned long long>(ids[i]) ^ 0x8000000000000000ULL;
        idx[i] = static_cast<uint32_t>(i);
    }
}

__global__ void k_permute_keys(const unsigned long long* __restrict__ score,
                               const uint32_t* __restrict__ idx, uint64_t n,
                               unsigned long long* __restrict__ out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = score[idx[i]];
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

// K2: sorted SoA gather
__global__ void k_gather_sorted(const double* __restrict__ v, const int64_t* __restrict__ ids,
                                const uint32_t* __restrict__ order, uint64_t n, int d,
                                double* __restrict__ sv, int64_t* __restrict__ sid,
                                uint32_t* __restrict__ spos) {
    for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < n;
         p += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t i = order[p];
        for (int k = 0; k < d; ++k) sv[k * n + p] = v[(uint64_t)i * d + k];
        sid[p] = ids[i];
        spos[p] = i;
    }
}

__global__ void k_iota(uint32_t* __restrict__ r, uint64_t n) {
    for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < n;
         p += (uint64_t)gridDim.x * blockDim.x)
        r[p] = static_cast<uint32_t>(p);
}

// Representative filter (partition.cpp:287-302): a tuple dominated by any
// representative never enters the local skylines.  reps: AoS [n_reps][d].
template <int D>
__global__ void k_rep_filter(const double* __restrict__ sv, uint64_t n, int d,
                             const double* __restrict__ reps, uint32_t n_reps,
                             uint8_t* __restrict__ keep, unsigned long long* __restrict__ tests) {
    const int dd = D > 0 ? D : d;
    double t[D > 0 ? D : kMaxDims];
    unsigned long long cnt = 0;
    for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < n;
         p += (uint64_t)gridDim.x * blockDim.x) {
#pragma unroll
        for (int k = 0; k < (D > 0 ? D : kMaxDims); ++k)
            if (k < dd) t[k] = sv[k * n + p];
        bool alive = true;
        for (uint32_t r = 0; r < n_reps && alive; ++r) {
            ++cnt;
            alive = !dom_f64_dyn(reps + (uint64_t)r * dd, t, dd);
        }
        keep[p] = alive;
    }
    add_count(tests, cnt);
}

template <int D>
constexpr int tile_of() { return D > 0 ? 256 : 128; }

// K3: candidates A[0..m) (ascending sorted positions) against their
// predecessors inside the same prefix.
template <int D>
__global__ void __launch_bounds__(kBlock)
k_sfs_intra(const double* __restrict__ sv, uint64_t stride, int d,
            const uint32_t* __restrict__ A, uint32_t m, uint8_t* __restrict__ keep,
            unsigned long long* __restrict__ tests) {
    constexpr int TILE = tile_of<D>();
    constexpr int DM = D > 0 ? D : kMaxDims;
    extern __shared__ double tile[];  // [dd][TILE]
    const int dd = D > 0 ? D : d;
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    const bool valid = i < m;
    double t[DM];
    if (valid) {
        const uint32_t p = A[i];
#pragma unroll
        for (int k = 0; k < DM; ++k)
            if (k < dd) t[k] = sv[k * stride + p];
    }
    bool alive = valid;
    unsigned long long cnt = 0;
    const uint32_t blk_end = min(m, (blockIdx.x + 1) * blockDim.x);
    for (uint32_t base = 0; base < blk_end; base += TILE) {
        const uint32_t nt = min((uint32_t)TILE, blk_end - base);
        for (uint32_t k = threadIdx.x; k < nt; k += blockDim.x) {
            const uint32_t p = A[base + k];
            for (int a = 0; a < dd; ++a) tile[a * TILE + k] = sv[a * stride + p];
        }
        __syncthreads();
        if (alive && i > base) {
            const uint32_t lim = min(nt, i - base);
            for (uint32_t k = 0; k < lim; ++k) {
                double s[DM];
#pragma unroll
                for (int a = 0; a < DM; ++a)
                    if (a < dd) s[a] = tile[a * TILE + k];
                ++cnt;
                bool dm = D > 0 ? dom_f64<(D > 0 ? D : 1)>(s, t) : dom_f64_dyn(s, t, dd);
                if (dm) {
                    alive = false;
                    break;
                }
            }
        }
        if (!__syncthreads_or(alive)) break;
    }
    if (valid) keep[i] = alive ? 1 : 0;
    add_count(tests, cnt);
}

// K4: candidates C[0..cn) against the newly confirmed skyline tuples
// P[0..np) (all of which precede every candidate in (sum, id) order).
template <int D>
__global__ void __launch_bounds__(kBlock)
k_sfs_filter(const double* __restrict__ sv, uint64_t stride, int d,
             const uint32_t* __restrict__ C, uint32_t cn, const uint32_t* __restrict__ P,
             uint32_t np, uint8_t* __restrict__ keep, unsigned long long* __restrict__ tests) {
    constexpr int TILE = tile_of<D>();
    constexpr int DM = D > 0 ? D : kMaxDims;
    extern __shared__ double tile[];
    const int dd = D > 0 ? D : d;
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    const bool valid = i < cn;
    double t[DM];
    if (valid) {
        const uint32_t p = C[i];
#pragma unroll
        for (int k = 0; k < DM; ++k)
            if (k < dd) t[k] = sv[k * stride + p];
    }
    bool alive = valid;
    unsigned long long cnt = 0;
    for (uint32_t base = 0; base < np; base += TILE) {
        const uint32_t nt = min((uint32_t)TILE, np - base);
        for (uint32_t k = threadIdx.x; k < nt; k += blockDim.x) {
            const uint32_t p = P[base + k];
            for (int a = 0; a < dd; ++a) tile[a * TILE + k] = sv[a * stride + p];
        }
        __syncthreads();
        if (alive) {
            for (uint32_t k = 0; k < nt; ++k) {
                double s[DM];
#pragma unroll
                for (int a = 0; a < DM; ++a)
                    if (a < dd) s[a] = tile[a * TILE + k];
                ++cnt;
                bool dm = D > 0 ? dom_f64<(D > 0 ? D : 1)>(s, t) : dom_f64_dyn(s, t, dd);
                if (dm) {
                    alive = false;
                    break;
                }
            }
        }
        if (!__syncthreads_or(alive)) break;
    }
    if (valid) keep[i] = alive ? 1 : 0;
    add_count(tests, cnt);
}

// compact SoA copy of the tuples at sorted positions list[0..m)
__global__ void k_gather_list(const double* __restrict__ sv, uint64_t stride, int d,
                              const uint32_t* __restrict__ list, uint64_t m,
                              double* __restrict__ out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m * d;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t a = i / m, k = i - a * m;
        out[i] = sv[a * stride + list[k]];
    }
}

// Warp-cooperative variants (warp-ballot early exit, north_star (a)): one
// candidate per warp, its d values broadcast in registers; the 32 lanes test
// 32 consecutive comparators per iteration (coalesced float64 SoA loads that
// hit L1/L2: the comparator block is small and shared by every warp) and the
// warp leaves the candidate at the first iteration whose ballot is non-zero.
// No divergence inside a warp, no block-level barrier.
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

template <int D>
__global__ void __launch_bounds__(kBlock)
k_sfs_filter_warp(const double* __restrict__ sv, uint64_t stride, int d,
                  const uint32_t* __restrict__ C, uint32_t cn, const double* __restrict__ Pv,
                  uint32_t np, uint8_t* __restrict__ keep, unsigned long long* __restrict__ tests) {
    constexpr int DM = D > 0 ? D : kMaxDims;
    const int dd = D > 0 ? D : d;
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    unsigned long long cnt = 0;
    for (uint32_t i = warp; i < cn; i += nwarps) {
        const uint32_t p = C[i];
        double t[DM];
#pragma unroll
        for (int k = 0; k < DM; ++k)
            if (k < dd) t[k] = sv[(uint64_t)k * stride + p];
        bool dominated = false;
        for (uint32_t j0 = 0; j0 < np; j0 += 32) {
            const uint32_t j = j0 + lane;
            bool hit = false;
            if (j < np) {
                double s[DM];
#pragma unroll
                for (int k = 0; k < DM; ++k)
                    if (k < dd) s[k] = Pv[(uint64_t)k * np + j];
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

__global__ void k_emit_skyline(const uint32_t* __restrict__ K, uint64_t S,
                               const double* __restrict__ sv, uint64_t n, int d,
                               const int64_t* __restrict__ sid, const uint32_t* __restrict__ spos,
                               uint32_t* __restrict__ inpos, int64_t* __restrict__ oid,
                               double* __restrict__ skyv) {
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < S;
         k += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t p = K[k];
        inpos[k] = spos[p];
        oid[k] = sid[p];
        for (int a = 0; a < d; ++a) skyv[a * S + k] = sv[a * n + p];
    }
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

// DeviceSelect::Flagged with the count landing in slot S_SEL; returns count.
uint64_t select_flagged(Ctx& c, const uint32_t* in, const uint8_t* flags, uint32_t* out,
                        uint64_t n) {
    if (n == 0) return 0;
    size_t tmp = 0;
    SKY_CUDA(cub::DeviceSelect::Flagged(nullptr, tmp, in, flags, out,
                                         c.d_slots + S_SEL, (int64_t)n, c.stream));
    void* t = c.buf[B_CUB].get(tmp);
    SKY_CUDA(cub::DeviceSelect::Flagged(t, tmp, in, flags, out, c.d_slots + S_SEL,
                                         (int64_t)n, c.stream));
    note_launch(c, 2);
    read_slots(c, S_SEL, 1);
    return c.h_slots[S_SEL];
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

}  // namespace

void aos_to_soa(Ctx& c, const double* d_aos, uint64_t n, int d, double* d_soa);

SkylineOut skyline_device(Ctx& c, const double* d_vals, const int64_t* d_ids, uint64_t n, int d,
                          const skygpu_plan& plan, const double* d_reps, uint64_t n_reps) {
    SkylineOut out;
    skygpu_stats& st = *c.st;
    st.tuples_in = n;
    if (n == 0) return out;
    if (n >= 0xFFFFFFFFull) invalid("parallel_skyline: more than 2^32-1 tuples");
    const unsigned gb = grid_for(n, kBlock);

    // contract checks: the reference's Relation::add rejects negatives
    // (core.cpp:14-17); NaN breaks the reference's strict weak ordering.
    zero_slots(c);
    auto* keys0 = c.buf[B_KEY0].as<unsigned long long>(n);
    auto* keys1 = c.buf[B_KEY1].as<unsigned long long>(n);
    auto* idx0 = c.buf[B_IDX0].as<uint32_t>(n);
    auto* idx1 = c.buf[B_IDX1].as<uint32_t>(n);
    k_score<<<gb, kBlock, 0, c.stream>>>(d_vals, n, d, keys0, idx0, c.d_slots);
    SKY_LAUNCH_CHECK();
    k_ids_check<<<gb, kBlock, 0, c.stream>>>(d_ids, n, c.d_slots);
    SKY_LAUNCH_CHECK();
    if (plan.strategy == SKYGPU_GRID) {
        k_grid_range<<<grid_for(n * d, kBlock), kBlock, 0, c.stream>>>(d_vals, n * d,
                                                                        c.d_slots);
        SKY_LAUNCH_CHECK();
    }
    note_launch(c, plan.strategy == SKYGPU_GRID ? 3 : 2);
    read_slots(c, S_BAD, 5);  // S_BAD .. S_GRIDBAD
    if (c.h_slots[S_BAD] != ~0ULL) {
        const uint64_t tuple = c.h_slots[S_BAD];
        invalid("parallel_skyline: tuple at position " + std::to_string(tuple) +
                " has a negative or NaN value (Relation::add contract, core.cpp:14-17)");
    }
    if (c.h_slots[S_GRIDBAD] != ~0ULL) {
        const uint64_t flat = c.h_slots[S_GRIDBAD];
        double v = 0;
        SKY_CUDA(cudaMemcpyAsync(&v, d_vals + flat, sizeof(double), cudaMemcpyDeviceToHost,
                                 c.stream));
        SKY_CUDA(cudaStreamSynchronize(c.stream));
        invalid("grid_cell: value " + std::to_string(v) + " in attribute " +
                std::to_string(flat % d + 1) + " outside [0,1]; normalize the data first");
    }
    const bool ids_sorted = c.h_slots[S_FLAG] == 0;

    // (sum, id) order
    unsigned long long* kcur;
    uint32_t* order;
    if (ids_sorted) {
        sort_pairs(c, keys0, keys1, idx0, idx1, n, &kcur, &order);
    } else {
        // stable LSD sorts: first by id, then by score
        auto* ik0 = c.buf[B_GTMP0].as<unsigned long long>(n);
        auto* ik1 = c.buf[B_GTMP1].as<unsigned long long>(n);
        k_id_keys<<<gb, kBlock, 0, c.stream>>>(d_ids, n, ik0, idx1);
        SKY_LAUNCH_CHECK();
        unsigned long long* ikc;
        uint32_t* by_id;
        // score keys live in keys0; sort (id key, idx) using idx1/idx0
        sort_pairs(c, ik0, ik1, idx1, idx0, n, &ikc, &by_id);
        uint32_t* other = by_id == idx0 ? idx1 : idx0;
        k_permute_keys<<<gb, kBlock, 0, c.stream>>>(keys0, by_id, n, keys1);
        SKY_LAUNCH_CHECK();
        note_launch(c, 2);
        sort_pairs(c, keys1, keys0, by_id, other, n, &kcur, &order);
    }

    // K2: sorted SoA arrays
    double* sv = c.buf[B_SV].as<double>(n * d);
    int64_t* sid = c.buf[B_SID].as<int64_t>(n);
    uint32_t* spos = c.buf[B_SPOS].as<uint32_t>(n);
    k_gather_sorted<<<gb, kBlock, 0, c.stream>>>(d_vals, d_ids, order, n, d, sv, sid, spos);
    SKY_LAUNCH_CHECK();
    note_launch(c);

    uint32_t* R = c.buf[B_R0].as<uint32_t>(n);
    uint32_t* R2 = c.buf[B_R1].as<uint32_t>(n);
    uint8_t* flags = c.buf[B_FLAGS].as<uint8_t>(n);
    uint32_t* K = c.buf[B_KLIST].as<uint32_t>(n);
    uint64_t r = n;
    k_iota<<<gb, kBlock, 0, c.stream>>>(R, n);
    SKY_LAUNCH_CHECK();
    note_launch(c);

    if (n_reps > 0) {
        dispatch_d(d, [&](auto DC) {
            constexpr int D = decltype(DC)::value;
            k_rep_filter<D><<<gb, kBlock, 0, c.stream>>>(sv, n, d, d_reps, (uint32_t)n_reps,
                                                          flags, c.d_slots + S_TESTS_SKY);
        });
        SKY_LAUNCH_CHECK();
        note_launch(c);
        r = select_flagged(c, R, flags, R2, n);
        std::swap(R, R2);
    }
    st.tuples_into_parallel = r;

    uint64_t kc = 0;
    uint64_t alpha = 4096;
    const uint64_t kFinal = 32768, kAlphaMax = 65536;
    int rounds = 0;
    cudaEvent_t e0 = c.ev[8], e1 = c.ev[9];
    double kernel_ms = 0;
    uint64_t kernel_launches = 0;
    double* Av = c.buf[B_MISC].as<double>(std::min<uint64_t>(n, kAlphaMax) * d);
    double* Pv = c.buf[B_CSUM].as<double>(std::min<uint64_t>(n, kAlphaMax) * d);
    auto warp_grid = [&](uint64_t items) {
        const uint64_t warps = std::min<uint64_t>(items, (uint64_t)c.num_sms * 64);
        return (unsigned)std::max<uint64_t>(1, (warps * 32 + kBlock - 1) / kBlock);
    };
    while (r > 0) {
        const uint64_t m = (r <= kFinal) ? r : std::min(alpha, r);
        if (m > kAlphaMax) Av = c.buf[B_MISC].as<double>(m * d);
        k_gather_list<<<grid_for(m * d, kBlock), kBlock, 0, c.stream>>>(sv, n, d, R, m, Av);
        SKY_LAUNCH_CHECK();
        dispatch_d(d, [&](auto DC) {
            constexpr int D = decltype(DC)::value;
            SKY_CUDA(cudaEventRecord(e0, c.stream));
            k_sfs_intra_warp<D><<<warp_grid(m), kBlock, 0, c.stream>>>(
                Av, (uint32_t)m, d, flags, c.d_slots + S_TESTS_SKY);
            SKY_CUDA(cudaEventRecord(e1, c.stream));
        });
        SKY_LAUNCH_CHECK();
        note_launch(c, 2);
        const uint64_t a = select_flagged(c, R, flags, K + kc, m);
        float ms = 0;
        SKY_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        kernel_ms += ms;
        ++kernel_launches;
        kc += a;
        ++rounds;
        if (m == r) break;
        const uint64_t cn = r - m;
        if (a > kAlphaMax) Pv = c.buf[B_CSUM].as<double>(a * d);
        k_gather_list<<<grid_for(a * d, kBlock), kBlock, 0, c.stream>>>(sv, n, d, K + kc - a, a,
                                                                         Pv);
        SKY_LAUNCH_CHECK();
        note_launch(c);
        dispatch_d(d, [&](auto DC) {
            constexpr int D = decltype(DC)::value;
            SKY_CUDA(cudaEventRecord(e0, c.stream));
            k_sfs_filter_warp<D><<<warp_grid(cn), kBlock, 0, c.stream>>>(
                sv, n, d, R + m, (uint32_t)cn, Pv, (uint32_t)a, flags, c.d_slots + S_TESTS_SKY);
            SKY_CUDA(cudaEventRecord(e1, c.stream));
        });
        SKY_LAUNCH_CHECK();
        note_launch(c);
        r = select_flagged(c, R + m, flags, R2, cn);
        SKY_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        kernel_ms += ms;
        ++kernel_launches;
        std::swap(R, R2);
        if (a * 2 > m && alpha < kAlphaMax) alpha *= 4;
    }
    st.sfs_rounds = rounds;
    st.tuples_into_final = kc;
    st.ms_sky_kernel += kernel_ms;
    st.sky_kernel_launches += kernel_launches;

    out.S = kc;
    out.d_inpos = c.buf[B_OUTPOS].as<uint32_t>(kc);
    out.d_ids = c.buf[B_SKYID].as<int64_t>(kc);
    out.d_skyv = c.buf[B_SKYV].as<double>(kc * d);
    k_emit_skyline<<<grid_for(kc, kBlock), kBlock, 0, c.stream>>>(
        K, kc, sv, n, d, sid, spos, out.d_inpos, out.d_ids, out.d_skyv);
    SKY_LAUNCH_CHECK();
    note_launch(c);
    read_slots(c, S_TESTS_SKY, 1);
    st.skyline_tests = c.h_slots[S_TESTS_SKY];
    st.skyline_size = kc;
    return out;
}

}  // namespace skygpu
