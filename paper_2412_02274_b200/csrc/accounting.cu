// accounting.cu — exact reference accounting ("metrics-parity" mode,
// SURVEY.md §8(f) rank 2).  NOT the hot path: results never depend on it.
//
// The reference reports, besides the skyline and the denominators, the
// number of dominance tests its CPU algorithm executes (DominanceCounter,
// core.hpp:46-67): per partition the representative filter
// (partition.cpp:287-302) plus the local SFS (core.cpp:48-73), and the SFS of
// the merge phase (parallel.cpp:83-86).  Those numbers are the paper's cost
// model (PhaseMetrics / IterationCost, simulated_cost) and the reference's
// tests pin them (test_parallel.cpp:25-43, acceptance criteria 8 and 10).
// They are a property of the SFS algorithm, not of the answer, so this file
// derives them exactly on the GPU:
//
//   SFS over a list L sorted by (sum, id): tuple t is tested against the
//   window (the kept tuples before it, in order) until the first dominator.
//   kept t        -> tests = #kept tuples before t in its partition
//   dominated t   -> tests = 1-based window position of the FIRST kept tuple
//                    (in order) that dominates t
//   rep filter    -> tests = 1-based index of the first dominating
//                    representative, else #representatives
//
// Kept flags follow the predecessor rule; the first kept
// dominator of a dominated tuple always lies inside its window, so a scan of
// the partition's kept list from its start finds exactly the reference's
// stopping point.  One warp per tuple, 32 window entries per ballot.
#include <cub/cub.cuh>

#include "sky_common.cuh"

namespace skygpu {
namespace {

constexpr int kAB = 256;

__device__ __forceinline__ bool dom_dyn(const double* __restrict__ A, uint64_t m, int d,
                                        uint32_t s, uint32_t t) {
    bool le = true, lt = false;
    for (int k = 0; k < d; ++k) {
        const double a = A[(uint64_t)k * m + s], b = A[(uint64_t)k * m + t];
        le &= a <= b;
        lt |= a < b;
    }
    return le & lt;
}

// sum keys (core.cpp:21-23, left to right from +0.0) of every tuple
__global__ void k_acc_keys(const double* __restrict__ v, uint64_t n, int d,
                           unsigned long long* __restrict__ key) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int k = 0; k < d; ++k) s = __dadd_rn(s, v[i * d + k]);
        key[i] = ord_bits(s);
    }
}

// representative filter: tests and survivors of every tuple still in phase 1
__global__ void k_acc_reps(const double* __restrict__ v, uint64_t n, int d,
                           const int32_t* __restrict__ gid, const double* __restrict__ reps,
                           uint32_t nr, uint8_t* __restrict__ alive,
                           unsigned long long* __restrict__ per_group) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const int32_t g = gid[i];
        if (g < 0) {
            alive[i] = 0;
            continue;
        }
        uint32_t k = 0;
        bool dom = false;
        for (; k < nr && !dom; ++k) dom = dom_f64_dyn(reps + (uint64_t)k * d, v + i * d, d);
        if (nr) atomicAdd(&per_group[g], (unsigned long long)(dom ? k : nr));
        alive[i] = dom ? 0 : 1;
    }
}

__global__ void k_acc_sortkeys(const uint32_t* __restrict__ L, uint64_t m,
                               const int64_t* __restrict__ ids,
                               const unsigned long long* __restrict__ key,
                               const int32_t* __restrict__ gid, int which,
                               unsigned long long* __restrict__ out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t p = L[i];
        out[i] = which == 0   ? (unsigned long long)ids[p] ^ 0x8000000000000000ULL  // signed order
                 : which == 1 ? key[p]
                              : (unsigned long long)(uint32_t)gid[p];
    }
}

// sorted list -> SoA values, group of every slot, group histogram
__global__ void k_acc_gather(const double* __restrict__ v, int d, const uint32_t* __restrict__ P,
                             uint64_t m, const int32_t* __restrict__ gid,
                             double* __restrict__ A, uint32_t* __restrict__ grp,
                             uint32_t* __restrict__ hist) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t p = P[i];
        for (int k = 0; k < d; ++k) A[(uint64_t)k * m + i] = v[(uint64_t)p * d + k];
        const uint32_t g = (uint32_t)gid[p];
        grp[i] = g;
        atomicAdd(&hist[g], 1u);
    }
}

// kept flags: warp per slot, predecessors inside its group
__global__ void __launch_bounds__(kAB)
k_acc_kept(const double* __restrict__ A, uint64_t m, int d, const uint32_t* __restrict__ grp,
           const uint32_t* __restrict__ gstart, uint32_t* __restrict__ kept) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t i = warp; i < m; i += nw) {
        const uint32_t g0 = gstart[grp[i]];
        bool dominated = false;
        for (uint64_t j0 = g0; j0 < i && !dominated; j0 += 32) {
            const uint64_t j = j0 + lane;
            const bool hit = j < i && dom_dyn(A, m, d, (uint32_t)j, (uint32_t)i);
            dominated = __any_sync(0xffffffffu, hit);
        }
        if (lane == 0) kept[i] = dominated ? 0u : 1u;
    }
}

// tests of every slot (see header); K = kept slots in order, kscan =
// exclusive scan of the kept flags
__global__ void __launch_bounds__(kAB)
k_acc_count(const double* __restrict__ A, uint64_t m, int d, const uint32_t* __restrict__ grp,
            const uint32_t* __restrict__ gstart, const uint32_t* __restrict__ kept,
            const uint32_t* __restrict__ kscan, const uint32_t* __restrict__ K,
            unsigned long long* __restrict__ per_group) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t i = warp; i < m; i += nw) {
        const uint32_t g = grp[i];
        const uint32_t kb = kscan[gstart[g]], ki = kscan[i];
        unsigned long long tests;
        if (kept[i]) {
            tests = ki - kb;
        } else {
            tests = 0;
            for (uint32_t k0 = kb; k0 < ki; k0 += 32) {
                const uint32_t k = k0 + lane;
                const bool hit = k < ki && dom_dyn(A, m, d, K[k], (uint32_t)i);
                const unsigned b = __ballot_sync(0xffffffffu, hit);
                if (b) {
                    tests = (unsigned long long)(k0 - kb) + (unsigned)__ffs(b);
                    break;
                }
            }
        }
        if (lane == 0 && tests) atomicAdd(&per_group[g], tests);
    }
}

__global__ void k_acc_kept_pos(const uint32_t* __restrict__ P, const uint32_t* __restrict__ K,
                               uint64_t nk, uint32_t* __restrict__ out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nk;
         i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = P[K[i]];
}

template <class KT>
void sort_pairs_acc(Ctx& c, KT*& k0, KT*& k1, uint32_t*& v0, uint32_t*& v1, uint64_t n, int bits) {
    cub::DoubleBuffer<KT> kb(k0, k1);
    cub::DoubleBuffer<uint32_t> vb(v0, v1);
    size_t tmp = 0;
    SKY_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, kb, vb, (int64_t)n, 0, bits, c.stream));
    void* t = c.buf[B_CUB].get(tmp);
    SKY_CUDA(cub::DeviceRadixSort::SortPairs(t, tmp, kb, vb, (int64_t)n, 0, bits, c.stream));
    note_launch(c, 4);
    k0 = kb.Current();
    k1 = kb.Alternate();
    v0 = vb.Current();
    v1 = vb.Alternate();
}

}  // namespace

// SFS accounting of the groups of one phase: gid[i] in [0, p) = group of
// tuple i (negative = not in this phase), optional representatives (nr,
// row-major) filtering every group first.  Adds every group's tests into
// d_per_group[p] (caller-zeroed) and writes the kept positions — group by
// group, each in (sum, id) order — into d_kept; returns their count.
uint64_t sfs_accounting_device(Ctx& c, const double* d_vals, const int64_t* d_ids, uint64_t n,
                               int d, const int32_t* d_gid, uint32_t p, const double* d_reps,
                               uint32_t nr, unsigned long long* d_per_group, uint32_t* d_kept) {
    if (n == 0 || p == 0) return 0;
    auto* key = c.buf[B_ACC0].as<unsigned long long>(n);
    auto* alive = c.buf[B_ACC1].as<uint8_t>(n);
    const unsigned gb = grid_for(n, kAB);
    k_acc_keys<<<gb, kAB, 0, c.stream>>>(d_vals, n, d, key);
    k_acc_reps<<<gb, kAB, 0, c.stream>>>(d_vals, n, d, d_gid, d_reps, nr, alive, d_per_group);
    SKY_LAUNCH_CHECK();
    note_launch(c, 2);
    // survivors, in position order
    uint32_t* L0 = c.buf[B_ACC2].as<uint32_t>(n);
    uint32_t* L1 = c.buf[B_ACC3].as<uint32_t>(n);
    {
        size_t tmp = 0;
        cub::CountingInputIterator<uint32_t> it(0);
        SKY_CUDA(cub::DeviceSelect::Flagged(nullptr, tmp, it, alive, L0, c.d_slots + S_SEL2,
                                             (int64_t)n, c.stream));
        void* t = c.buf[B_CUB].get(tmp);
        SKY_CUDA(cub::DeviceSelect::Flagged(t, tmp, it, alive, L0, c.d_slots + S_SEL2, (int64_t)n,
                                             c.stream));
        note_launch(c, 2);
    }
    read_slots(c, S_SEL2, 1);
    const uint64_t m = c.h_slots[S_SEL2];
    if (m == 0) return 0;
    // stable LSD passes: id (signed), sum key, group
    auto* k0 = c.buf[B_ACC4].as<unsigned long long>(m);
    auto* k1 = c.buf[B_ACC5].as<unsigned long long>(m);
    for (int which = 0; which < 3; ++which) {
        k_acc_sortkeys<<<grid_for(m, kAB), kAB, 0, c.stream>>>(L0, m, d_ids, key, d_gid, which, k0);
        SKY_LAUNCH_CHECK();
        note_launch(c);
        sort_pairs_acc<unsigned long long>(c, k0, k1, L0, L1, m, which == 2 ? 32 : 64);
    }
    uint32_t* P = L0;  // sorted slots -> positions
    double* A = c.buf[B_ACC6].as<double>(m * d);
    uint32_t* grp = c.buf[B_ACC7].as<uint32_t>(m);
    uint32_t* hist = c.buf[B_ACC8].as<uint32_t>(2 * ((uint64_t)p + 1));
    uint32_t* gstart = hist + p + 1;
    SKY_CUDA(cudaMemsetAsync(hist, 0, sizeof(uint32_t) * (p + 1), c.stream));
    k_acc_gather<<<grid_for(m, kAB), kAB, 0, c.stream>>>(d_vals, d, P, m, d_gid, A, grp, hist);
    SKY_LAUNCH_CHECK();
    note_launch(c);
    uint32_t* kept = c.buf[B_ACC9].as<uint32_t>(m + 1);
    uint32_t* kscan = c.buf[B_ACC10].as<uint32_t>(m + 1);
    uint32_t* K = c.buf[B_ACC11].as<uint32_t>(m);
    {
        size_t tmp = 0;
        SKY_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, hist, gstart, (int)p + 1, c.stream));
        void* t = c.buf[B_CUB].get(tmp);
        SKY_CUDA(cub::DeviceScan::ExclusiveSum(t, tmp, hist, gstart, (int)p + 1, c.stream));
        note_launch(c);
    }
    const unsigned wg = grid_for(m * 32, kAB, c.num_sms * 16);
    k_acc_kept<<<wg, kAB, 0, c.stream>>>(A, m, d, grp, gstart, kept);
    SKY_LAUNCH_CHECK();
    SKY_CUDA(cudaMemsetAsync(kept + m, 0, sizeof(uint32_t), c.stream));
    {
        size_t tmp = 0;
        SKY_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, kept, kscan, (int)m + 1, c.stream));
        void* t = c.buf[B_CUB].get(tmp);
        SKY_CUDA(cub::DeviceScan::ExclusiveSum(t, tmp, kept, kscan, (int)m + 1, c.stream));
        cub::CountingInputIterator<uint32_t> it(0);
        size_t tmp2 = 0;
        SKY_CUDA(cub::DeviceSelect::Flagged(nullptr, tmp2, it, kept, K, c.d_slots + S_SEL2,
                                             (int64_t)m, c.stream));
        void* t2 = c.buf[B_CUB].get(tmp2);
        SKY_CUDA(cub::DeviceSelect::Flagged(t2, tmp2, it, kept, K, c.d_slots + S_SEL2, (int64_t)m,
                                             c.stream));
        note_launch(c, 4);
    }
    k_acc_count<<<wg, kAB, 0, c.stream>>>(A, m, d, grp, gstart, kept, kscan, K, d_per_group);
    SKY_LAUNCH_CHECK();
    note_launch(c, 2);
    read_slots(c, S_SEL2, 1);
    const uint64_t nk = c.h_slots[S_SEL2];
    if (nk) {
        k_acc_kept_pos<<<grid_for(nk, kAB), kAB, 0, c.stream>>>(P, K, nk, d_kept);
        SKY_LAUNCH_CHECK();
        note_launch(c);
    }
    return nk;
}

}  // namespace skygpu
