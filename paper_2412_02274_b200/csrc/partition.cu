// partition.cu — the paper's partitioning on sm_100a (north_star (c),
// SURVEY.md §8 a7 + a10).
//
// Reference: parallel_skyline (proj/src/parallel.cpp:22-101) assigns every
// tuple a partition (assign_partitions, partition.cpp:183-213), runs one SFS
// per partition on an OpenMP pool (parallel.cpp:59-73) and merges the union of
// the local skylines with one more SFS (parallel.cpp:83-86).
//
// GPU recast — local-skyline PRUNING before the merge:
//   P1 pid       assign_partitions on the device: grid cells (partition.cpp:
//                85-109), hyperspherical angles (:139-174), or equal-count
//                slices of the (attribute 0, id) order (:176-181, one CUB
//                radix sort).  Bit-exact with the reference for grid and
//                sliced; angular uses the device atan2 (the ids may differ
//                from glibc's in the last ulp at a slice boundary — results
//                are plan-invariant, acceptance_main.cpp:145-184).
//   P2 window    per partition, a window of its lowest-sum tuples: a sampled
//                (partition x sum-bucket) histogram picks a per-partition
//                bucket threshold; the tuples below it are scattered into the
//                partition's window (at most kWinCap, the excess is simply
//                not a window member — any subset of a partition is a valid
//                set of dominators).
//   P3 reduce    one CTA per partition: the window's own skyline (members
//                dominated by a preceding member dropped), ranked by (sum,
//                tie) so the strongest dominators come first.
//   P4 filter    every tuple against its partition's window skyline: a tuple
//                dominated by a PRECEDING (in (sum, id) order) member of its
//                own partition cannot be in the local skyline, nor — by the
//                predecessor rule the merge implements (skyline.cu header) —
//                in the result, so it is dropped before the merge.
// The survivors (a superset of the union of local skylines; every local
// skyline tuple survives) feed the exact merge engine (prefix rounds or rank
// grid), which decides them by the predecessor rule.  Dropping a tuple u that
// a preceding tuple w dominates never changes another tuple's verdict: if u
// dominated t, so does w, and w (or, by induction, w's earliest undropped
// dominator) precedes t.
#include <cub/cub.cuh>

#include "sky_common.cuh"

namespace skygpu {

namespace {

constexpr double kPi = 3.14159265358979323846;  // partition.cpp:13
constexpr int kPBlock = 256;
constexpr int kBuckets = 256;      // sum buckets per partition (window threshold)
constexpr uint32_t kWinCap = 1024;  // window members per partition (P3 is one CTA)
constexpr uint32_t kMaxLocalParts = 4096;

template <class F>
void dispatch_dims(int d, F&& f) {
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

// ------------------------------------------------------------------ P1 pid
// grid_cell + cell_partition_id (partition.cpp:85-109); values outside [0,1]
// report the first offending flat index (S_GRIDBAD) for the reference's error
template <int D>
__global__ void k_pid_grid(const double* __restrict__ v, uint64_t n, int d, int m,
                           int32_t* __restrict__ pid, unsigned long long* __restrict__ slots) {
    pdl_wait();
    const int dd = D > 0 ? D : d;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        long long id = 0, w = 1;
#pragma unroll(D > 0 ? D : 1)
        for (int k = 0; k < dd; ++k) {
            const double x = v[i * dd + k];
            if (x < 0.0 || x > 1.0)
                atomicMin(&slots[S_GRIDBAD], (unsigned long long)(i * dd + k));
            int idx = (int)__dmul_rn(x, (double)m);
            if (idx >= m) idx = m - 1;
            if (idx < 0) idx = 0;
            id += (long long)idx * w;
            w *= m;
        }
        pid[i] = (int32_t)id;
    }
}

// assign_angular + to_hyperspherical (partition.cpp:139-174): tail norms
// accumulated from the last attribute, angle_i = atan2(sqrt(tail[i+1]), v_i),
// slice = int((2 angle / pi) * m) clamped; the origin goes to partition 0
template <int D>
__global__ void k_pid_angular(const double* __restrict__ v, uint64_t n, int d, int m,
                              int32_t* __restrict__ pid) {
    pdl_wait();
    const int dd = D > 0 ? D : d;
    constexpr int DT = D > 0 ? D + 1 : kMaxDims + 1;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const double* t = v + i * dd;
        double tail[DT];
        tail[dd] = 0.0;
        bool all_zero = true;
#pragma unroll(D > 0 ? D : 1)
        for (int k = dd - 1; k >= 0; --k) {
            const double x = t[k];
            all_zero &= (x == 0.0);
            tail[k] = __dadd_rn(tail[k + 1], __dmul_rn(x, x));
        }
        long long id = 0, w = 1;
        if (!all_zero) {
#pragma unroll(D > 0 ? D : 1)
            for (int k = 0; k + 1 < dd; ++k) {
                const double ang = atan2(__dsqrt_rn(tail[k + 1]), t[k]);
                int idx = (int)__dmul_rn(__ddiv_rn(__dmul_rn(2.0, ang), kPi), (double)m);
                if (idx >= m) idx = m - 1;
                id += (long long)idx * w;
                w *= m;
            }
        }
        pid[i] = (int32_t)id;
    }
}

// sliced (partition.cpp:176-213): the radix-sort key of attribute 0 (-0.0 as
// +0.0, so equal values tie and fall back to the id order)
__global__ void k_attr0_keys(const double* __restrict__ v, uint64_t n, int d,
                             const uint32_t* __restrict__ order,
                             unsigned long long* __restrict__ key) {
    pdl_wait();
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t p = order ? order[i] : i;
        const double x = v[p * d];
        unsigned long long b = x == 0.0 ? 0ULL : (unsigned long long)__double_as_longlong(x);
        b = (b >> 63) ? ~b : (b | 0x8000000000000000ULL);  // total order of doubles
        key[i] = b;
    }
}

__global__ void k_id_sort_keys(const int64_t* __restrict__ ids, uint64_t n,
                               unsigned long long* __restrict__ key, uint32_t* __restrict__ pos) {
    pdl_wait();
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        key[i] = (unsigned long long)ids[i] ^ 0x8000000000000000ULL;  // signed order
        pos[i] = (uint32_t)i;
    }
}

__global__ void k_iota_u32(uint32_t* __restrict__ a, uint64_t n) {
    pdl_wait();
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        a[i] = (uint32_t)i;
}

__global__ void k_pid_sliced(const uint32_t* __restrict__ order, uint64_t n, long long parts,
                             int32_t* __restrict__ pid) {
    pdl_wait();
    for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < n;
         r += (uint64_t)gridDim.x * blockDim.x)
        pid[order[r]] = (int32_t)((long long)r * parts / (long long)n);  // (rank-1)*p/n
}

// ------------------------------------------------------------ P2 windows
__device__ __forceinline__ int sum_bucket(unsigned long long key, double lo, double inv) {
    const double s = __longlong_as_double((long long)key);
    if (!(s > lo)) return 0;
    const double f = (s - lo) * inv;
    return f >= (double)(kBuckets - 1) ? kBuckets - 1 : (int)f;
}

__device__ __forceinline__ void bucket_range(const unsigned long long* slots, double* lo,
                                             double* inv) {
    const unsigned long long a = slots[S_SMIN], b = slots[S_SMAX];
    *lo = a == ~0ULL ? 0.0 : __longlong_as_double((long long)a);
    const double hi = __longlong_as_double((long long)b);
    *inv = hi > *lo ? (double)kBuckets / (hi - *lo) : 0.0;
}

// sampled (partition x sum bucket) histogram: every `stride`-th tuple
__global__ void k_win_hist(const unsigned long long* __restrict__ key,
                           const int32_t* __restrict__ pid, const uint8_t* __restrict__ mask,
                           uint64_t n, uint32_t stride, const unsigned long long* __restrict__ slots,
                           uint32_t* __restrict__ hist) {
    pdl_wait();
    double lo, inv;
    bucket_range(slots, &lo, &inv);
    const uint64_t ns = (n + stride - 1) / stride;
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < ns;
         j += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t i = j * stride;
        if (mask && !mask[i]) continue;
        atomicAdd(&hist[(uint64_t)pid[i] * kBuckets + sum_bucket(key[i], lo, inv)], 1u);
    }
}

// per partition: the smallest bucket threshold whose sampled count reaches
// the window target; zero the window cursors
__global__ void k_win_thresh(const uint32_t* __restrict__ hist, uint32_t parts, uint32_t want,
                             uint32_t* __restrict__ thr, uint32_t* __restrict__ cur) {
    pdl_wait();
    for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < parts;
         p += gridDim.x * blockDim.x) {
        const uint32_t* h = hist + (uint64_t)p * kBuckets;
        uint32_t cum = 0, b = 0;
        while (b < kBuckets && cum < want) cum += h[b++];
        thr[p] = b == 0 ? 1 : b;
        cur[p] = 0;
    }
}

// window members: the tuples below their partition's threshold (first come,
// first served up to kWinCap)
__global__ void k_win_scatter(const unsigned long long* __restrict__ key,
                              const int32_t* __restrict__ pid, const uint8_t* __restrict__ mask,
                              uint64_t n, const unsigned long long* __restrict__ slots,
                              const uint32_t* __restrict__ thr, uint32_t* __restrict__ cur,
                              uint32_t* __restrict__ wpos) {
    pdl_wait();
    double lo, inv;
    bucket_range(slots, &lo, &inv);
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        if (mask && !mask[i]) continue;
        const int32_t p = pid[i];
        if (sum_bucket(key[i], lo, inv) >= (int)thr[p]) continue;
        const uint32_t s = atomicAdd(&cur[p], 1u);
        if (s < kWinCap) wpos[(uint64_t)p * kWinCap + s] = (uint32_t)i;
    }
}

// (sum, tie) strict precedence: the reference's SFS order (core.cpp:53-56);
// ties are ids, or input positions while the ids are still in flight
__device__ __forceinline__ bool precedes(unsigned long long ka, long long ta,
                                         unsigned long long kb, long long tb) {
    return ka < kb || (ka == kb && ta < tb);
}

// ------------------------------------------------------------ P3 reduce
// one CTA per partition: the window's skyline, ranked by (sum, tie), written
// AoS + keys + ties; wcnt[p] = its size
template <int D>
__global__ void __launch_bounds__(kPBlock)
k_win_reduce(const double* __restrict__ v, int d, const unsigned long long* __restrict__ key,
             const int64_t* __restrict__ tie_ids, const uint32_t* __restrict__ cur,
             const uint32_t* __restrict__ wpos, double* __restrict__ wv,
             unsigned long long* __restrict__ wkey, long long* __restrict__ wtie,
             uint32_t* __restrict__ wcnt, unsigned long long* __restrict__ tests) {
    pdl_wait();
    extern __shared__ __align__(16) unsigned char smem[];
    const int dd = D > 0 ? D : d;
    const uint32_t p = blockIdx.x;
    const uint32_t m = min(cur[p], kWinCap);
    double* sv = reinterpret_cast<double*>(smem);                    // [dd][kWinCap]
    unsigned long long* sk = reinterpret_cast<unsigned long long*>(sv + (size_t)dd * kWinCap);
    long long* st = reinterpret_cast<long long*>(sk + kWinCap);
    uint32_t* sidx = reinterpret_cast<uint32_t*>(st + kWinCap);      // survivor list
    __shared__ uint32_t nsurv;
    if (threadIdx.x == 0) nsurv = 0;
    for (uint32_t a = threadIdx.x; a < m; a += blockDim.x) {
        const uint32_t i = wpos[(uint64_t)p * kWinCap + a];
        for (int k = 0; k < dd; ++k) sv[(size_t)k * kWinCap + a] = v[(uint64_t)i * dd + k];
        sk[a] = key[i];
        st[a] = tie_ids ? (long long)tie_ids[i] : (long long)i;
    }
    __syncthreads();
    unsigned long long ntest = 0;
    for (uint32_t a = threadIdx.x; a < m; a += blockDim.x) {
        const unsigned long long ka = sk[a];
        const long long ta = st[a];
        bool dom = false;
        for (uint32_t b = 0; b < m && !dom; ++b) {
            if (!precedes(sk[b], st[b], ka, ta)) continue;
            ++ntest;
            bool le = true, lt = false;
            for (int k = 0; k < dd; ++k) {
                const double x = sv[(size_t)k * kWinCap + b], y = sv[(size_t)k * kWinCap + a];
                le &= x <= y;
                lt |= x < y;
            }
            dom = le & lt;
        }
        if (!dom) sidx[atomicAdd(&nsurv, 1u)] = a;
    }
    __syncthreads();
    const uint32_t ns = nsurv;
    // rank among the survivors by (sum, tie): strongest dominators first
    for (uint32_t j = threadIdx.x; j < ns; j += blockDim.x) {
        const uint32_t a = sidx[j];
        uint32_t rank = 0;
        for (uint32_t q = 0; q < ns; ++q) {
            const uint32_t b = sidx[q];
            rank += precedes(sk[b], st[b], sk[a], st[a]);
        }
        const uint64_t o = (uint64_t)p * kWinCap + rank;
        for (int k = 0; k < dd; ++k) wv[o * dd + k] = sv[(size_t)k * kWinCap + a];
        wkey[o] = sk[a];
        wtie[o] = st[a];
    }
    if (threadIdx.x == 0) wcnt[p] = ns;
    add_count(tests, ntest);
}

// ------------------------------------------------------------ P4 filter
// keep[i] = 1 iff tuple i (in the mask) is not dominated by a preceding
// member of its partition's window skyline
template <int D>
__global__ void __launch_bounds__(kPBlock)
k_local_filter(const double* __restrict__ v, uint64_t n, int d,
               const unsigned long long* __restrict__ key, const int64_t* __restrict__ tie_ids,
               const int32_t* __restrict__ pid, const uint8_t* __restrict__ mask,
               const double* __restrict__ wv, const unsigned long long* __restrict__ wkey,
               const long long* __restrict__ wtie, const uint32_t* __restrict__ wcnt,
               uint8_t* __restrict__ keep, unsigned long long* __restrict__ tests,
               uint32_t sample, unsigned long long* __restrict__ slots) {
    pdl_wait();
    const int dd = D > 0 ? D : d;
    constexpr int DA = D > 0 ? D : kMaxDims;
    unsigned long long ntest = 0;
    // sample > 0: the probe pass — every sample-th tuple, counted in
    // S_LPS_N / S_LPS_HIT, keep untouched.  sample == 0: the full pass; when
    // the probe saw the windows dominate under a quarter of its tuples (a
    // skyline-heavy relation: C5 loses 3 % of its tuples to 64 partitions'
    // windows for 37 ms of scans) nothing is pruned here and the merge engine
    // decides everything — pruning any subset is valid.
    const uint64_t step = sample ? sample : 1;
    const uint64_t cnt = (n + step - 1) / step;
    const bool idle = !sample && slots[S_LPS_HIT] * 4 < slots[S_LPS_N];
    unsigned long long nprobe = 0, nhit = 0;
    for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < cnt;
         q += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t i = q * step;
        if (mask && !mask[i]) {
            if (!sample) keep[i] = 0;
            continue;
        }
        if (idle) {
            keep[i] = 1;
            continue;
        }
        const uint32_t p = (uint32_t)pid[i];
        const unsigned long long ki = key[i];
        const long long ti = tie_ids ? (long long)tie_ids[i] : (long long)i;
        double t[DA];
#pragma unroll(D > 0 ? D : 1)
        for (int k = 0; k < dd; ++k) t[k] = v[i * dd + k];
        const uint32_t m = wcnt[p];
        const uint64_t base = (uint64_t)p * kWinCap;
        bool dom = false;
        for (uint32_t j = 0; j < m; ++j) {
            const unsigned long long kj = wkey[base + j];
            if (kj > ki) break;  // ranked by sum: no later member precedes i
            if (!precedes(kj, wtie[base + j], ki, ti)) continue;
            ++ntest;
            const double* s = wv + (base + j) * dd;
            bool le = true, lt = false;
#pragma unroll(D > 0 ? D : 1)
            for (int k = 0; k < dd; ++k) {
                le &= s[k] <= t[k];
                lt |= s[k] < t[k];
            }
            if (le & lt) {
                dom = true;
                break;
            }
        }
        if (sample) {
            ++nprobe;
            nhit += dom;
        } else {
            keep[i] = !dom;
        }
    }
    add_count(tests, ntest);
    if (sample) {
        add_count(slots + S_LPS_N, nprobe);
        add_count(slots + S_LPS_HIT, nhit);
    }
}

template <class KT>
void radix_pairs(Ctx& c, KT* k0, KT* k1, uint32_t* v0, uint32_t* v1, uint64_t n,
                 uint32_t** vout) {
    cub::DoubleBuffer<KT> kb(k0, k1);
    cub::DoubleBuffer<uint32_t> vb(v0, v1);
    size_t tmp = 0;
    SKY_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, kb, vb, (int64_t)n, 0, 64, c.stream));
    void* t = c.buf[B_CUB].get(tmp);
    SKY_CUDA(cub::DeviceRadixSort::SortPairs(t, tmp, kb, vb, (int64_t)n, 0, 64, c.stream));
    note_launch(c, 4);
    *vout = vb.Current();
}

}  // namespace

// the plan's partition ids must index [0, partitions): slices^d (grid),
// slices^(d-1) (angular) — a hand-built inconsistent plan is not pruned
bool plan_ids_in_range(const skygpu_plan& plan, int d) {
    if (plan.partitions < 1) return false;
    if (plan.strategy != SKYGPU_GRID && plan.strategy != SKYGPU_ANGULAR) return true;
    if (plan.slices < 1) return false;
    const int e = plan.strategy == SKYGPU_GRID ? d : d - 1;
    long long v = 1;
    for (int k = 0; k < e; ++k) {
        v *= plan.slices;
        if (v > plan.partitions) return false;
    }
    return v <= plan.partitions;
}

bool local_prune_applies(const skygpu_plan& plan, int d) {
    return d >= 1 && d <= 8 && plan.partitions >= 1 &&
           (uint64_t)plan.partitions <= kMaxLocalParts && plan_ids_in_range(plan, d) &&
           !(plan.strategy == SKYGPU_ANGULAR && d < 2);
}

void assign_partitions_device(Ctx& c, const double* d_vals, const int64_t* d_ids, bool ids_sorted,
                              uint64_t n, int d, const skygpu_plan& plan, int32_t* d_pid) {
    if (n == 0) return;
    const unsigned gb = grid_for(n, kPBlock, c.num_sms * 16);
    switch (plan.strategy) {
        case SKYGPU_GRID:
            dispatch_dims(d, [&](auto DC) {
                constexpr int D = decltype(DC)::value;
                pdl_launch(k_pid_grid<D>, gb, kPBlock, 0, c.stream, d_vals, n, d, plan.slices,
                           d_pid, c.d_slots);
            });
            SKY_LAUNCH_CHECK();
            note_launch(c);
            break;
        case SKYGPU_ANGULAR:
            dispatch_dims(d, [&](auto DC) {
                constexpr int D = decltype(DC)::value;
                pdl_launch(k_pid_angular<D>, gb, kPBlock, 0, c.stream, d_vals, n, d, plan.slices,
                           d_pid);
            });
            SKY_LAUNCH_CHECK();
            note_launch(c);
            break;
        case SKYGPU_SLICED: {
            // positions ordered by (attribute 0, id): CUB's radix sort is
            // stable, so with ids strictly increasing in position order one
            // sort of the positions by attribute 0 suffices; otherwise sort
            // by id first (LSD)
            auto* k0 = c.buf[B_PSK0].as<unsigned long long>(n);
            auto* k1 = c.buf[B_PSK1].as<unsigned long long>(n);
            uint32_t* v0 = c.buf[B_PSV0].as<uint32_t>(n);
            uint32_t* v1 = c.buf[B_PSV1].as<uint32_t>(n);
            const bool by_id = !ids_sorted && d_ids;
            if (by_id) {
                pdl_launch(k_id_sort_keys, gb, kPBlock, 0, c.stream, d_ids, n, k0, v1);
                SKY_LAUNCH_CHECK();
                note_launch(c);
                uint32_t* o = nullptr;
                radix_pairs<unsigned long long>(c, k0, k1, v1, v0, n, &o);
                if (o != v0)
                    SKY_CUDA(cudaMemcpyAsync(v0, o, n * sizeof(uint32_t), cudaMemcpyDeviceToDevice,
                                             c.stream));
            } else {
                pdl_launch(k_iota_u32, gb, kPBlock, 0, c.stream, v0, n);
                SKY_LAUNCH_CHECK();
                note_launch(c);
            }
            // v0 = positions in id order; their attribute-0 keys into k0
            pdl_launch(k_attr0_keys, gb, kPBlock, 0, c.stream, d_vals, n, d,
                       (const uint32_t*)v0, k0);
            SKY_LAUNCH_CHECK();
            note_launch(c);
            uint32_t* order = nullptr;
            radix_pairs<unsigned long long>(c, k0, k1, v0, v1, n, &order);
            pdl_launch(k_pid_sliced, gb, kPBlock, 0, c.stream, (const uint32_t*)order, n,
                       plan.partitions, d_pid);
            SKY_LAUNCH_CHECK();
            note_launch(c);
            break;
        }
        default:
            SKY_CUDA(cudaMemsetAsync(d_pid, 0, n * sizeof(int32_t), c.stream));
    }
}

uint64_t local_prune_device(Ctx& c, const double* d_vals, const unsigned long long* keys,
                            const int64_t* tie_ids, uint64_t n, int d, const skygpu_plan& plan,
                            const uint8_t* mask, uint8_t* keep, uint32_t* stats_parts) {
    const uint32_t parts = (uint32_t)plan.partitions;
    int32_t* pid = c.buf[B_PPID].as<int32_t>(n);
    // (sliced ties: by position; a pruning heuristic needs no exact ids, the
    // precedence tests below use the real tie order)
    assign_partitions_device(c, d_vals, nullptr, true, n, d, plan, pid);
    uint32_t* hist = c.buf[B_PHIST].as<uint32_t>((uint64_t)parts * kBuckets);
    uint32_t* thr = c.buf[B_PTHR].as<uint32_t>(2 * (uint64_t)parts + parts);
    uint32_t* cur = thr + parts;
    uint32_t* wcnt = cur + parts;
    uint32_t* wpos = c.buf[B_PWPOS].as<uint32_t>((uint64_t)parts * kWinCap);
    double* wv = c.buf[B_PWV].as<double>((uint64_t)parts * kWinCap * d);
    auto* wkey = c.buf[B_PWKEY].as<unsigned long long>((uint64_t)parts * kWinCap);
    auto* wtie = c.buf[B_PWTIE].as<long long>((uint64_t)parts * kWinCap);
    SKY_CUDA(cudaMemsetAsync(hist, 0, (uint64_t)parts * kBuckets * sizeof(uint32_t), c.stream));
    // window target: ~256 tuples per partition, from a sample of ~1/8 of n
    static const uint32_t want_total = [] {
        const char* e = getenv("SKYGPU_LOCAL_WINDOW");
        const long long v = e ? atoll(e) : 0;
        return v > 0 && v <= (long long)kWinCap ? (uint32_t)v : 256u;
    }();
    const uint64_t per_part = n / parts;
    const uint32_t stride = per_part >= 65536 ? 16 : (per_part >= 8192 ? 4 : 1);
    const uint32_t want = (want_total + stride - 1) / stride;
    const unsigned gb = grid_for(n, kPBlock, c.num_sms * 16);
    pdl_launch(k_win_hist, grid_for((n + stride - 1) / stride, kPBlock, c.num_sms * 16), kPBlock,
               0, c.stream, keys, (const int32_t*)pid, mask, n, stride,
               (const unsigned long long*)c.d_slots, hist);
    SKY_LAUNCH_CHECK();
    pdl_launch(k_win_thresh, grid_for(parts, kPBlock), kPBlock, 0, c.stream,
               (const uint32_t*)hist, parts, want, thr, cur);
    SKY_LAUNCH_CHECK();
    pdl_launch(k_win_scatter, gb, kPBlock, 0, c.stream, keys, (const int32_t*)pid, mask, n,
               (const unsigned long long*)c.d_slots, (const uint32_t*)thr, cur, wpos);
    SKY_LAUNCH_CHECK();
    note_launch(c, 3);
    const size_t smem = (size_t)kWinCap * (d * 8 + 8 + 8 + 4);
    dispatch_dims(d, [&](auto DC) {
        constexpr int D = decltype(DC)::value;
        SKY_CUDA(cudaFuncSetAttribute(k_win_reduce<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem));
        pdl_launch(k_win_reduce<D>, parts, kPBlock, smem, c.stream, d_vals, d, keys, tie_ids,
                   (const uint32_t*)cur, (const uint32_t*)wpos, wv, wkey, wtie, wcnt,
                   c.d_slots + S_TESTS_SKY);
        SKY_LAUNCH_CHECK();
        // probe (every probe-th tuple, ~8k of them), then the full pass gated
        // on the probe's yield (SKYGPU_LOCAL_PROBE=0: always the full pass)
        static const bool probe_on = [] {
            const char* e = getenv("SKYGPU_LOCAL_PROBE");
            return !(e && e[0] == '0');
        }();
        const uint32_t probe = probe_on && n >= (1u << 18) ? (uint32_t)(n >> 13) : 0u;
        SKY_CUDA(cudaMemsetAsync(c.d_slots + S_LPS_N, 0, 2 * sizeof(unsigned long long),
                                 c.stream));
        if (probe) {
            pdl_launch(k_local_filter<D>, grid_for((n + probe - 1) / probe, kPBlock), kPBlock, 0,
                       c.stream, d_vals, n, d, keys, tie_ids, (const int32_t*)pid, mask,
                       (const double*)wv, (const unsigned long long*)wkey,
                       (const long long*)wtie, (const uint32_t*)wcnt, keep,
                       c.d_slots + S_TESTS_SKY, probe, c.d_slots);
            SKY_LAUNCH_CHECK();
            note_launch(c);
        }
        pdl_launch(k_local_filter<D>, gb, kPBlock, 0, c.stream, d_vals, n, d, keys, tie_ids,
                   (const int32_t*)pid, mask, (const double*)wv,
                   (const unsigned long long*)wkey, (const long long*)wtie,
                   (const uint32_t*)wcnt, keep, c.d_slots + S_TESTS_SKY, 0u, c.d_slots);
        SKY_LAUNCH_CHECK();
    });
    note_launch(c, 2);
    if (stats_parts) *stats_parts = parts;
    return parts;
}

}  // namespace skygpu
