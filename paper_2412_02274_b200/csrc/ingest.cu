// ingest.cu — device-side input preparation: the
// reference's min-max normalisation (harness.cpp:161-177) and its
// representative selection (partition.cpp:229-271), so a relation can go
// from raw values to the skyline without a host pass over it.
//
// normalize: per attribute lo = min, hi = max; value (v - lo) / (hi - lo), or
// 0 for a constant attribute.  IEEE subtraction and division in the same
// order as the reference, no FMA: bit-identical.
//
// select_representatives: the k best tuples by (sum, id) — the reference's
// bounded max-heap keeps exactly the k smallest under that total order —
// then, in (sum, id) order, a pick is dropped when another pick dominates it
// (partition.cpp:229-245).  The DominanceCounter total is reproduced too: pick
// i tests the other picks in order until the first dominator, so it adds the
// 1-based index of that dominator among the others (or k - 1).
#include <cub/cub.cuh>

#include "sky_common.cuh"

namespace skygpu {
namespace {

constexpr int kIB = 256;

// Per attribute: min and max (order-preserving bits of the non-negative
// values), and the first position holding a zero — std::min keeps the FIRST
// of equal candidates, so when the minimum is zero the reference's lo carries
// the sign of the first zero in input order (-0.0 or +0.0).
__global__ void k_col_minmax(const double* __restrict__ v, uint64_t n, int d,
                             unsigned long long* __restrict__ lo_bits,
                             unsigned long long* __restrict__ hi_bits,
                             unsigned long long* __restrict__ first_zero) {
    for (int j = blockIdx.y; j < d; j += gridDim.y) {
        unsigned long long lo = ~0ULL, hi = 0, fz = ~0ULL;
        for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
             i += (uint64_t)gridDim.x * blockDim.x) {
            const double x = v[i * d + j];
            const unsigned long long b = ord_bits(x);
            lo = b < lo ? b : lo;
            hi = b > hi ? b : hi;
            if (x == 0.0 && i < fz) fz = i;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long x = __shfl_down_sync(0xffffffffu, lo, o);
            const unsigned long long y = __shfl_down_sync(0xffffffffu, hi, o);
            lo = x < lo ? x : lo;
            hi = y > hi ? y : hi;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long z = __shfl_down_sync(0xffffffffu, fz, o);
            fz = z < fz ? z : fz;
        }
        if ((threadIdx.x & 31) == 0) {
            atomicMin(&lo_bits[j], lo);
            atomicMax(&hi_bits[j], hi);
            atomicMin(&first_zero[j], fz);
        }
    }
}

__global__ void k_normalize(const double* __restrict__ v, uint64_t n, int d,
                            const unsigned long long* __restrict__ lo_bits,
                            const unsigned long long* __restrict__ hi_bits,
                            const unsigned long long* __restrict__ first_zero,
                            double* __restrict__ out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n * d;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const int j = (int)(i % d);
        double lo = __longlong_as_double((long long)lo_bits[j]);
        if (lo == 0.0) lo = v[first_zero[j] * d + j];  // the sign of the first zero
        const double hi = __longlong_as_double((long long)hi_bits[j]);
        out[i] = hi > lo ? __ddiv_rn(__dsub_rn(v[i], lo), __dsub_rn(hi, lo)) : 0.0;
    }
}

__global__ void k_score_id(const double* __restrict__ v, const int64_t* __restrict__ ids,
                           uint64_t n, int d, unsigned long long* __restrict__ key,
                           unsigned long long* __restrict__ idkey, uint32_t* __restrict__ pos) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int k = 0; k < d; ++k) s = __dadd_rn(s, v[i * d + k]);
        key[i] = ord_bits(s);
        idkey[i] = (unsigned long long)ids[i] ^ 0x8000000000000000ULL;  // signed order
        pos[i] = (uint32_t)i;
    }
}

__global__ void k_gather_u64(const unsigned long long* __restrict__ a,
                             const uint32_t* __restrict__ idx, uint64_t n,
                             unsigned long long* __restrict__ o) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        o[i] = a[idx[i]];
}

// one thread per pick: dominated by another pick?  tests = 1-based index of
// the first dominating pick among the others in order, else k - 1
__global__ void k_rep_prune(const double* __restrict__ v, int d, const uint32_t* __restrict__ pick,
                            uint32_t k, uint8_t* __restrict__ keep,
                            unsigned long long* __restrict__ tests) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < k; i += gridDim.x * blockDim.x) {
        const double* t = v + (uint64_t)pick[i] * d;
        uint32_t tested = 0;
        bool dom = false;
        for (uint32_t j = 0; j < k && !dom; ++j) {
            if (j == i) continue;
            ++tested;
            dom = dom_f64_dyn(v + (uint64_t)pick[j] * d, t, d);
        }
        keep[i] = dom ? 0 : 1;
        atomicAdd(tests, (unsigned long long)tested);
    }
}

}  // namespace

void normalize_device(Ctx& c, const double* d_in, uint64_t n, int d, double* d_out) {
    if (n == 0) return;
    auto* lo = c.buf[B_ACC0].as<unsigned long long>(3 * kMaxDims);
    auto* hi = lo + kMaxDims;
    auto* fz = hi + kMaxDims;
    SKY_CUDA(cudaMemsetAsync(lo, 0xFF, sizeof(unsigned long long) * kMaxDims, c.stream));
    SKY_CUDA(cudaMemsetAsync(hi, 0, sizeof(unsigned long long) * kMaxDims, c.stream));
    SKY_CUDA(cudaMemsetAsync(fz, 0xFF, sizeof(unsigned long long) * kMaxDims, c.stream));
    k_col_minmax<<<dim3(grid_for(n, kIB, 296), (unsigned)d), kIB, 0, c.stream>>>(d_in, n, d, lo,
                                                                                 hi, fz);
    k_normalize<<<grid_for(n * d, kIB), kIB, 0, c.stream>>>(d_in, n, d, lo, hi, fz, d_out);
    SKY_LAUNCH_CHECK();
    note_launch(c, 2);
}

uint64_t select_representatives_device(Ctx& c, const double* d_vals, const int64_t* d_ids,
                                       uint64_t n, int d, uint64_t k, uint32_t* d_out,
                                       unsigned long long* d_tests) {
    if (k == 0 || n == 0) return 0;
    k = k < n ? k : n;
    auto* key = c.buf[B_ACC1].as<unsigned long long>(n);
    auto* kalt = c.buf[B_ACC2].as<unsigned long long>(n);
    auto* idk = c.buf[B_ACC3].as<unsigned long long>(n);
    uint32_t* p0 = c.buf[B_ACC4].as<uint32_t>(n);
    uint32_t* p1 = c.buf[B_ACC5].as<uint32_t>(n);
    k_score_id<<<grid_for(n, kIB), kIB, 0, c.stream>>>(d_vals, d_ids, n, d, key, idk, p0);
    SKY_LAUNCH_CHECK();
    note_launch(c);
    // (sum, id) order by two stable LSD passes: id first, then the sum key
    auto sort = [&](unsigned long long* k0, uint32_t*& v0, uint32_t*& v1) {
        cub::DoubleBuffer<unsigned long long> kb(k0, kalt);
        cub::DoubleBuffer<uint32_t> vb(v0, v1);
        size_t tmp = 0;
        SKY_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, kb, vb, (int64_t)n, 0, 64, c.stream));
        void* t = c.buf[B_CUB].get(tmp);
        SKY_CUDA(cub::DeviceRadixSort::SortPairs(t, tmp, kb, vb, (int64_t)n, 0, 64, c.stream));
        v0 = vb.Current();
        v1 = vb.Alternate();
        note_launch(c, 4);
    };
    sort(idk, p0, p1);
    auto* ks = c.buf[B_ACC6].as<unsigned long long>(n);
    k_gather_u64<<<grid_for(n, kIB), kIB, 0, c.stream>>>(key, p0, n, ks);
    SKY_LAUNCH_CHECK();
    note_launch(c);
    sort(ks, p0, p1);
    // the k best, then the pairwise pruning among them
    uint8_t* keep = c.buf[B_ACC7].as<uint8_t>(k);
    k_rep_prune<<<grid_for(k, kIB), kIB, 0, c.stream>>>(d_vals, d, p0, (uint32_t)k, keep, d_tests);
    SKY_LAUNCH_CHECK();
    note_launch(c);
    size_t tmp = 0;
    SKY_CUDA(cub::DeviceSelect::Flagged(nullptr, tmp, p0, keep, d_out, c.d_slots + S_SEL2,
                                         (int64_t)k, c.stream));
    void* t = c.buf[B_CUB].get(tmp);
    SKY_CUDA(cub::DeviceSelect::Flagged(t, tmp, p0, keep, d_out, c.d_slots + S_SEL2, (int64_t)k,
                                         c.stream));
    note_launch(c, 2);
    read_slots(c, S_SEL2, 1);
    return c.h_slots[S_SEL2];
}

}  // namespace skygpu
