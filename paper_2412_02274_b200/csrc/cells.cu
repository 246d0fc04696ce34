// cells.cu — the cell-occupancy gres engine.
//
// At step g a skyline tuple t is ejected iff some skyline tuple's code vector
// dominates t's (gres.cu header).  Equivalently: some OCCUPIED cell c' of the
// code grid satisfies c' <= c(t) componentwise and c' != c(t), i.e.
//     OR_j  P[c(t) - e_j]      (over j with c_j(t) >= 1)
// where P is the inclusive prefix-OR of the cell occupancy.  The cost per step
// is O(cells + S) instead of O(S^2): the right engine for huge skylines
// (ANT d=7 at n=10^7, where S ~ n and the pair engine needs ~10^15 tests).
//
// Layout: one bit per cell along attribute 0 (extent e_0 <= 64 -> a u32/u64
// word per "row"), rows indexed by attributes 1..d-1 (attribute 1 fastest).
// Per step: memset, mark (atomicOr per skyline tuple), the prefix-OR over
// every attribute, then one query per undecided candidate.  The prefix-OR is
// HBM-bound (every pass reads and writes every row once), so passes are
// fused: attributes 0 (in-word), 1 and 2 in one shared-memory slab pass,
// then the remaining attributes two at a time (k_cells_or_pair) — 3 passes
// for d = 7 instead of 7.  Exactness: the same codes floor(v*g) as the pair
// engine.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <vector>

#include "sky_common.cuh"

namespace skygpu {

namespace {

constexpr int kBlock = 256;
constexpr int kMaxCellDims = 16;

// Steps run back to back with no host round trip: each step's kernels read
// the previous step's undecided count (live) and return at once when it is
// zero (live == nullptr: the first step, always run).
__device__ __forceinline__ bool step_dead(const unsigned long long* live) {
    return live && *(volatile const unsigned long long*)live == 0ULL;
}

__global__ void k_clear_slot_c(unsigned long long* p) {
    pdl_wait();
    *p = 0;
}

// zero a step's grid (replaces a memset so that a dead step costs nothing)
__global__ void k_cells_zero(uint4* __restrict__ p, uint64_t n16, const unsigned long long* live) {
    pdl_wait();
    if (step_dead(live)) return;
    const uint4 z = make_uint4(0u, 0u, 0u, 0u);
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n16;
         i += (uint64_t)gridDim.x * blockDim.x)
        p[i] = z;
}

struct CellGeom {
    int d;
    int g;
    uint64_t rows;
    uint64_t stride[kMaxCellDims];  // stride of attribute j >= 1 in rows
    uint64_t ext[kMaxCellDims];     // code extent (max code + 1) of attribute j
};

template <class W>
__global__ void k_cells_mark(const double* __restrict__ v, uint64_t S, CellGeom geo,
                             W* __restrict__ rows, const unsigned long long* live) {
    pdl_wait();
    if (step_dead(live)) return;
    const double gd = (double)geo.g;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < S;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t r = 0;
        for (int j = 1; j < geo.d; ++j) r += (uint64_t)floor(__dmul_rn(v[j * S + i], gd)) * geo.stride[j];
        const W bit = (W)1 << (unsigned)floor(__dmul_rn(v[i], gd));
        if (!(rows[r] & bit)) atomicOr(&rows[r], bit);
    }
}

// prefix-OR inside each word: bit k |= bits 0..k-1 (attribute 0)
template <class W>
__global__ void k_cells_or_word(W* __restrict__ rows, uint64_t n, const unsigned long long* live) {
    pdl_wait();
    if (step_dead(live)) return;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        W x = rows[i];
        x |= x << 1;
        x |= x << 2;
        x |= x << 4;
        x |= x << 8;
        x |= x << 16;
        if (sizeof(W) == 8) x |= x << (sizeof(W) == 8 ? 32 : 0);
        rows[i] = x;
    }
}

// prefix-OR along attribute j: each thread sweeps one line of e_j rows;
// consecutive threads own consecutive lines (coalesced when stride >= 32)
template <class W>
__global__ void k_cells_or_dim(W* __restrict__ rows, uint64_t nrows, uint64_t ext,
                               uint64_t stride, const unsigned long long* live) {
    pdl_wait();
    if (step_dead(live)) return;
    const uint64_t lines = nrows / ext;
    for (uint64_t l = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; l < lines;
         l += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t lo = l % stride, hi = l / stride;
        W* p = rows + hi * stride * ext + lo;
        W acc = 0;
        for (uint64_t k = 0; k < ext; ++k) {
            acc |= p[k * stride];
            p[k * stride] = acc;
        }
    }
}

// ---- fused sweeps (the default): 3 passes instead of d for d = 7
template <class W>
__device__ __forceinline__ W word_prefix(W x) {
    x |= x << 1;
    x |= x << 2;
    x |= x << 4;
    x |= x << 8;
    x |= x << 16;
    if (sizeof(W) == 8) x |= x << (sizeof(W) == 8 ? 32 : 0);
    return x;
}

// attribute 0 (in-word) + attributes 1 and 2 (e2 = 1 when d == 2): the
// slab of e1*e2 rows of fixed attributes 3.. is contiguous; a block stages
// whole slabs in shared memory (coalesced), sweeps them there, writes back
constexpr uint32_t kSlabWords = 4096;

template <class W>
__global__ void __launch_bounds__(kBlock)
k_cells_or_slab(W* __restrict__ rows, uint64_t nrows, uint32_t e1, uint32_t e2,
                uint32_t spb, const unsigned long long* live) {
    pdl_wait();
    if (step_dead(live)) return;
    extern __shared__ __align__(16) unsigned char smraw[];
    W* sm = reinterpret_cast<W*>(smraw);
    const uint32_t slab = e1 * e2;
    const uint64_t nslabs = nrows / slab;
    constexpr uint32_t kPer = 16 / sizeof(W);  // words per 16-byte vector
    // 16-byte vector loads/stores when every batch starts 16-byte aligned
    // (spb * slab a multiple of kPer words): 4x fewer memory instructions,
    // more bytes in flight per thread
    const bool vec = (spb * slab) % kPer == 0;
    for (uint64_t s0 = (uint64_t)blockIdx.x * spb; s0 < nslabs; s0 += (uint64_t)gridDim.x * spb) {
        const uint32_t ns = (uint32_t)min((uint64_t)spb, nslabs - s0);
        const uint32_t words = ns * slab;
        W* g = rows + s0 * slab;
        const uint32_t nv = vec ? words / kPer : 0;
        for (uint32_t i = threadIdx.x; i < nv; i += blockDim.x) {
            uint4 x = reinterpret_cast<const uint4*>(g)[i];
            W* w = reinterpret_cast<W*>(&x);
#pragma unroll
            for (uint32_t k = 0; k < kPer; ++k) w[k] = word_prefix(w[k]);
            reinterpret_cast<uint4*>(sm)[i] = x;
        }
        for (uint32_t i = nv * kPer + threadIdx.x; i < words; i += blockDim.x)
            sm[i] = word_prefix(g[i]);
        __syncthreads();
        for (uint32_t l = threadIdx.x; l < ns * e2; l += blockDim.x) {  // attribute 1
            W* p = sm + (uint64_t)l * e1;
            W acc = 0;
            for (uint32_t a = 0; a < e1; ++a) {
                acc |= p[a];
                p[a] = acc;
            }
        }
        __syncthreads();
        if (e2 > 1) {
            for (uint32_t l = threadIdx.x; l < ns * e1; l += blockDim.x) {  // attribute 2
                W* p = sm + (uint64_t)(l / e1) * slab + (l % e1);
                W acc = 0;
                for (uint32_t b = 0; b < e2; ++b) {
                    acc |= p[b * e1];
                    p[b * e1] = acc;
                }
            }
            __syncthreads();
        }
        for (uint32_t i = threadIdx.x; i < nv; i += blockDim.x)
            reinterpret_cast<uint4*>(g)[i] = reinterpret_cast<const uint4*>(sm)[i];
        for (uint32_t i = nv * kPer + threadIdx.x; i < words; i += blockDim.x) g[i] = sm[i];
        __syncthreads();
    }
}

// two attributes a, b = a + 1 at once (stride sa, sb = sa * ea): one thread
// per line of the (ea x eb) plane, consecutive threads on consecutive lo
// (coalesced); P[x][y] = v[x][y] | P[x-1][y] | P[x][y-1], a row of ea words
// loaded ahead (ILP) and the previous row's prefixes held in registers
constexpr int kPairMax = 32;

template <class W>
__global__ void __launch_bounds__(kBlock)
k_cells_or_pair(W* __restrict__ rows, uint64_t nrows, uint32_t ea, uint32_t eb, uint64_t sa,
                const unsigned long long* live) {
    pdl_wait();
    if (step_dead(live)) return;
    const uint64_t plane = (uint64_t)ea * eb;
    const uint64_t lines = nrows / plane;
    for (uint64_t l = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; l < lines;
         l += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t lo = l % sa, hi = l / sa;
        W* base = rows + hi * sa * plane + lo;
        W prev[kPairMax];
#pragma unroll
        for (int x = 0; x < kPairMax; ++x) prev[x] = 0;
        for (uint32_t y = 0; y < eb; ++y) {
            W* p = base + (uint64_t)y * ea * sa;
            W v[kPairMax];
#pragma unroll
            for (int x = 0; x < kPairMax; ++x) v[x] = (uint32_t)x < ea ? p[(uint64_t)x * sa] : (W)0;
            W run = 0;
#pragma unroll
            for (int x = 0; x < kPairMax; ++x) {
                run |= v[x] | prev[x];
                prev[x] = run;
                if ((uint32_t)x < ea) p[(uint64_t)x * sa] = run;
            }
        }
    }
}

template <class W>
__global__ void k_cells_query(const double* __restrict__ v, uint64_t S, CellGeom geo,
                              const W* __restrict__ P, const uint32_t* __restrict__ act_in,
                              uint64_t na, const unsigned long long* n_in,
                              int32_t* __restrict__ den, uint32_t* __restrict__ act_out,
                              unsigned long long* __restrict__ n_out) {
    pdl_wait();
    if (n_in) na = *(volatile const unsigned long long*)n_in;
    const double gd = (double)geo.g;
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warp0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) & ~31ULL;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t k0 = warp0; k0 < na; k0 += stride) {
        const uint64_t k = k0 + lane;
        bool keep = false;
        uint32_t t = 0;
        if (k < na) {
            t = act_in[k];
            uint64_t r = 0;
            unsigned cj[kMaxCellDims];
            for (int j = 1; j < geo.d; ++j) {
                cj[j] = (unsigned)floor(__dmul_rn(v[j * S + t], gd));
                r += (uint64_t)cj[j] * geo.stride[j];
            }
            const unsigned c0 = (unsigned)floor(__dmul_rn(v[t], gd));
            bool hit = c0 >= 1 && ((P[r] >> (c0 - 1)) & 1);
            for (int j = 1; j < geo.d && !hit; ++j)
                if (cj[j] >= 1) hit = (P[r - geo.stride[j]] >> c0) & 1;
            if (hit) den[t] = geo.g;
            keep = !hit;
        }
        const unsigned m = __ballot_sync(0xffffffffu, keep);
        if (!m) continue;
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(n_out, (unsigned long long)__popc(m));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (keep) act_out[base + __popc(m & ((1u << lane) - 1u))] = t;
    }
}

// ---- packed-code variants: the codes floor(v*g) of every step computed
// once (one byte per attribute, codes <= 127 on this engine's path), so each
// step reads S code words instead of S x d float64 values, twice
// the steps whose codes one launch computes (descending g; <= 64 at a time)
struct StepList {
    int n;
    int g[64];
};

template <class CW>
__global__ void k_cells_codes(const double* __restrict__ v, uint64_t S, int d, StepList steps,
                              CW* __restrict__ codes) {
    pdl_wait();
    // one thread per tuple: its d values read once, the codes of the listed
    // steps written (coalesced across the warp at every step)
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < S;
         t += (uint64_t)gridDim.x * blockDim.x) {
        double x[8];
        for (int k = 0; k < d; ++k) x[k] = v[(uint64_t)k * S + t];
        for (int li = 0; li < steps.n; ++li) {
            const double gd = (double)steps.g[li];
            CW w = 0;
            for (int k = 0; k < d; ++k) w |= (CW)(unsigned)floor(__dmul_rn(x[k], gd)) << (8 * k);
            codes[(uint64_t)li * S + t] = w;
        }
    }
}

template <class W, class CW>
__global__ void k_cells_mark_c(const CW* __restrict__ code, uint64_t S, CellGeom geo,
                               W* __restrict__ rows, const unsigned long long* live) {
    pdl_wait();
    if (step_dead(live)) return;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < S;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const CW w = code[i];
        uint64_t r = 0;
        for (int j = 1; j < geo.d; ++j) r += (uint64_t)((w >> (8 * j)) & 0xFF) * geo.stride[j];
        const W bit = (W)1 << (unsigned)(w & 0xFF);
        if (!(rows[r] & bit)) atomicOr(&rows[r], bit);
    }
}

// one query per undecided candidate (act_in[0 .. *n_in), or na when n_in
// is null); ejected ones get den = g, the rest are appended to act_out
// (warp-aggregated) and counted in *n_out — the next step's candidates
template <class W, class CW>
__global__ void k_cells_query_c(const CW* __restrict__ code, CellGeom geo,
                                const W* __restrict__ P, const uint32_t* __restrict__ act_in,
                                uint64_t na, const unsigned long long* n_in,
                                int32_t* __restrict__ den, uint32_t* __restrict__ act_out,
                                unsigned long long* __restrict__ n_out) {
    pdl_wait();
    if (n_in) na = *(volatile const unsigned long long*)n_in;
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warp0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) & ~31ULL;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t k0 = warp0; k0 < na; k0 += stride) {
        const uint64_t k = k0 + lane;
        bool keep = false;
        uint32_t t = 0;
        if (k < na) {
            t = act_in[k];
            const CW w = code[t];
            uint64_t r = 0;
            for (int j = 1; j < geo.d; ++j) r += (uint64_t)((w >> (8 * j)) & 0xFF) * geo.stride[j];
            const unsigned c0 = (unsigned)(w & 0xFF);
            bool hit = c0 >= 1 && ((P[r] >> (c0 - 1)) & 1);
            for (int j = 1; j < geo.d && !hit; ++j)
                if (((w >> (8 * j)) & 0xFF) >= 1) hit = (P[r - geo.stride[j]] >> c0) & 1;
            if (hit) den[t] = geo.g;
            keep = !hit;
        }
        const unsigned m = __ballot_sync(0xffffffffu, keep);
        if (!m) continue;
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(n_out, (unsigned long long)__popc(m));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (keep) act_out[base + __popc(m & ((1u << lane) - 1u))] = t;
    }
}

__global__ void k_col_max(const double* __restrict__ v, uint64_t S, int d,
                          unsigned long long* __restrict__ out) {
    pdl_wait();
    for (int j = blockIdx.y; j < d; j += gridDim.y) {
        unsigned long long best = 0;
        for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < S;
             i += (uint64_t)gridDim.x * blockDim.x) {
            const unsigned long long b = ord_bits(v[(uint64_t)j * S + i]);
            best = b > best ? b : best;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long x = __shfl_down_sync(0xffffffffu, best, o);
            best = x > best ? x : best;
        }
        if ((threadIdx.x & 31) == 0) atomicMax(&out[j], best);
    }
}

}  // namespace

// Per-step extents of the code grid; false when the engine does not apply
// (d > 16, a code extent beyond 64 along attribute 0, or a grid that would
// not fit the memory budget).
static bool cells_geometry(const std::vector<double>& amax, int d, int g, uint64_t budget_rows,
                           CellGeom* geo, uint64_t* e0) {
    if (d < 1 || d > kMaxCellDims) return false;
    geo->d = d;
    geo->g = g;
    uint64_t rows = 1;
    for (int j = 0; j < d; ++j) {
        const double k = std::floor(amax[j] * (double)g);  // same rounding as __dmul_rn
        if (!(k >= 0) || k > 1e12) return false;
        const uint64_t ext = (uint64_t)k + 1;
        geo->ext[j] = ext;
        if (j == 0) {
            if (ext > 64) return false;
            *e0 = ext;
            continue;
        }
        geo->stride[j] = rows;
        if (rows > budget_rows / ext) return false;
        rows *= ext;
    }
    geo->rows = rows;
    return true;
}

// the prefix-OR of one step's occupancy over every attribute: fused passes
// (slab: attributes 0-2 in shared memory; pairs of the rest in registers),
// or one pass per attribute (SKYGPU_CELLS_UNFUSED=1, or extents too large)
template <class W>
void sweeps(Ctx& c, W* R, const CellGeom& geo, bool fused, const unsigned long long* live) {
    const int d = geo.d;
    auto single = [&](int j) {
        pdl_launch(k_cells_or_dim<W>, grid_for(geo.rows / geo.ext[j], kBlock), kBlock, 0, c.stream,
            R, geo.rows, geo.ext[j], geo.stride[j], live);
        note_launch(c);
    };
    const uint32_t e1 = d >= 2 ? (uint32_t)geo.ext[1] : 1, e2 = d >= 3 ? (uint32_t)geo.ext[2] : 1;
    if (!fused || d < 2 || (uint64_t)e1 * e2 * sizeof(W) > 128 * 1024) {
        pdl_launch(k_cells_or_word<W>, grid_for(geo.rows, kBlock), kBlock, 0, c.stream, R,
                   geo.rows, live);
        note_launch(c);
        for (int j = 1; j < d; ++j) single(j);
        return;
    }
    static const uint32_t slab_words = [] {
        const char* e = getenv("SKYGPU_SLAB_WORDS");
        const int v = e ? atoi(e) : 0;
        return v >= 1024 && v <= 16384 ? (uint32_t)v : kSlabWords;
    }();
    const uint32_t slab = e1 * e2;
    uint32_t spb = std::max(1u, slab_words / slab);
    if (spb >= 4) spb &= ~3u;  // batches 16-byte aligned (vector loads)
    const size_t smem = (size_t)spb * slab * sizeof(W);
    static bool attr_set = false;
    if (!attr_set) {
        SKY_CUDA(cudaFuncSetAttribute(k_cells_or_slab<unsigned>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
        SKY_CUDA(cudaFuncSetAttribute(k_cells_or_slab<unsigned long long>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
        attr_set = true;
    }
    const uint64_t nslabs = geo.rows / slab;
    pdl_launch(k_cells_or_slab<W>, grid_for((nslabs + spb - 1) / spb, 1, c.num_sms * 8), kBlock,
               smem, c.stream, R, geo.rows, e1, e2, spb, live);
    note_launch(c);
    int j = 3;
    while (j < d) {
        if (j + 1 < d && geo.ext[j] <= (uint64_t)kPairMax) {
            const uint64_t lines = geo.rows / (geo.ext[j] * geo.ext[j + 1]);
            pdl_launch(k_cells_or_pair<W>, grid_for(lines, kBlock), kBlock, 0, c.stream,
                R, geo.rows, (uint32_t)geo.ext[j], (uint32_t)geo.ext[j + 1], geo.stride[j], live);
            note_launch(c);
            j += 2;
        } else {
            single(j);
            j += 1;
        }
    }
}

// ---------------------------------------------------------------------------
// Min-grid form (the default for packed codes).  The bitset row above is,
// after its in-word prefix-OR, a run of ones from the smallest attribute-0
// code of any tuple whose other codes are <= the row's: the whole row is that
// ONE number.  So the grid keeps ONE BYTE per cell r of the other d-1
// attributes (m = the min'd attribute, the one of largest extent):
//     P[r] = min { c_m(s) : row(s) <= r componentwise }
//     M[r] = 2 P[r] + G[r],  G[r] = 0 iff P[r] is also attained by a row
//                            strictly below r (0x7F: no tuple at all)
// A skyline tuple t sits in its own cell r, so P[r] <= c_m(t), and t is
// dominated iff P[r] < c_m(t) (a smaller code in a row <= r) or P[r] =
// c_m(t) attained strictly below r:  M[r] <= 2 c_m(t).  ONE byte read per
// query (the bitset form reads the row and one row below per attribute).
// Sweeping keeps the encoding: along a dim, a predecessor contributes its
// value with the low bit cleared (min(v, acc & ~1) — "attained below"), the
// cell itself its own value; the mark writes 2 c_m + 1.  c_m <= 62 (extent
// <= 63) keeps every value at most 125 < 0x7F.  Byte grids are 4x smaller
// than u32 rows; every step below g ~ 22 of C5 stays resident in the 126 MB
// L2 across its passes.  Grid dim 0 (the fastest) is padded to a multiple of
// 4 bytes so that every other dim's stride is a whole number of u32 words.
namespace {

struct MinGeom {
    int nd;                        // grid dims (d - 1)
    int m;                         // the min'd attribute
    int g;
    uint32_t attr[kMaxCellDims];   // attribute of grid dim k
    uint32_t ext[kMaxCellDims];    // its code extent (grid dim 0: padded to 4)
    uint64_t stride[kMaxCellDims]; // its byte stride (stride[0] = 1)
    uint64_t bytes;                // grid bytes (a multiple of 16)
};

// Cells hold 7-bit values (<= 125; 0x7F = empty), so a bytewise
// minimum is 3 instructions instead of __vminu4's emulated 7: t = a + 0x80 -
// b per byte cannot carry or borrow across bytes, its top bit is a >= b,
// PRMT replicates that bit over the byte, a LOP3 selects.
constexpr uint32_t kEmpty = 0x7Fu;
constexpr uint32_t kEmpty4 = 0x7F7F7F7Fu;
constexpr uint32_t kPred4 = 0xFEFEFEFEu;  // a predecessor's value: its "own cell only" bit cleared

__device__ __forceinline__ uint32_t min7(uint32_t a, uint32_t b) {
    const uint32_t t = a + 0x80808080u - b;
    uint32_t m;
    asm("prmt.b32 %0, %1, 0, 0xBA98;" : "=r"(m) : "r"(t));  // 0xFF where a >= b
    return (b & m) | (a & ~m);
}

template <class CW>
__device__ __forceinline__ uint64_t mg_row(CW w, const MinGeom& geo) {
    uint64_t r = 0;
    for (int k = 0; k < geo.nd; ++k)
        r += (uint64_t)((uint32_t)(w >> (8 * geo.attr[k])) & 0xFFu) * geo.stride[k];
    return r;
}

// (`clear`: the step's undecided counter, zeroed here — before the step's
// query appends to it — instead of by a one-thread launch of its own)
__global__ void k_mg_fill(uint4* __restrict__ p, uint64_t n16, const unsigned long long* live,
                          unsigned long long* clear) {
    pdl_wait();
    if (clear && blockIdx.x == 0 && threadIdx.x == 0) *clear = 0;
    if (step_dead(live)) return;
    const uint4 f = make_uint4(kEmpty4, kEmpty4, kEmpty4, kEmpty4);
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n16;
         i += (uint64_t)gridDim.x * blockDim.x)
        p[i] = f;
}

// every skyline tuple lowers its cell's byte to 2 c_m + 1 ("attained in
// this cell"): one CAS, optimistic about a fresh (empty) word, retried with
// the bytewise minimum when the word already holds marks
template <class CW, bool LOADFIRST>
__global__ void __launch_bounds__(kBlock)
k_mg_mark(const CW* __restrict__ code, uint64_t S, MinGeom geo, uint8_t* __restrict__ M,
          const unsigned long long* live) {
    pdl_wait();
    if (step_dead(live)) return;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < S;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const CW w = code[i];
        const uint64_t r = mg_row(w, geo);
        const uint32_t c0 = (uint32_t)(w >> (8 * geo.m)) & 0xFFu;
        const uint32_t sh = 8u * (uint32_t)(r & 3u);
        const uint32_t mine = (kEmpty4 & ~(0xFFu << sh)) | ((2u * c0 + 1u) << sh);
        uint32_t* word = reinterpret_cast<uint32_t*>(M) + (r >> 2);
        uint32_t old = kEmpty4;
        if (LOADFIRST) {
            // most tuples do not lower their cell (a cell's minimum changes
            // ~ln k times over its k tuples): one L2 load settles them
            old = __ldcg(word);
            if (old == kEmpty4) old = atomicCAS(word, kEmpty4, mine);
        } else {
            old = atomicCAS(word, kEmpty4, mine);
        }
        while (old != kEmpty4) {
            const uint32_t nw = min7(old, mine);
            if (nw == old) break;
            const uint32_t prev = atomicCAS(word, old, nw);
            if (prev == old) break;
            old = prev;
        }
    }
}

// small grids (<= kPrivCells cells: the low steps, where CAS contention on
// few words would serialise the mark): each block takes a contiguous share
// of the tuples into a private u32-per-cell copy in shared memory (native
// atomicMin), then stores it packed to its staging slot; k_mg_mark_reduce
// takes the bytewise minimum over the slots (and so also fills the grid)
constexpr uint32_t kPrivCells = 40960;

template <class CW>
__global__ void __launch_bounds__(kBlock)
k_mg_mark_priv(const CW* __restrict__ code, uint64_t S, MinGeom geo, uint32_t* __restrict__ stage,
               const unsigned long long* live, unsigned long long* clear) {
    pdl_wait();
    if (clear && blockIdx.x == 0 && threadIdx.x == 0) *clear = 0;
    if (step_dead(live)) return;
    extern __shared__ uint32_t cm[];
    const uint32_t ncells = (uint32_t)geo.bytes;
    for (uint32_t i = threadIdx.x; i < ncells; i += blockDim.x) cm[i] = kEmpty;
    __syncthreads();
    const uint64_t per = (S + gridDim.x - 1) / gridDim.x;
    const uint64_t lo = blockIdx.x * per, hi = min(S, lo + per);
    for (uint64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        const CW w = code[i];
        const uint32_t r = (uint32_t)mg_row(w, geo);
        const uint32_t c0 = (uint32_t)(w >> (8 * geo.m)) & 0xFFu;
        const uint32_t v = 2u * c0 + 1u;
        if (cm[r] > v) atomicMin(&cm[r], v);
    }
    __syncthreads();
    uint32_t* out = stage + (uint64_t)blockIdx.x * (ncells / 4);
    for (uint32_t q = threadIdx.x; q < ncells / 4; q += blockDim.x)
        out[q] = cm[4 * q] | (cm[4 * q + 1] << 8) | (cm[4 * q + 2] << 16) | (cm[4 * q + 3] << 24);
}

__global__ void k_mg_mark_reduce(const uint32_t* __restrict__ stage, uint32_t nslots,
                                 uint32_t nwords, uint32_t* __restrict__ M,
                                 const unsigned long long* live) {
    pdl_wait();
    if (step_dead(live)) return;
    for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < nwords; q += gridDim.x * blockDim.x) {
        uint32_t acc = kEmpty4;
        for (uint32_t b = 0; b < nslots; ++b) acc = min7(acc, stage[(uint64_t)b * nwords + q]);
        M[q] = acc;
    }
}

// mid-size grids: marks into a u32-per-cell copy with the native one-way
// atomicMin (RED.MIN: no value returns, no CAS retry loop under contention),
// then packed to the byte grid.  The copy is 4 x the grid: only worth it while
// it stays in L2.
__global__ void k_mg_fill32(uint4* __restrict__ p, uint64_t n16, const unsigned long long* live,
                            unsigned long long* clear) {
    pdl_wait();
    if (clear && blockIdx.x == 0 && threadIdx.x == 0) *clear = 0;
    if (step_dead(live)) return;
    const uint4 f = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n16;
         i += (uint64_t)gridDim.x * blockDim.x)
        p[i] = f;
}

template <class CW>
__global__ void __launch_bounds__(kBlock)
k_mg_mark32(const CW* __restrict__ code, uint64_t S, MinGeom geo, uint32_t* __restrict__ G,
            const unsigned long long* live) {
    pdl_wait();
    if (step_dead(live)) return;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < S;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const CW w = code[i];
        const uint64_t r = mg_row(w, geo);
        const uint32_t c0 = (uint32_t)(w >> (8 * geo.m)) & 0xFFu;
        atomicMin(&G[r], 2u * c0 + 1u);
    }
}

__global__ void k_mg_pack(const uint4* __restrict__ G, uint64_t nwords, uint32_t* __restrict__ M,
                          const unsigned long long* live) {
    pdl_wait();
    if (step_dead(live)) return;
    for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < nwords;
         q += (uint64_t)gridDim.x * blockDim.x) {
        const uint4 g = G[q];
        M[q] = g.x | (g.y << 8) | (g.z << 16) | (g.w << 24);
    }
}

// prefix minimum along the 4 bytes of a word (byte k = lower address first),
// then against the previous word's last byte
__device__ __forceinline__ uint32_t bytes_prefix_min(uint32_t x, uint32_t carry) {
    x = min7(x, ((x << 8) | kEmpty) & kPred4);
    x = min7(x, ((x << 16) | (kEmpty4 >> 16)) & kPred4);
    return min7(x, (carry & 0xFEu) * 0x01010101u);
}

// grid dims 0, 1, 2 (ND of them) of ns whole slabs staged in shared memory
template <int ND>
__device__ __forceinline__ void slab_prefix(uint32_t* sw, uint32_t ns, uint32_t w0, uint32_t e1,
                                            uint32_t e2) {
    const uint32_t slab = w0 * e1 * e2;
    const uint32_t words = ns * slab;
    for (uint32_t l = threadIdx.x; l < words / w0; l += blockDim.x) {  // dim 0: bytes of a line
        uint32_t* p = sw + (uint64_t)l * w0;
        uint32_t carry = kEmpty;
        for (uint32_t a = 0; a < w0; ++a) {
            const uint32_t x = bytes_prefix_min(p[a], carry);
            p[a] = x;
            carry = x >> 24;
        }
    }
    __syncthreads();
    if (ND >= 2) {  // dim 1: u32 columns, stride w0
        for (uint32_t l = threadIdx.x; l < ns * e2 * w0; l += blockDim.x) {
            uint32_t* p = sw + (uint64_t)(l / w0) * w0 * e1 + (l % w0);
            uint32_t acc = kEmpty4;
            for (uint32_t a = 0; a < e1; ++a) {
                acc = min7(p[a * w0], acc & kPred4);
                p[a * w0] = acc;
            }
        }
        __syncthreads();
    }
    if (ND >= 3) {  // dim 2: u32 columns, stride w0 * e1
        const uint32_t plane = w0 * e1;
        for (uint32_t l = threadIdx.x; l < ns * plane; l += blockDim.x) {
            uint32_t* p = sw + (uint64_t)(l / plane) * slab + (l % plane);
            uint32_t acc = kEmpty4;
            for (uint32_t b = 0; b < e2; ++b) {
                acc = min7(p[b * plane], acc & kPred4);
                p[b * plane] = acc;
            }
        }
        __syncthreads();
    }
}

template <int ND>
__global__ void __launch_bounds__(kBlock)
k_mg_slab(uint32_t* __restrict__ M, uint64_t nwords, uint32_t w0, uint32_t e1, uint32_t e2,
          uint32_t spb, const unsigned long long* live) {
    pdl_wait();
    if (step_dead(live)) return;
    extern __shared__ __align__(16) uint32_t sw[];
    const uint32_t slab = w0 * e1 * e2;  // words per slab
    const uint64_t nslabs = nwords / slab;
    for (uint64_t s0 = (uint64_t)blockIdx.x * spb; s0 < nslabs; s0 += (uint64_t)gridDim.x * spb) {
        const uint32_t ns = (uint32_t)min((uint64_t)spb, nslabs - s0);
        const uint32_t words = ns * slab;
        const uint32_t* g = M + s0 * slab;
        const bool vec = (words & 3u) == 0 && ((s0 * slab) & 3u) == 0;
        if (vec) {
            for (uint32_t i = threadIdx.x; i < words / 4; i += blockDim.x)
                reinterpret_cast<uint4*>(sw)[i] = reinterpret_cast<const uint4*>(g)[i];
        } else {
            for (uint32_t i = threadIdx.x; i < words; i += blockDim.x) sw[i] = g[i];
        }
        __syncthreads();
        slab_prefix<ND>(sw, ns, w0, e1, e2);
        uint32_t* o = M + s0 * slab;
        if (vec) {
            for (uint32_t i = threadIdx.x; i < words / 4; i += blockDim.x)
                reinterpret_cast<uint4*>(o)[i] = reinterpret_cast<const uint4*>(sw)[i];
        } else {
            for (uint32_t i = threadIdx.x; i < words; i += blockDim.x) o[i] = sw[i];
        }
        __syncthreads();
    }
}

// grid dims 0..3 in ONE pass: a block owns a column of e3 consecutive slabs
// (dims 0..2; fixed dims 4..), prefixes each in shared memory and carries a
// running elementwise minimum from slab to slab — the prefix along dim 3.
// The next slab's words are loaded into registers (kPer per thread) while
// the current one is swept.
constexpr int kColPer = 20;  // slab words per thread (slab <= 5120 words)

template <int PER>  // slab words per thread (PER * kBlock >= slab words)
__global__ void __launch_bounds__(kBlock)
k_mg_slabcol(uint32_t* __restrict__ M, uint32_t ncols, uint32_t w0, uint32_t e1, uint32_t e2,
             uint32_t e3, const unsigned long long* live) {
    pdl_wait();
    if (step_dead(live)) return;
    extern __shared__ __align__(16) uint32_t sw[];
    const uint32_t slab = w0 * e1 * e2;
    uint32_t* run = sw + slab;
    for (uint32_t col = blockIdx.x; col < ncols; col += gridDim.x) {
        uint32_t* base = M + (uint64_t)col * e3 * slab;
        uint32_t pre[PER];
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const uint32_t i = threadIdx.x + k * kBlock;
            pre[k] = i < slab ? base[i] : kEmpty4;
        }
        for (uint32_t c3 = 0; c3 < e3; ++c3) {
#pragma unroll
            for (int k = 0; k < PER; ++k) {
                const uint32_t i = threadIdx.x + k * kBlock;
                if (i < slab) sw[i] = pre[k];
            }
            __syncthreads();
            if (c3 + 1 < e3) {
                const uint32_t* nx = base + (uint64_t)(c3 + 1) * slab;
#pragma unroll
                for (int k = 0; k < PER; ++k) {
                    const uint32_t i = threadIdx.x + k * kBlock;
                    pre[k] = i < slab ? nx[i] : kEmpty4;
                }
            }
            slab_prefix<3>(sw, 1, w0, e1, e2);
            uint32_t* o = base + (uint64_t)c3 * slab;
            for (uint32_t i = threadIdx.x; i < slab; i += blockDim.x) {
                uint32_t x = sw[i];
                if (c3) x = min7(x, run[i] & kPred4);
                run[i] = x;
                o[i] = x;
            }
            __syncthreads();
        }
    }
}

// two grid dims a, b = a + 1 at once (word stride sa of dim a), one thread
// per u32 column of the (ea x eb) plane: P = min(v, P[x-1][y], P[x][y-1])
template <int EA>
__global__ void __launch_bounds__(kBlock)
k_mg_pair(uint32_t* __restrict__ M, uint64_t nwords, uint32_t ea, uint32_t eb, uint64_t sa,
          const unsigned long long* live) {
    pdl_wait();
    if (step_dead(live)) return;
    const uint64_t plane = (uint64_t)ea * eb;
    const uint64_t lines = nwords / plane;
    for (uint64_t l = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; l < lines;
         l += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t lo = l % sa, hi = l / sa;
        uint32_t* base = M + hi * sa * plane + lo;
        uint32_t prev[EA];
#pragma unroll
        for (int x = 0; x < EA; ++x) prev[x] = kEmpty4;
        for (uint32_t y = 0; y < eb; ++y) {
            uint32_t* p = base + (uint64_t)y * ea * sa;
            uint32_t v[EA];
#pragma unroll
            for (int x = 0; x < EA; ++x) v[x] = (uint32_t)x < ea ? p[(uint64_t)x * sa] : kEmpty4;
            uint32_t run = kEmpty4;
#pragma unroll
            for (int x = 0; x < EA; ++x) {
                run = min7(v[x], min7(run, prev[x]) & kPred4);
                prev[x] = run;
                if ((uint32_t)x < ea) p[(uint64_t)x * sa] = run;
            }
        }
    }
}

// the same two dims staged through shared memory: a block takes a tile of
// 32 consecutive u32 columns (128-byte lines) over the whole (ea x eb) plane,
// all of it requested at once with cp.async (every load in flight), then
// sweeps dim a and dim b in shared memory with every thread busy, and
// writes the tile back — the register form above holds only ~16 warps per
// SM (125 registers) and its loads wait row by row
constexpr int kPT = 32;

__device__ __forceinline__ void cp_async4(uint32_t* dst, const uint32_t* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
                 "l"(src)
                 : "memory");
}

__global__ void __launch_bounds__(kBlock)
k_mg_pair_smem(uint32_t* __restrict__ M, uint64_t nwords, uint32_t ea, uint32_t eb, uint64_t sa,
               const unsigned long long* live) {
    pdl_wait();
    if (step_dead(live)) return;
    extern __shared__ __align__(16) uint32_t tile[];  // [ea * eb][kPT]
    const uint32_t plane = ea * eb;
    const uint64_t nhi = nwords / (sa * plane);
    const uint64_t tph = (sa + kPT - 1) / kPT;  // tiles per hi index
    for (uint64_t t = blockIdx.x; t < nhi * tph; t += gridDim.x) {
        const uint64_t hi = t / tph;
        const uint32_t lo0 = (uint32_t)(t - hi * tph) * kPT;
        const uint32_t ncol = (uint32_t)min((uint64_t)kPT, sa - lo0);
        uint32_t* base = M + hi * sa * plane + lo0;
        for (uint32_t i = threadIdx.x; i < plane * kPT; i += blockDim.x) {
            const uint32_t e = i / kPT, col = i % kPT;
            if (col < ncol) cp_async4(&tile[i], base + (uint64_t)e * sa + col);
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncthreads();
        for (uint32_t l = threadIdx.x; l < eb * kPT; l += blockDim.x) {  // dim a
            uint32_t* q = tile + (l / kPT) * ea * kPT + (l % kPT);
            uint32_t acc = kEmpty4;
            for (uint32_t x = 0; x < ea; ++x) {
                acc = min7(q[x * kPT], acc & kPred4);
                q[x * kPT] = acc;
            }
        }
        __syncthreads();
        for (uint32_t l = threadIdx.x; l < ea * kPT; l += blockDim.x) {  // dim b
            uint32_t* q = tile + l;
            uint32_t acc = kEmpty4;
            for (uint32_t y = 0; y < eb; ++y) {
                acc = min7(q[y * ea * kPT], acc & kPred4);
                q[y * ea * kPT] = acc;
            }
        }
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < plane * kPT; i += blockDim.x) {
            const uint32_t e = i / kPT, col = i % kPT;
            if (col < ncol) base[(uint64_t)e * sa + col] = tile[i];
        }
        __syncthreads();
    }
}

// one grid dim (word stride s, extent e <= E): one thread per u32 column,
// the column's words loaded together (independent loads in flight)
template <int E>
__global__ void __launch_bounds__(kBlock)
k_mg_dim(uint32_t* __restrict__ M, uint64_t nwords, uint32_t e, uint64_t s,
         const unsigned long long* live) {
    pdl_wait();
    if (step_dead(live)) return;
    const uint64_t lines = nwords / e;
    for (uint64_t l = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; l < lines;
         l += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t* p = M + (l / s) * s * e + (l % s);
        if (E > 0) {
            uint32_t v[E > 0 ? E : 1];
#pragma unroll
            for (int k = 0; k < E; ++k) v[k] = (uint32_t)k < e ? p[(uint64_t)k * s] : kEmpty4;
            uint32_t acc = kEmpty4;
#pragma unroll
            for (int k = 0; k < E; ++k) {
                acc = min7(v[k], acc & kPred4);
                if ((uint32_t)k < e) p[(uint64_t)k * s] = acc;
            }
        } else {
            uint32_t acc = kEmpty4;
            for (uint64_t k = 0; k < e; ++k) {
                acc = min7(p[k * s], acc & kPred4);
                p[k * s] = acc;
            }
        }
    }
}

template <class CW>
__global__ void k_mg_query(const CW* __restrict__ code, MinGeom geo, const uint8_t* __restrict__ M,
                           const uint32_t* __restrict__ act_in, uint64_t na,
                           const unsigned long long* n_in, int32_t* __restrict__ den,
                           const uint32_t* __restrict__ perm,
                           uint32_t* __restrict__ act_out, unsigned long long* __restrict__ n_out) {
    pdl_wait();
    if (n_in) na = *(volatile const unsigned long long*)n_in;
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warp0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) & ~31ULL;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t k0 = warp0; k0 < na; k0 += stride) {
        const uint64_t k = k0 + lane;
        bool keep = false;
        uint32_t t = 0;
        if (k < na) {
            t = act_in ? act_in[k] : (uint32_t)k;
            const CW w = code[t];
            const uint64_t r = mg_row(w, geo);
            const uint32_t c0 = (uint32_t)(w >> (8 * geo.m)) & 0xFFu;
            // one byte: P = M[r] >> 1 is the smallest c_m over rows <= r, and
            // its low bit is 0 iff that minimum is also attained strictly
            // below r; t (which is in cell r itself) is dominated iff
            // P < c_m(t) or (P == c_m(t) and attained below): M[r] <= 2 c_m(t)
            const bool hit = (uint32_t)M[r] <= 2u * c0;
            if (hit) den[perm ? perm[t] : t] = geo.g;
            keep = !hit;
        }
        const unsigned msk = __ballot_sync(0xffffffffu, keep);
        if (!msk) continue;
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(n_out, (unsigned long long)__popc(msk));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (keep) act_out[base + __popc(msk & ((1u << lane) - 1u))] = t;
    }
}

// locality order of the skyline for the min-grid steps: the row of every
// tuple in the top step's grid (its codes there), sorted once per call — at
// every lower step consecutive tuples then mark and query nearby cells
__global__ void k_mg_sortkey(const double* __restrict__ v, uint64_t S, int d, MinGeom geo,
                             unsigned long long* __restrict__ key, uint32_t* __restrict__ idx) {
    pdl_wait();
    const double gd = (double)geo.g;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < S;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t r = 0;
        for (int k = 0; k < geo.nd; ++k)
            r += (uint64_t)floor(__dmul_rn(v[(uint64_t)geo.attr[k] * S + i], gd)) * geo.stride[k];
        key[i] = r;
        idx[i] = (uint32_t)i;
    }
}

// the SoA values in that order
__global__ void k_mg_permute(const double* __restrict__ v, uint64_t S, int d,
                             const uint32_t* __restrict__ perm, double* __restrict__ out) {
    pdl_wait();
    for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < S;
         q += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t t = perm[q];
        for (int j = 0; j < d; ++j) out[(uint64_t)j * S + q] = v[(uint64_t)j * S + t];
    }
}

}  // namespace

// Min-grid geometry of step g; false when it does not apply (a code above
// 127 or a grid beyond the budget).  m = the attribute of largest extent.
static bool min_geometry(const std::vector<double>& amax, int d, int g, uint64_t budget,
                         MinGeom* geo) {
    if (d < 2 || d > 8) return false;
    uint32_t e[8];
    int m = 0;
    for (int j = 0; j < d; ++j) {
        const double k = std::floor(amax[j] * (double)g);  // same rounding as __dmul_rn
        if (!(k >= 0) || k > 127) return false;
        e[j] = (uint32_t)k + 1;
        if (e[j] > e[m]) m = j;
    }
    if (e[m] > 63) return false;  // 2 c_m + 1 must stay below the empty value 0x7F
    geo->nd = d - 1;
    geo->m = m;
    geo->g = g;
    uint64_t bytes = 1;
    int k = 0;
    for (int j = 0; j < d; ++j) {
        if (j == m) continue;
        const uint32_t ext = k == 0 ? (e[j] + 3u) & ~3u : e[j];
        geo->attr[k] = (uint32_t)j;
        geo->ext[k] = ext;
        geo->stride[k] = bytes;
        if (bytes > budget / ext) return false;
        bytes *= ext;
        ++k;
    }
    geo->bytes = (bytes + 15) & ~15ULL;
    return true;
}

// the prefix minimum over every grid dim: dims 0..3 in one slab-column pass
// (k_mg_slabcol; dims 0..2 in a slab pass when there is no dim 3 or the slab
// is too large), the rest two at a time in registers (k_mg_pair) or one at a
// time (k_mg_dim) — 2 passes for d = 7
static int min_sweeps(Ctx& c, uint8_t* M, const MinGeom& geo, const unsigned long long* live) {
    constexpr size_t kSlabMax = 48 * 1024;
    static const bool nocol = [] {
        const char* e = getenv("SKYGPU_MG_NOCOL");
        return e && e[0] == '1';
    }();
    // SKYGPU_MG_PAIRSMEM=1: the shared-memory staged two-dim sweep (measured
    // slower on C5: 6.47 vs 6.20 ms of gres kernels; kept for A/B)
    static const bool nosmem = [] {
        const char* e = getenv("SKYGPU_MG_PAIRSMEM");
        return !(e && e[0] == '1');
    }();
    constexpr size_t kPairSmemMax = 112 * 1024;
    uint32_t* W = reinterpret_cast<uint32_t*>(M);
    // (whole rows only: the 16-byte padding of the fill stays empty)
    const uint64_t real_words = geo.stride[geo.nd - 1] * geo.ext[geo.nd - 1] / 4;
    int nl = 0;
    const uint32_t w0 = geo.ext[0] / 4;
    int sd = std::min(geo.nd, 3);
    auto slab_bytes = [&](int k) {
        uint64_t b = geo.ext[0];
        for (int j = 1; j < k; ++j) b *= geo.ext[j];
        return b;
    };
    while (sd > 1 && slab_bytes(sd) > kSlabMax) --sd;
    const uint32_t e1 = sd >= 2 ? geo.ext[1] : 1, e2 = sd >= 3 ? geo.ext[2] : 1;
    const uint64_t slab = slab_bytes(sd);
    static bool attr_set = false;
    if (!attr_set) {
        SKY_CUDA(cudaFuncSetAttribute(k_mg_slab<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSlabMax));
        SKY_CUDA(cudaFuncSetAttribute(k_mg_slab<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSlabMax));
        SKY_CUDA(cudaFuncSetAttribute(k_mg_slab<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSlabMax));
        SKY_CUDA(cudaFuncSetAttribute(k_mg_slabcol<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSlabMax));
        SKY_CUDA(cudaFuncSetAttribute(k_mg_slabcol<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSlabMax));
        SKY_CUDA(cudaFuncSetAttribute(k_mg_slabcol<12>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSlabMax));
        SKY_CUDA(cudaFuncSetAttribute(k_mg_slabcol<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSlabMax));
        SKY_CUDA(cudaFuncSetAttribute(k_mg_slabcol<kColPer>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSlabMax));
        SKY_CUDA(cudaFuncSetAttribute(k_mg_pair_smem, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)kPairSmemMax));
        attr_set = true;
    }
    const uint64_t nslabs = real_words / (slab / 4);
    int j = sd;
    if (!nocol && sd == 3 && geo.nd >= 4 && slab / 4 <= (uint64_t)kColPer * kBlock) {
        const uint32_t e3 = geo.ext[3];
        const uint64_t ncols = nslabs / e3;
        const uint64_t per = (slab / 4 + kBlock - 1) / kBlock;  // words per thread
        const unsigned gc = grid_for(ncols, 1, c.num_sms * 8);
        if (per <= 4)
            pdl_launch(k_mg_slabcol<4>, gc, kBlock, (size_t)2 * slab, c.stream, W, (uint32_t)ncols,
                       w0, e1, e2, e3, live);
        else if (per <= 8)
            pdl_launch(k_mg_slabcol<8>, gc, kBlock, (size_t)2 * slab, c.stream, W, (uint32_t)ncols,
                       w0, e1, e2, e3, live);
        else if (per <= 12)
            pdl_launch(k_mg_slabcol<12>, gc, kBlock, (size_t)2 * slab, c.stream, W,
                       (uint32_t)ncols, w0, e1, e2, e3, live);
        else if (per <= 16)
            pdl_launch(k_mg_slabcol<16>, gc, kBlock, (size_t)2 * slab, c.stream, W,
                       (uint32_t)ncols, w0, e1, e2, e3, live);
        else
            pdl_launch(k_mg_slabcol<kColPer>, gc, kBlock, (size_t)2 * slab, c.stream, W,
                       (uint32_t)ncols, w0, e1, e2, e3, live);
        j = 4;
    } else {
        const uint32_t spb = (uint32_t)std::max<uint64_t>(1, (kSlabMax / 2) / slab);
        const size_t smem = (size_t)spb * slab;
        const unsigned gsl = grid_for((nslabs + spb - 1) / spb, 1, c.num_sms * 8);
        if (sd == 1)
            pdl_launch(k_mg_slab<1>, gsl, kBlock, smem, c.stream, W, real_words, w0, e1, e2, spb, live);
        else if (sd == 2)
            pdl_launch(k_mg_slab<2>, gsl, kBlock, smem, c.stream, W, real_words, w0, e1, e2, spb, live);
        else
            pdl_launch(k_mg_slab<3>, gsl, kBlock, smem, c.stream, W, real_words, w0, e1, e2, spb, live);
    }
    ++nl;
    while (j < geo.nd) {
        const uint64_t sa = geo.stride[j] / 4;
        const uint32_t ea = geo.ext[j];
        if (j + 1 < geo.nd && !nosmem && (size_t)ea * geo.ext[j + 1] * kPT * 4 <= kPairSmemMax &&
            sa >= (uint64_t)kPT) {
            const uint32_t eb = geo.ext[j + 1];
            const size_t smem = (size_t)ea * eb * kPT * 4;
            const uint64_t tiles = real_words / (sa * ea * eb) * ((sa + kPT - 1) / kPT);
            pdl_launch(k_mg_pair_smem, grid_for(tiles, 1, c.num_sms * 2), kBlock, smem, c.stream, W,
                       real_words, ea, eb, sa, live);
            j += 2;
        } else if (j + 1 < geo.nd && ea <= 32) {
            const uint64_t lines = real_words / ((uint64_t)ea * geo.ext[j + 1]);
            const unsigned gp = grid_for(lines, kBlock);
            const uint32_t eb = geo.ext[j + 1];
            if (ea <= 8)
                pdl_launch(k_mg_pair<8>, gp, kBlock, 0, c.stream, W, real_words, ea, eb, sa, live);
            else if (ea <= 12)
                pdl_launch(k_mg_pair<12>, gp, kBlock, 0, c.stream, W, real_words, ea, eb, sa, live);
            else if (ea <= 16)
                pdl_launch(k_mg_pair<16>, gp, kBlock, 0, c.stream, W, real_words, ea, eb, sa, live);
            else if (ea <= 20)
                pdl_launch(k_mg_pair<20>, gp, kBlock, 0, c.stream, W, real_words, ea, eb, sa, live);
            else if (ea <= 26)  // (cap 25: extents up to 26)
                pdl_launch(k_mg_pair<26>, gp, kBlock, 0, c.stream, W, real_words, ea, eb, sa, live);
            else
                pdl_launch(k_mg_pair<32>, gp, kBlock, 0, c.stream, W, real_words, ea, eb, sa, live);
            j += 2;
        } else {
            const unsigned gd = grid_for(real_words / ea, kBlock);
            if (ea <= 8)
                pdl_launch(k_mg_dim<8>, gd, kBlock, 0, c.stream, W, real_words, ea, sa, live);
            else if (ea <= 32)
                pdl_launch(k_mg_dim<32>, gd, kBlock, 0, c.stream, W, real_words, ea, sa, live);
            else
                pdl_launch(k_mg_dim<0>, gd, kBlock, 0, c.stream, W, real_words, ea, sa, live);
            j += 1;
        }
        ++nl;
    }
    return nl;
}

namespace {

constexpr int kSmemBlock = 512;
constexpr size_t kSmemGridMax = 200 * 1024;  // bytes of row words per step

// Every step in ONE launch, each step's grid in shared memory (small grids:
// d <= 4 and code extent e <= 32, so the grid is e^(d-1) u32 row words).
// blockIdx.y = step (g = g_max - y); every block of a step builds that
// step's prefix-OR grid from all S tuples (cheap: S shared-memory atomics),
// then answers its slice of the candidates.  den = the largest g at which t
// is dominated = the first ejection of the descending scan (atomicMax).
//
// spec != nullptr (speculative launch, gres_cells_smem_spec): g_max and the
// value maximum come from the device (the gap witness, slots[S_FLAG] bit 0 and
// slots[S_MAXV]); every block checks the launch applies — g_max = cap and the
// top code extent within ealloc — or block (0,0) raises slots[S_SPEC].
__global__ void __launch_bounds__(kSmemBlock)
    k_cells_smem(const double* __restrict__ v, uint32_t S, int d, int g_max, double maxv,
                 const uint32_t* __restrict__ act, uint32_t na, uint32_t per_block,
                 int32_t* __restrict__ den, unsigned long long* __restrict__ spec,
                 uint32_t ealloc) {
    pdl_wait();
    extern __shared__ uint32_t P[];
    if (spec) {
        maxv = __longlong_as_double((long long)spec[S_MAXV]);
        const bool ok = (spec[S_FLAG] & 1ULL) &&
                        floor(__dmul_rn(maxv, (double)g_max)) + 1.0 <= (double)ealloc;
        if (!ok) {
            if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) spec[S_SPEC] = 1;
            return;
        }
    }
    const int g = g_max - (int)blockIdx.y;
    const double gd = (double)g;
    const uint32_t e = (uint32_t)floor(__dmul_rn(maxv, gd)) + 1;  // codes 0 .. e-1
    uint32_t stride[4] = {0, 1, e, e * e};
    uint32_t rows = 1;
    for (int j = 1; j < d; ++j) rows *= e;
    for (uint32_t w = threadIdx.x; w < rows; w += blockDim.x) P[w] = 0;
    __syncthreads();
    auto code = [&](uint32_t i, int j) { return (uint32_t)floor(__dmul_rn(v[(uint64_t)j * S + i], gd)); };
    for (uint32_t i = threadIdx.x; i < S; i += blockDim.x) {
        uint32_t r = 0;
#pragma unroll
        for (int j = 1; j < 4; ++j)
            if (j < d) r += code(i, j) * stride[j];
        atomicOr(&P[r], 1u << code(i, 0));
    }
    __syncthreads();
    for (uint32_t w = threadIdx.x; w < rows; w += blockDim.x) {  // attribute 0, in-word
        uint32_t x = P[w];
        x |= x << 1;
        x |= x << 2;
        x |= x << 4;
        x |= x << 8;
        x |= x << 16;
        P[w] = x;
    }
    __syncthreads();
#pragma unroll
    for (int j = 1; j < 4; ++j) {  // attributes 1 .. d-1: one thread per line
        if (j < d) {
            const uint32_t sj = stride[j], lines = rows / e;
            for (uint32_t l = threadIdx.x; l < lines; l += blockDim.x) {
                uint32_t at = (l / sj) * sj * e + l % sj;
                uint32_t acc = P[at];
                for (uint32_t k = 1; k < e; ++k) {
                    at += sj;
                    acc |= P[at];
                    P[at] = acc;
                }
            }
        }
        __syncthreads();
    }
    const uint32_t q0 = blockIdx.x * per_block;
    const uint32_t q1 = min(na, q0 + per_block);
    for (uint32_t q = q0 + threadIdx.x; q < q1; q += blockDim.x) {
        const uint32_t t = act[q];
        uint32_t c[4] = {0, 0, 0, 0}, r = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (j < d) c[j] = code(t, j);
#pragma unroll
        for (int j = 1; j < 4; ++j) r += c[j] * stride[j];
        // dominated iff some occupied cell <= c, != c: OR_j P[c - e_j]
        bool dom = c[0] >= 1 && ((P[r] >> (c[0] - 1)) & 1u);
#pragma unroll
        for (int j = 1; j < 4; ++j)
            if (j < d && c[j] >= 1) dom |= (P[r - stride[j]] >> c[0]) & 1u;
        if (dom) atomicMax(&den[t], g);
    }
}

}  // namespace

// All steps in one launch with the grids in shared memory; false (nothing
// done) unless d <= 4 and every step's grid fits (kSmemGridMax).
bool gres_cells_smem_device(Ctx& c, const double* d_skyv, uint64_t S, int d, int g_max,
                            double maxv, const uint32_t* act, uint64_t na, int32_t* d_den) {
    if (g_max < 2 || S == 0 || na == 0 || d < 1 || d > 4 || !(maxv >= 0.0)) return false;
    const char* off = getenv("SKYGPU_CELLS_SMEM");  // "0": the per-step HBM variant (tests)
    if (off && off[0] == '0') return false;
    const double emax = std::floor(maxv * (double)g_max) + 1.0;
    if (emax > 32.0) return false;
    const uint64_t e = (uint64_t)emax;
    uint64_t rows = 1;
    for (int j = 1; j < d; ++j) rows *= e;
    const size_t smem = rows * sizeof(uint32_t);
    if (smem > kSmemGridMax) return false;
    static bool attr_set = false;
    if (!attr_set) {
        SKY_CUDA(cudaFuncSetAttribute(k_cells_smem, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)kSmemGridMax));
        attr_set = true;
    }
    const uint32_t G = (uint32_t)(g_max - 1);
    // ~2 blocks per SM over all steps, at least 64 candidates per block
    uint64_t per_step = ((uint64_t)c.num_sms * 2 + G - 1) / G;
    per_step = std::max<uint64_t>(1, std::min<uint64_t>(per_step, (na + 63) / 64));
    const uint32_t per_block = (uint32_t)((na + per_step - 1) / per_step);
    pdl_launch(k_cells_smem, dim3((unsigned)per_step, G), kSmemBlock, smem, c.stream,
        d_skyv, (uint32_t)S, d, g_max, maxv, act, (uint32_t)na, per_block, d_den, nullptr, 0);
    SKY_LAUNCH_CHECK();
    note_launch(c);
    return true;
}

bool gres_cells_smem_spec(Ctx& c, const double* d_skyv, uint64_t S, int d, int cap,
                          const uint32_t* act, uint64_t na, int32_t* d_den) {
    if (cap < 2 || cap > 31 || S < 2 || na == 0 || d < 1 || d > 4) return false;
    const char* off = getenv("SKYGPU_CELLS_SMEM");
    if (off && off[0] == '0') return false;
    const uint32_t ealloc = (uint32_t)cap + 1;  // values in [0, 1]: codes 0 .. cap
    uint64_t rows = 1;
    for (int j = 1; j < d; ++j) rows *= ealloc;
    const size_t smem = rows * sizeof(uint32_t);
    if (smem > kSmemGridMax) return false;
    static bool attr_set = false;
    if (!attr_set) {
        SKY_CUDA(cudaFuncSetAttribute(k_cells_smem, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)kSmemGridMax));
        attr_set = true;
    }
    const uint32_t G = (uint32_t)(cap - 1);
    uint64_t per_step = ((uint64_t)c.num_sms * 2 + G - 1) / G;
    per_step = std::max<uint64_t>(1, std::min<uint64_t>(per_step, (na + 63) / 64));
    const uint32_t per_block = (uint32_t)((na + per_step - 1) / per_step);
    pdl_launch(k_cells_smem, dim3((unsigned)per_step, G), kSmemBlock, smem, c.stream,
        d_skyv, (uint32_t)S, d, cap, 0.0, act, (uint32_t)na, per_block, d_den, c.d_slots,
        ealloc);
    SKY_LAUNCH_CHECK();
    note_launch(c);
    return true;
}

// Cell engine over S skyline tuples (SoA d_skyv), candidates act[0..na),
// denominators into d_den (pre-zeroed); returns false (nothing done) when the
// engine does not apply.  Runs steps g_max .. 2, stopping once every
// candidate has its answer.
// The steps a shard of the scan runs (shard_world > 1: the cell engine is
// split by STEP, every candidate on every rank — den = the MAX over ranks of
// each rank's largest dominated step, so one MAX all-reduce combines them).
// Longest-processing-time assignment over a per-step cost model (grid bytes
// swept ~7 x rows x word, plus the mark and query reads of S codes); the
// same on every rank (it depends only on the replicated skyline).
std::vector<int> cells_step_plan(const std::vector<double>& amax, int d, int g_max, uint64_t S,
                                 int rank, int world) {
    std::vector<int> mine;
    if (world <= 1) {
        for (int g = g_max; g >= 2; --g) mine.push_back(g);
        return mine;
    }
    std::vector<std::pair<double, int>> cost;
    for (int g = g_max; g >= 2; --g) {
        // bytes swept (~7 x the grid: filled, three read+write passes) plus
        // the mark and query reads of S code words
        MinGeom mg;
        CellGeom geo;
        uint64_t e0 = 0;
        double grid = 0.0;
        if (min_geometry(amax, d, g, ~0ULL, &mg))
            grid = (double)mg.bytes;
        else if (cells_geometry(amax, d, g, ~0ULL, &geo, &e0))
            grid = 4.0 * (double)geo.rows;
        cost.push_back({7.0 * grid + 24.0 * (double)S, g});
    }
    std::stable_sort(cost.begin(), cost.end(),
                     [](const std::pair<double, int>& x, const std::pair<double, int>& y) {
                         return x.first > y.first;
                     });
    std::vector<double> load(world, 0.0);
    for (const auto& cg : cost) {
        int best = 0;
        for (int r = 1; r < world; ++r)
            if (load[r] < load[best]) best = r;
        load[best] += cg.first;
        if (best == rank) mine.push_back(cg.second);
    }
    std::sort(mine.begin(), mine.end(), [](int x, int y) { return x > y; });
    return mine;
}

// Cell engine over S skyline tuples (SoA d_skyv), candidates act[0..na),
// denominators into d_den (pre-zeroed); returns false (nothing done) when the
// engine does not apply.  Runs this shard's steps (all of g_max .. 2 when
// unsharded) in descending order, each step's candidates the previous step's
// undecided ones.
bool gres_cells_device(Ctx& c, const double* d_skyv, uint64_t S, int d, int g_max,
                       const uint32_t* act, uint64_t na, int32_t* d_den, uint64_t* cells_swept,
                       int* steps_run, int step_rank, int step_world) {
    if (g_max < 2 || S == 0 || d > kMaxCellDims) return false;
    auto* colmax = c.buf[B_AMAX].as<unsigned long long>(kMaxDims);
    SKY_CUDA(cudaMemsetAsync(colmax, 0, sizeof(unsigned long long) * kMaxDims, c.stream));
    pdl_launch(k_col_max, dim3(grid_for(S, kBlock, 296), (unsigned)d), kBlock, 0, c.stream, d_skyv,
               S, d, colmax);
    SKY_LAUNCH_CHECK();
    note_launch(c);
    std::vector<unsigned long long> bits(d);
    SKY_CUDA(cudaMemcpyAsync(bits.data(), colmax, sizeof(unsigned long long) * d,
                             cudaMemcpyDeviceToHost, c.stream));
    SKY_CUDA(cudaStreamSynchronize(c.stream));
    std::vector<double> amax(d);
    for (int j = 0; j < d; ++j) memcpy(&amax[j], &bits[j], 8);
    // memory budget: 16 GiB of rows at most
    const uint64_t budget_rows = (16ull << 30) / 8;
    // the min-grid form (default; SKYGPU_CELLS_BITSET=1: the bitset rows)
    static const bool bitset = [] {
        const char* e = getenv("SKYGPU_CELLS_BITSET");
        return e && e[0] == '1';
    }();
    MinGeom mg0;
    const bool minform = !bitset && d <= 8 && S * 8 <= (16ull << 30) &&
                         min_geometry(amax, d, g_max, 16ull << 30, &mg0);
    CellGeom geo0;
    uint64_t e0 = 0;
    if (!minform && !cells_geometry(amax, d, g_max, budget_rows, &geo0, &e0)) return false;
    const bool w64 = e0 > 32;
    const std::vector<int> steps = cells_step_plan(amax, d, g_max, S, step_rank, step_world);
    *cells_swept = 0;
    *steps_run = 0;
    if (steps.empty()) return true;  // (more ranks than steps: nothing here)
    if (minform) {
        MinGeom top;
        min_geometry(amax, d, steps[0], 16ull << 30, &top);
        uint8_t* M = static_cast<uint8_t*>(c.buf[B_CELLS].get(top.bytes));
        const bool cw32 = d <= 4;
        const size_t cwb = cw32 ? 4 : 8;
        const uint64_t chunk = std::min<uint64_t>(64, steps.size());
        void* codes = c.buf[B_CODES].get(S * chunk * cwb);
        uint32_t* lists[2] = {c.buf[B_CACT0].as<uint32_t>(na), c.buf[B_CACT1].as<uint32_t>(na)};
        unsigned long long* cnt[2] = {c.d_slots + S_LIVE0, c.d_slots + S_LIVE1};
        const uint32_t* in = act;
        const unsigned long long* n_in = nullptr;
        int cur = 0, nrun = 0;
        uint64_t swept = 0;
        // locality order (SKYGPU_CELLS_SORT=1; every candidate asked: na ==
        // S with act the identity, the only way this engine is called):
        // values permuted by the top step's row, candidates = sorted
        // positions, den written through the permutation.  Off by default:
        // with one-byte queries the sort and permutation cost more than the
        // locality saves (C5: 1.1 ms against ~0.7 ms)
        static const bool nosort = [] {
            const char* e = getenv("SKYGPU_CELLS_SORT");
            return !(e && e[0] == '1');
        }();
        const double* vals = d_skyv;
        const uint32_t* perm = nullptr;
        static const bool nopriv = [] {  // SKYGPU_MG_NOPRIV=1: every step marks in HBM
            const char* e = getenv("SKYGPU_MG_NOPRIV");
            return e && e[0] == '1';
        }();
        uint32_t* stage = c.buf[B_MGSTAGE].as<uint32_t>((uint64_t)c.num_sms * 4 * kPrivCells / 4);
        static bool priv_attr = false;
        if (!priv_attr) {
            SKY_CUDA(cudaFuncSetAttribute(k_mg_mark_priv<uint32_t>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)(kPrivCells * 4)));
            SKY_CUDA(cudaFuncSetAttribute(k_mg_mark_priv<unsigned long long>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)(kPrivCells * 4)));
            priv_attr = true;
        }
        if (!nosort && na == S) {
            auto* k0 = c.buf[B_MGKEY0].as<unsigned long long>(S);
            auto* k1 = c.buf[B_MGKEY1].as<unsigned long long>(S);
            auto* i0 = c.buf[B_MGIDX0].as<uint32_t>(S);
            auto* i1 = c.buf[B_MGIDX1].as<uint32_t>(S);
            double* pv = c.buf[B_MGVALS].as<double>(S * (uint64_t)d);
            pdl_launch(k_mg_sortkey, grid_for(S, kBlock), kBlock, 0, c.stream, d_skyv, S, d, top, k0,
                       i0);
            SKY_LAUNCH_CHECK();
            cub::DoubleBuffer<unsigned long long> kb(k0, k1);
            cub::DoubleBuffer<uint32_t> vb(i0, i1);
            const int end_bit = std::max(1, 64 - __builtin_clzll(top.bytes));
            size_t tmp = 0;
            SKY_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, kb, vb, (int64_t)S, 0, end_bit,
                                                     c.stream));
            void* t = c.buf[B_CUB].get(tmp);
            SKY_CUDA(cub::DeviceRadixSort::SortPairs(t, tmp, kb, vb, (int64_t)S, 0, end_bit,
                                                     c.stream));
            perm = vb.Current();
            pdl_launch(k_mg_permute, grid_for(S, kBlock), kBlock, 0, c.stream, d_skyv, S, d, perm, pv);
            SKY_LAUNCH_CHECK();
            note_launch(c, 6);
            vals = pv;
            in = nullptr;  // the identity over sorted positions
            swept += S * (uint64_t)d * 8 * 2 + S * 24;
        }
        // marks through a u32 copy of the grid while the copy stays small (see
        // k_mg_mark32; SKYGPU_MG_RED_MB = the copy's size limit, 0 = never;
        // C5 gres: never 6.26 ms, 16 MB 6.16, 64 MB 6.09, 128 MB 6.14, 256 MB
        // 6.53, always 7.61).  (B_MGVALS holds the permuted values of the
        // locality order otherwise)
        static const uint64_t red_bytes = [] {
            const char* e = getenv("SKYGPU_MG_RED_MB");
            const double mb = e ? atof(e) : 64.0;
            return (uint64_t)(mb * 1048576.0);
        }();
        uint32_t* G32 = nullptr;
        if (red_bytes && vals == d_skyv)
            G32 = static_cast<uint32_t*>(
                c.buf[B_MGVALS].get(std::min<uint64_t>(red_bytes, top.bytes * 4)));
        for (size_t s0 = 0; s0 < steps.size(); s0 += chunk) {
            StepList sl;
            sl.n = (int)std::min<uint64_t>(chunk, steps.size() - s0);
            for (int i = 0; i < sl.n; ++i) sl.g[i] = steps[s0 + i];
            if (cw32)
                pdl_launch(k_cells_codes<uint32_t>, grid_for(S, kBlock), kBlock, 0, c.stream,
                           vals, S, d, sl, (uint32_t*)codes);
            else
                pdl_launch(k_cells_codes<unsigned long long>, grid_for(S, kBlock), kBlock, 0,
                           c.stream, vals, S, d, sl, (unsigned long long*)codes);
            SKY_LAUNCH_CHECK();
            note_launch(c);
            swept += S * (uint64_t)d * sizeof(double) + S * (uint64_t)sl.n * cwb;
            for (int li = 0; li < sl.n; ++li) {
                MinGeom geo;
                min_geometry(amax, d, sl.g[li], 16ull << 30, &geo);
                // (SKYGPU_MG_PRIV_CELLS: the privatised range, at most kPrivCells;
                // the u32 RED marks take over above it.  C5 gres: 40960 cells
                // 6.09 ms, 20000 (g <= 4) 6.03, 2000 6.20, none 6.78)
                static const uint64_t priv_cells = [] {
                    const char* e = getenv("SKYGPU_MG_PRIV_CELLS");
                    const long long v = e ? atoll(e) : 20000;
                    return v > 0 && v <= (long long)kPrivCells ? (uint64_t)v : (uint64_t)kPrivCells;
                }();
                const bool priv = !nopriv && geo.bytes <= priv_cells;
                const uint32_t nslots =
                    (uint32_t)c.num_sms * (geo.bytes * 4 <= 48 * 1024 ? 4u : 1u);
                const unsigned gs = grid_for(S, kBlock);
                const unsigned gq = grid_for(na, kBlock);
                int nl = 0, nl_extra = 0;
                auto run = [&](auto* cg) {
                    using CW = std::remove_const_t<std::remove_pointer_t<decltype(cg)>>;
                    if (priv) {
                        pdl_launch(k_mg_mark_priv<CW>, nslots, kBlock, (size_t)geo.bytes * 4,
                                   c.stream, cg, S, geo, stage, n_in, cnt[cur]);
                        pdl_launch(k_mg_mark_reduce, grid_for(geo.bytes / 4, kBlock), kBlock, 0,
                                   c.stream, (const uint32_t*)stage, nslots,
                                   (uint32_t)(geo.bytes / 4), (uint32_t*)M, n_in);
                    } else if (G32 && geo.bytes * 4 <= red_bytes) {
                        uint32_t* G = G32;
                        pdl_launch(k_mg_fill32, grid_for(geo.bytes / 4, kBlock), kBlock, 0,
                                   c.stream, (uint4*)G, geo.bytes / 4, n_in, cnt[cur]);
                        pdl_launch(k_mg_mark32<CW>, gs, kBlock, 0, c.stream, cg, S, geo, G, n_in);
                        pdl_launch(k_mg_pack, grid_for(geo.bytes / 4, kBlock), kBlock, 0, c.stream,
                                   (const uint4*)G, geo.bytes / 4, (uint32_t*)M, n_in);
                        ++nl_extra;
                    } else {
                        pdl_launch(k_mg_fill, grid_for(geo.bytes / 16, kBlock), kBlock, 0,
                                   c.stream, (uint4*)M, geo.bytes / 16, n_in, cnt[cur]);
                        // an L2 load before the CAS for the small grids (up to
                        // SKYGPU_MG_LOADFIRST_MB, default 4 MB: many tuples per
                        // cell, most of them lower nothing — the load spares the
                        // serialised same-address atomics); CAS first for the
                        // large ones, where the load would be a second DRAM trip
                        // (C5 gres: always 6.54 ms, never 6.41 ms, <= 4 MB 6.27 ms)
                        static const uint64_t lf_bytes = [] {
                            const char* e = getenv("SKYGPU_MG_LOADFIRST_MB");
                            const double mb = e ? atof(e) : 4.0;
                            return (uint64_t)(mb * 1048576.0);
                        }();
                        const bool load_first = geo.bytes <= lf_bytes;
                        if (load_first)
                            pdl_launch(k_mg_mark<CW, true>, gs, kBlock, 0, c.stream, cg, S, geo, M,
                                       n_in);
                        else
                            pdl_launch(k_mg_mark<CW, false>, gs, kBlock, 0, c.stream, cg, S, geo, M,
                                       n_in);
                    }
                    nl = min_sweeps(c, M, geo, n_in);
                    pdl_launch(k_mg_query<CW>, gq, kBlock, 0, c.stream, cg, geo, (const uint8_t*)M,
                               in, na, n_in, d_den, perm, lists[cur], cnt[cur]);
                };
                if (cw32)
                    run((const uint32_t*)codes + (uint64_t)li * S);
                else
                    run((const unsigned long long*)codes + (uint64_t)li * S);
                SKY_LAUNCH_CHECK();
                note_launch(c, 3 + nl + nl_extra);
                // algorithmic bytes of the step: the grid filled, read and
                // written once by an ideal fused prefix minimum, plus the
                // mark and query reads of the S code words
                swept += 3 * geo.bytes + 2 * S * cwb;
                ++nrun;
                in = lists[cur];
                n_in = cnt[cur];
                cur ^= 1;
            }
        }
        *cells_swept = swept;
        *steps_run = nrun;
        return true;
    }
    {
        CellGeom gt;
        uint64_t et = 0;
        cells_geometry(amax, d, steps[0], budget_rows, &gt, &et);
        c.buf[B_CELLS].get(gt.rows * (w64 ? 8 : 4));
    }
    void* rows = c.buf[B_CELLS].p;
    // codes of up to 64 steps at a time (packed bytes; d <= 8 here)
    const bool cw32 = d <= 4;
    const size_t cwb = cw32 ? 4 : 8;
    const uint64_t chunk = std::min<uint64_t>(64, steps.size());
    const bool use_codes = d <= 8 && S * chunk * cwb <= (16ull << 30);
    void* codes = use_codes ? c.buf[B_CODES].get(S * chunk * cwb) : nullptr;
    uint64_t swept = 0;
    int nrun = 0;
    const char* uf = getenv("SKYGPU_CELLS_UNFUSED");
    const bool fused = !(uf && uf[0] == '1');
    // undecided candidates ping-pong between two lists; a step's count lives
    // in a device slot that gates every kernel of the next step, so the
    // steps are queued back to back without a host round trip
    uint32_t* lists[2] = {c.buf[B_CACT0].as<uint32_t>(na), c.buf[B_CACT1].as<uint32_t>(na)};
    unsigned long long* cnt[2] = {c.d_slots + S_LIVE0, c.d_slots + S_LIVE1};
    const uint32_t* in = act;
    const unsigned long long* n_in = nullptr;
    int cur = 0;
    for (size_t s0 = 0; s0 < steps.size(); s0 += chunk) {
        StepList sl;
        sl.n = (int)std::min<uint64_t>(chunk, steps.size() - s0);
        for (int i = 0; i < sl.n; ++i) sl.g[i] = steps[s0 + i];
        if (codes) {
            if (cw32)
                pdl_launch(k_cells_codes<uint32_t>, grid_for(S, kBlock), kBlock, 0, c.stream,
                           d_skyv, S, d, sl, (uint32_t*)codes);
            else
                pdl_launch(k_cells_codes<unsigned long long>, grid_for(S, kBlock), kBlock, 0,
                           c.stream, d_skyv, S, d, sl, (unsigned long long*)codes);
            SKY_LAUNCH_CHECK();
            note_launch(c);
            swept += S * (uint64_t)d * sizeof(double) + S * (uint64_t)sl.n * cwb;
        }
        for (int li = 0; li < sl.n; ++li) {
            const int g = sl.g[li];
            CellGeom geo;
            uint64_t e0g = 0;
            cells_geometry(amax, d, g, budget_rows, &geo, &e0g);
            const size_t wb = w64 ? 8 : 4;
            const uint64_t n16 = (geo.rows * wb + 15) / 16;
            pdl_launch(k_cells_zero, grid_for(n16, kBlock), kBlock, 0, c.stream, (uint4*)rows, n16,
                       n_in);
            pdl_launch(k_clear_slot_c, 1, 1, 0, c.stream, cnt[cur]);
            const unsigned gs = grid_for(S, kBlock);
            const unsigned gq = grid_for(na, kBlock);
            auto run_codes = [&](auto* R, auto* cg) {
                using WR = std::remove_pointer_t<decltype(R)>;
                using CW = std::remove_const_t<std::remove_pointer_t<decltype(cg)>>;
                pdl_launch(k_cells_mark_c<WR, CW>, gs, kBlock, 0, c.stream, cg, S, geo, R, n_in);
                sweeps<WR>(c, R, geo, fused, n_in);
                pdl_launch(k_cells_query_c<WR, CW>, gq, kBlock, 0, c.stream, cg, geo,
                           (const WR*)R, in, na, n_in, d_den, lists[cur], cnt[cur]);
            };
            auto run_vals = [&](auto* R) {
                using WR = std::remove_pointer_t<decltype(R)>;
                pdl_launch(k_cells_mark<WR>, gs, kBlock, 0, c.stream, d_skyv, S, geo, R, n_in);
                sweeps<WR>(c, R, geo, fused, n_in);
                pdl_launch(k_cells_query<WR>, gq, kBlock, 0, c.stream, d_skyv, S, geo,
                           (const WR*)R, in, na, n_in, d_den, lists[cur], cnt[cur]);
            };
            const uint64_t coff = (uint64_t)li * S;
            if (codes && w64 && cw32)
                run_codes(static_cast<unsigned long long*>(rows), (const uint32_t*)codes + coff);
            else if (codes && w64)
                run_codes(static_cast<unsigned long long*>(rows),
                          (const unsigned long long*)codes + coff);
            else if (codes && cw32)
                run_codes(static_cast<unsigned*>(rows), (const uint32_t*)codes + coff);
            else if (codes)
                run_codes(static_cast<unsigned*>(rows), (const unsigned long long*)codes + coff);
            else if (w64)
                run_vals(static_cast<unsigned long long*>(rows));
            else
                run_vals(static_cast<unsigned*>(rows));
            SKY_LAUNCH_CHECK();
            note_launch(c, 4);
            // algorithmic bytes of the step: the grid zeroed, read and
            // written once by an ideal fused prefix-OR, plus the mark and
            // query reads of the S codes (or values)
            swept += 3 * geo.rows * wb + 2 * S * (codes ? cwb : (uint64_t)d * sizeof(double));
            ++nrun;
            in = lists[cur];
            n_in = cnt[cur];
            cur ^= 1;
        }
    }
    *cells_swept = swept;
    *steps_run = nrun;
    return true;
}

}  // namespace skygpu
