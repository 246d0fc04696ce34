// sky_common.cuh — shared pieces of libskygpu: per-device context with cached
// device buffers, error plumbing, and the dominance primitives.
//
// Dominance (core.hpp:55-67): s dominates t iff s_i <= t_i for every i and
// s_i < t_i for some i.  Values are compared as float64 with exact IEEE
// semantics (no epsilon); -0.0 == +0.0 as in the reference.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "skygpu.h"

namespace skygpu {

constexpr int kMaxDims = 32;  // generic-path limit (template paths cover d <= 8)

struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define SKY_CUDA(call)                                                                   \
    do {                                                                                 \
        cudaError_t e_ = (call);                                                         \
        if (e_ != cudaSuccess)                                                           \
            throw ::skygpu::Error(e_ == cudaErrorMemoryAllocation ? SKYGPU_ENOMEM          \
                                                                  : SKYGPU_ECUDA,        \
                                  std::string(#call) + ": " + cudaGetErrorString(e_));   \
    } while (0)

#define SKY_LAUNCH_CHECK() SKY_CUDA(cudaGetLastError())

// Programmatic dependent launch: every kernel of the library starts with
// pdl_wait() (griddepcontrol.wait: a no-op for a normally launched grid; for a
// PDL-launched one it waits until the preceding grid's memory is visible), so
// each launch may let the next grid be scheduled early — the kernel-to-kernel
// bubble of a ~30-launch call shrinks.  SKYGPU_PDL=0 launches normally.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

inline bool pdl_enabled() {
    static const bool on = [] {
        const char* e = getenv("SKYGPU_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}

template <typename... KArgs, typename... Args>
inline void pdl_launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t stream, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    SKY_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

inline void invalid(const std::string& m) { throw Error(SKYGPU_EINVAL, m); }

// Growable device buffer owned by the context (never shrinks until release).
struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    void* get(size_t bytes) {
        if (bytes == 0) bytes = 16;
        if (bytes > cap) {
            if (p) cudaFree(p);
            p = nullptr;
            cap = 0;
            size_t want = bytes + bytes / 8 + 256;
            SKY_CUDA(cudaMalloc(&p, want));
            cap = want;
        }
        return p;
    }
    template <class T>
    T* as(size_t count) { return static_cast<T*>(get(count * sizeof(T))); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
};

enum BufId {
    B_IN_VALS, B_IN_IDS, B_KEY0, B_KEY1, B_IDX0, B_IDX1, B_SV, B_SID, B_SPOS,
    B_R0, B_R1, B_FLAGS, B_KLIST, B_CUB, B_SKYV, B_SKYID, B_CODES, B_ACT0, B_ACT1,
    B_DEN, B_GTMP0, B_GTMP1, B_OUTPOS, B_PROJ, B_REPS, B_MISC, B_CELLS, B_CSUM,
    B_ORDER, B_AMAX, B_AQ, B_PQ, B_GCODE, B_GCELL, B_GSCODE, B_GSIDX, B_GITEMS, B_GCNT,
    B_ACC0, B_ACC1, B_ACC2, B_ACC3, B_ACC4, B_ACC5, B_ACC6, B_ACC7, B_ACC8, B_ACC9, B_ACC10,
    B_ACC11, B_ACC12, B_ACC13, B_ACC14, B_ACC15, B_ACC16, B_SEED, B_AMAX2, B_IOTA, B_NORM, B_CSV, B_CSVVAL, B_CHIST, B_CCUR, B_GREC, B_CACT0, B_CACT1, B_MGKEY0, B_MGKEY1, B_MGIDX0, B_MGIDX1, B_MGVALS, B_MGSTAGE, B_GIOTA, B_GSKEY,
    B_PPID, B_PHIST, B_PTHR, B_PWPOS, B_PWV, B_PWKEY, B_PWTIE, B_PSK0, B_PSK1, B_PSV0, B_PSV1,
    B_PFLAGS, B_COUNT
};

// Device-side scalar slots (one small allocation, read back through pinned memory).
enum Slot {
    S_SEL = 0,         // DeviceSelect count
    S_TESTS_SKY = 1,   // dominance tests, skyline stage
    S_TESTS_GRES = 2,  // code tests, gres stage
    S_UNITS_SKY = 3,  // rank-grid K6: (comparator, item) bitset tests
    S_MINGAP = 4,      // bits of the min positive gap (atomicMin)
    S_MAXV = 5,        // bits of max |value| (atomicMax)
    S_BAD = 6,         // first tuple index with a negative/NaN value (atomicMin; ~0 = none)
    S_FLAG = 7,        // generic flag
    S_PAIR = 8,        // check_skyline: min (a*S + b) (~0 = none)
    S_SEL2 = 9,
    S_GRIDBAD = 10,     // first flat index of a Grid value outside [0,1]
    S_SMIN = 11,       // ord bits of the min / max tuple sum (skyline rounds)
    S_SMAX = 12,
    S_THR = 13,        // bits of the prefix threshold T (double)
    S_C1 = 14,         // prefix size
    S_C2 = 15,         // new skyline tuples of the round
    S_C3 = 16,         // survivors of the round
    S_GATE = 17,       // 1: the first round asks for the rank-grid engine (K5 skipped)
    S_SPEC = 18,       // 1: the speculative gres launch did not apply (gres.cu), redo
    S_IDSBAD = 19,     // 1: ids that arrived late were not strictly increasing, redo
    S_LIVE0 = 20,      // cell engine: undecided candidates after a step (ping-pong)
    S_LIVE1 = 21,
    S_LPS_N = 22,      // local pruning: sampled tuples / those the windows dominate
    S_LPS_HIT = 23,
    S_COUNT_ = 24
};

struct Ctx {
    int device = 0;
    cudaStream_t own = nullptr;
    cudaStream_t stream = nullptr;
    DevBuf buf[B_COUNT];
    unsigned long long* d_slots = nullptr;
    unsigned long long* h_slots = nullptr;  // pinned mirror
    cudaEvent_t ev[18];
    skygpu_stats* st = nullptr;
    uint64_t launches = 0;
    int num_sms = 148;
    bool gres_timing_pending = false;  // ev[10]/ev[11] span awaiting the final sync
    // SKYGPU_TRACE=1: device timestamps between phases (events only, no sync),
    // printed to stderr at the end of the call
    bool trace = false;
    int ntrace = 0;
    cudaStream_t copy = nullptr;  // H2D of streamed pipeline inputs
    // sharded pipeline call in progress (skygpu_set_collective installed)
    skygpu_allreduce_max_fn coll = nullptr;
    void* coll_user = nullptr;
    // NCCL communicator of the shard group (skygpu_nccl_init): when set, the
    // exchange steps are ncclAllReduce(MAX) queued on this context's stream
    void* nccl = nullptr;
    int nccl_rank = 0, nccl_world = 1;
    int shard_rank = 0, shard_world = 1;
    cudaEvent_t xev[10];          // chunk-ready events of the streamed input
    cudaEvent_t tev[96];
    const char* tlabel[96];
    double thost[96];  // host clock at each mark (us): where the GPU waits for the CPU
    int trace_chunks = 0;  // streamed chunks whose arrival the trace reports
    bool gres_spec = false;  // a speculative gres launch awaits its S_SPEC check
    bool counters_fetched = false;  // test counters already read with the outputs
    bool chist_zeroed = false;      // the A' cell histogram (B_CHIST) starts zeroed
    // event spans of the current call, resolved by end_stats after the call's
    // final synchronisation (per context: one host thread per device may run
    // calls concurrently with another device's)
    struct Span {
        int a;
        double* dst;
    } spans[8];
    int nspans = 0;
    skygpu_stats scratch_stats;  // the call's stats when the caller passed none
    void* hbuf[4] = {nullptr, nullptr, nullptr, nullptr};  // pinned staging (skygpu_host_buffer)
    size_t hcap[4] = {0, 0, 0, 0};
    // host-pointer pipeline: the ids are still in flight (copy stream) until
    // this event; the skyline runs on the speculation that they are strictly
    // increasing (ties by position) and checks them at the end (S_IDSBAD)
    cudaEvent_t ids_ready = nullptr;
    // (or not yet issued: the copy of these host ids is queued by the
    // skyline itself when K5 starts — a latency-bound kernel the copy's
    // traffic barely slows, unlike the HBM-bound ones before it)
    const int64_t* ids_host = nullptr;
    int64_t* ids_dev = nullptr;
    uint64_t ids_n = 0;
    // SKYGPU_SKY_PARTS: local-skyline pruning per plan partition before the
    // merge (partition.cu), set for the duration of one call
    bool local_prune = false;
};

// record a labelled device timestamp when tracing is on
void trace_mark(Ctx& c, const char* label);

Ctx& ctx();  // current device's context (created lazily)

inline void note_launch(Ctx& c, uint64_t k = 1) { c.launches += k; }

// Read `count` slots back (synchronises the stream).
void read_slots(Ctx& c, int first, int count);
// Stream-ordered (re)initialisation of the scalar slots, no host sync.
// zero_slots keeps the two test counters; reset_tests clears them;
// reset_counts clears only the round counters S_C1..S_C3.
void zero_slots(Ctx& c);
void reset_tests(Ctx& c);
void reset_counts(Ctx& c);
void reset_range(Ctx& c);  // S_SMIN / S_SMAX

// ---------------------------------------------------------------- dominance
// s dominates t on D float64 attributes (branch-free form of core.hpp:55-67).
template <int D>
__device__ __forceinline__ bool dom_f64(const double* s, const double* t) {
    bool le = true, lt = false;
#pragma unroll
    for (int k = 0; k < D; ++k) {
        le &= (s[k] <= t[k]);
        lt |= (s[k] < t[k]);
    }
    return le & lt;
}

__device__ __forceinline__ bool dom_f64_dyn(const double* s, const double* t, int d) {
    bool le = true, lt = false;
    for (int k = 0; k < d; ++k) {
        le &= (s[k] <= t[k]);
        lt |= (s[k] < t[k]);
    }
    return le & lt;
}

// Packed u8 codes (one byte per attribute, code <= 127, d <= 8): s dominates
// t at this step iff every byte of s <= the byte of t and the words differ.
// tg = t | H: bit 7 of each byte of (tg - s) is set iff t_byte >= s_byte
// (no borrow can cross a byte since 128 + t - s >= 1).
constexpr uint64_t kGuard = 0x8080808080808080ULL;
__device__ __forceinline__ bool dom_u8(uint64_t s, uint64_t t, uint64_t tg) {
    return (((tg - s) & kGuard) == kGuard) & (s != t);
}

__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    return v;
}

// lane 0 of each warp adds the warp's total into *dst
__device__ __forceinline__ void add_count(unsigned long long* dst, unsigned long long v) {
    v = warp_sum_u64(v);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(dst, v);
}

// bits of a non-negative double, canonicalising -0.0 to +0.0 so that the
// unsigned order of the bits equals the numeric order
__device__ __forceinline__ unsigned long long ord_bits(double v) {
    return v == 0.0 ? 0ULL : static_cast<unsigned long long>(__double_as_longlong(v));
}

inline unsigned grid_for(uint64_t n, int block, int cap_blocks = 148 * 32) {
    uint64_t b = (n + block - 1) / block;
    if (b < 1) b = 1;
    if (b > (uint64_t)cap_blocks) b = cap_blocks;
    return static_cast<unsigned>(b);
}

// ------------------------------------------------------------- stage APIs
struct SkylineOut {
    uint64_t S = 0;
    // device: sorted-order positions of skyline tuples (u32), S entries, in
    // (sum, id) order; input positions (u32) and ids (i64) of the same.
    uint32_t* d_inpos = nullptr;
    int64_t* d_ids = nullptr;
    double* d_skyv = nullptr;  // SoA [d][S]
    uint64_t* d_pos64 = nullptr;  // the input positions widened to u64 (the output format)
    bool aborted = false;      // kSkyAbortIfLarge: the first round asked for the rank grid
};

// internal sky_engine bit: give up (aborted = true) instead of switching to
// the rank-grid engine — the streamed head only wants a small skyline
constexpr unsigned kSkyAbortIfLarge = 0x100u;
// internal sky_engine bit: stop after the first round and return that
// prefix's skyline (a seed: not final, any dominating predecessor filters)
constexpr unsigned kSkyFirstPrefix = 0x200u;

// Skyline of n tuples already resident on the device (AoS vals, ids).
// Input still arriving (host-pointer pipeline): chunk ch = positions
// [bound[ch], bound[ch+1]) is on the device once ready[ch] has fired.
// The first prefix of chunk 0 (the head) is decided while the rest is in
// flight; its skyline then filters every chunk as it lands (skyline.cu).
struct TailFeed {
    int nchunks = 0;
    uint64_t bound[9] = {};
    cudaEvent_t ready[8] = {};
};

// sky_engine: 0 auto, SKYGPU_SKY_ROUNDS or SKYGPU_SKY_GRID (skygpu.h flags)
SkylineOut skyline_device(Ctx& c, const double* d_vals, const int64_t* d_ids, uint64_t n, int d,
                          const skygpu_plan& plan, const double* d_reps, uint64_t n_reps,
                          unsigned sky_engine = 0, const TailFeed* feed = nullptr);

// skyline_grid.cu: the one-pass rank-grid engine for large skylines.
// sky_grid_bins = bins per attribute for r tuples (0: shape unsupported, d > 8);
// sky_grid_decide writes keep[i] = 1 iff tuple R[i] (R == nullptr: i) is kept
// by the predecessor rule over R; adds the decide kernel's time to *kernel_ms
// (synchronising on it) when kernel_ms != nullptr.
int sky_grid_bins(uint64_t r, int d);
void sky_grid_decide(Ctx& c, const double* d_vals, int d, const unsigned long long* keys,
                     const int64_t* d_ids, const uint32_t* R, uint64_t r, uint8_t* keep,
                     double* kernel_ms, int shard_rank = 0, int shard_world = 1);

// the installed MAX all-reduce over the shard group (see skygpu.h)
void shard_allreduce_max(Ctx& c, void* dev_ptr, uint64_t count, int elem_bytes);

struct GresOut {
    int g_max = 1;
    int steps = 0;
};

// Grid resistance of S skyline tuples held SoA on the device (d_skyv[d][S]).
// d_den (S entries) receives the denominators (0 for tuples outside this
// shard).  Throws Error(EINVAL, ...) exactly where the reference throws.
// allow_spec: the caller checks gres_spec_failed() after its final
// synchronisation (and re-runs with allow_spec = false when it did)
GresOut gres_device(Ctx& c, const double* d_skyv, const int64_t* d_ids, uint64_t S, int d,
                    int cap, int engine, int shard_rank, int shard_world, bool check_skyline,
                    int32_t* d_den, bool allow_spec = false);
// queue the deferred copy of the host ids (Ctx::ids_host), once
void issue_late_ids(Ctx& c);
// queue the read of the speculation flag (before the caller's final sync)
void gres_spec_fetch(Ctx& c);
// after that sync: true when the speculative launch did not apply
bool gres_spec_failed(Ctx& c);

// Grid plan inside the scan: throw the reference's grid_cell error when a
// projection at step g leaves [0,1]
void check_grid_projection(Ctx& c, const double* d_skyv, uint64_t S, int d, int g);

// cells.cu: the cell-occupancy gres engine; false when it does not apply
// step_rank / step_world: this shard's steps of the scan (cells_step_plan);
// (0, 1) runs them all
bool gres_cells_device(Ctx& c, const double* d_skyv, uint64_t S, int d, int g_max,
                       const uint32_t* act, uint64_t na, int32_t* d_den, uint64_t* cells_swept,
                       int* steps_run, int step_rank = 0, int step_world = 1);
std::vector<int> cells_step_plan(const std::vector<double>& amax, int d, int g_max, uint64_t S,
                                 int rank, int world);
// cells.cu: the same engine with every step in one launch and the grids in
// shared memory (d <= 4, small code extents); false when it does not apply
bool gres_cells_smem_device(Ctx& c, const double* d_skyv, uint64_t S, int d, int g_max,
                            double maxv, const uint32_t* act, uint64_t na, int32_t* d_den);
// the same launch before g_max and the value range are known on the host
// (capped scans): g_max = cap when the device gap witness fired, codes within
// an extent of cap + 1; otherwise it sets S_SPEC and does nothing
bool gres_cells_smem_spec(Ctx& c, const double* d_skyv, uint64_t S, int d, int cap,
                          const uint32_t* act, uint64_t na, int32_t* d_den);

// accounting.cu: exact SFS DominanceCounter totals of one phase (groups =
// partitions, gid < 0 = not in the phase, optional representatives); adds
// the tests per group into d_per_group and writes the kept positions (group
// by group, (sum, id) order) into d_kept; returns how many
uint64_t sfs_accounting_device(Ctx& c, const double* d_vals, const int64_t* d_ids, uint64_t n,
                               int d, const int32_t* d_gid, uint32_t p, const double* d_reps,
                               uint32_t nr, unsigned long long* d_per_group, uint32_t* d_kept);

// ingest.cu: min-max normalisation (harness.cpp:161-177), bit-exact; and the
// representative selection (partition.cpp:229-271): writes the kept picks'
// positions in (sum, id) order, adds the pruning tests to *d_tests
void normalize_device(Ctx& c, const double* d_in, uint64_t n, int d, double* d_out);
uint64_t select_representatives_device(Ctx& c, const double* d_vals, const int64_t* d_ids,
                                       uint64_t n, int d, uint64_t k, uint32_t* d_out,
                                       unsigned long long* d_tests);

// csv.cu: the reference's read_dataset_csv on the device (data lines only;
// the header fixes dims).  0 ok; 1 d_vals too small (*rows set); 2 a format
// error at (*err_line, *err_col, *err_kind: 1 field count, 2 not a number,
// 3 negative); *internal != 0 when a field exceeded the device parser's limits
int csv_parse_device(Ctx& c, const char* d_bytes, uint64_t len, int dims, uint64_t* rows,
                     double* d_vals, uint64_t vals_cap, uint64_t* err_line, int* err_col,
                     int* err_kind, int* internal);

// partition.cu: assign_partitions (partition.cpp:183-213) on the device —
// d_pid[i] = partition of tuple i in [0, plan.partitions); Grid values outside
// [0,1] set slot S_GRIDBAD (first flat index).  ids_sorted: ids strictly
// increasing in position order (sliced ties then follow positions).
void assign_partitions_device(Ctx& c, const double* d_vals, const int64_t* d_ids, bool ids_sorted,
                              uint64_t n, int d, const skygpu_plan& plan, int32_t* d_pid);
// local-skyline pruning (partition.cu header): keep[i] = 0 for tuples dominated
// by a preceding member of their partition's window skyline (and for tuples
// outside `mask` when given); keys = K1's sum keys, tie_ids = ids or nullptr
// (ties by position)
bool local_prune_applies(const skygpu_plan& plan, int d);
bool plan_ids_in_range(const skygpu_plan& plan, int d);
uint64_t local_prune_device(Ctx& c, const double* d_vals, const unsigned long long* keys,
                            const int64_t* tie_ids, uint64_t n, int d, const skygpu_plan& plan,
                            const uint8_t* mask, uint8_t* keep, uint32_t* stats_parts);

// float64 AoS -> SoA transpose on the device
void aos_to_soa(Ctx& c, const double* d_aos, uint64_t n, int d, double* d_soa);

}  // namespace skygpu
