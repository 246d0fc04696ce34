// abi.cu — the C-ABI of libskygpu (include/skygpu.h): per-device context,
// host<->device staging, exception -> status translation, plan sizing.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <mutex>
#include <string>

#include <dlfcn.h>

#include "sky_common.cuh"

namespace skygpu {

namespace {
Ctx* g_ctx[64] = {nullptr};
cudaStream_t g_user_stream[64] = {nullptr};
bool g_user_stream_set[64] = {false};

void write_err(char* err, size_t errlen, const std::string& m) {
    if (!err || errlen == 0) return;
    size_t k = std::min(errlen - 1, m.size());
    memcpy(err, m.data(), k);
    err[k] = 0;
}

int current_device() {
    int dev = 0;
    SKY_CUDA(cudaGetDevice(&dev));
    return dev;
}
}  // namespace

Ctx& ctx() {
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0)
        throw Error(SKYGPU_ECUDA, std::string("no CUDA device available (") +
                                      cudaGetErrorString(e) + "); libskygpu has no CPU fallback");
    const int dev = current_device();
    if (!g_ctx[dev]) {
        cudaDeviceProp prop;
        SKY_CUDA(cudaGetDeviceProperties(&prop, dev));
        if (prop.major < 10)
            throw Error(SKYGPU_ECUDA, "device " + std::to_string(dev) + " is sm_" +
                                          std::to_string(prop.major) +
                                          std::to_string(prop.minor) +
                                          "; libskygpu is built for sm_100a only");
        Ctx* c = new Ctx();
        c->device = dev;
        c->num_sms = prop.multiProcessorCount;
        SKY_CUDA(cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking));
        c->stream = c->own;
        SKY_CUDA(cudaMalloc(&c->d_slots, sizeof(unsigned long long) * S_COUNT_));
        SKY_CUDA(cudaMallocHost(&c->h_slots, sizeof(unsigned long long) * S_COUNT_));
        for (auto& ev : c->ev) SKY_CUDA(cudaEventCreate(&ev));
        const char* tr = getenv("SKYGPU_TRACE");
        c->trace = tr && tr[0] == '1';
        if (c->trace)
            for (auto& ev : c->tev) SKY_CUDA(cudaEventCreate(&ev));
        g_ctx[dev] = c;
    }
    Ctx& c = *g_ctx[dev];
    c.stream = g_user_stream_set[dev] ? g_user_stream[dev] : c.own;
    return c;
}

void trace_mark(Ctx& c, const char* label) {
    // SKYGPU_TRACE=2: synchronise and print every mark at once (localises a
    // kernel that never returns; timings are meaningless in this mode)
    static const bool sync_marks = [] {
        const char* e = getenv("SKYGPU_TRACE");
        return e && e[0] == '2';
    }();
    if (sync_marks) {
        fprintf(stderr, "[skygpu mark] queued: %s\n", label);
        fflush(stderr);
        const cudaError_t e = cudaStreamSynchronize(c.stream);
        fprintf(stderr, "[skygpu mark] done:   %s (%s)\n", label, cudaGetErrorString(e));
        fflush(stderr);
    }
    if (!c.trace || c.ntrace >= 96) return;
    c.tlabel[c.ntrace] = label;
    c.thost[c.ntrace] = std::chrono::duration<double, std::micro>(
                            std::chrono::steady_clock::now().time_since_epoch())
                            .count();
    SKY_CUDA(cudaEventRecord(c.tev[c.ntrace++], c.stream));
}

void read_slots(Ctx& c, int first, int count) {
    SKY_CUDA(cudaMemcpyAsync(c.h_slots + first, c.d_slots + first,
                             sizeof(unsigned long long) * count, cudaMemcpyDeviceToHost,
                             c.stream));
    SKY_CUDA(cudaStreamSynchronize(c.stream));
}

namespace {
__global__ void k_init_slots(unsigned long long* slots, int mode) {
    pdl_wait();
    const int i = threadIdx.x;
    if (i >= S_COUNT_) return;
    if (mode == 1) {  // test counters only
        if (i == S_TESTS_SKY || i == S_TESTS_GRES || i == S_UNITS_SKY) slots[i] = 0;
        return;
    }
    if (mode == 2) {  // round counters only
        if (i == S_C1 || i == S_C2 || i == S_C3) slots[i] = 0;
        return;
    }
    if (mode == 3) {  // sum range only
        if (i == S_SMIN) slots[i] = ~0ULL;
        if (i == S_SMAX) slots[i] = 0;
        return;
    }
    if (i == S_TESTS_SKY || i == S_TESTS_GRES || i == S_UNITS_SKY || i == S_SPEC || i == S_IDSBAD)
        return;
    unsigned long long v = 0;
    if (i == S_BAD || i == S_PAIR || i == S_GRIDBAD || i == S_SMIN) v = ~0ULL;
    if (i == S_MINGAP) v = 0x7FF0000000000000ULL;
    slots[i] = v;
}
}  // namespace

void zero_slots(Ctx& c) {
    pdl_launch(k_init_slots, 1, 32, 0, c.stream, c.d_slots, 0);
    SKY_LAUNCH_CHECK();
    note_launch(c);
}

void reset_tests(Ctx& c) {
    pdl_launch(k_init_slots, 1, 32, 0, c.stream, c.d_slots, 1);
    SKY_LAUNCH_CHECK();
    note_launch(c);
}

void reset_counts(Ctx& c) {
    pdl_launch(k_init_slots, 1, 32, 0, c.stream, c.d_slots, 2);
    SKY_LAUNCH_CHECK();
    note_launch(c);
}

void reset_range(Ctx& c) {
    pdl_launch(k_init_slots, 1, 32, 0, c.stream, c.d_slots, 3);
    SKY_LAUNCH_CHECK();
    note_launch(c);
}

// gres.cu
bool min_positive_gap_device(Ctx& c, const double* d_soa, uint64_t S, int d, double* gap,
                             double* maxv);

namespace {

__global__ void k_aos_to_soa(const double* __restrict__ a, uint64_t n, int d,
                             double* __restrict__ s) {
    pdl_wait();
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n * d;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t t = i / d;
        int k = (int)(i % d);
        s[(uint64_t)k * n + t] = a[i];
    }
}

__global__ void k_snap(const double* __restrict__ v, uint64_t total, int g,
                       double* __restrict__ out) {
    pdl_wait();
    const double gd = (double)g;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
         i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = __ddiv_rn(floor(__dmul_rn(v[i], gd)), gd);
}

__global__ void k_check_values(const double* __restrict__ v, uint64_t total,
                               unsigned long long* __restrict__ slots) {
    pdl_wait();
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
         i += (uint64_t)gridDim.x * blockDim.x)
        if (!(v[i] >= 0.0)) atomicMin(&slots[S_BAD], (unsigned long long)i);
}

// Event span on the call's stream; stop() only records — the elapsed time
// is resolved by end_stats after the call's single final synchronisation.
struct Timer {
    Ctx& c;
    int a;
    Timer(Ctx& cc, int ea) : c(cc), a(ea) { SKY_CUDA(cudaEventRecord(c.ev[a], c.stream)); }
    void stop(double* dst) {
        SKY_CUDA(cudaEventRecord(c.ev[a + 1], c.stream));
        if (c.nspans < 8) c.spans[c.nspans++] = Ctx::Span{a, dst};
    }
};

void validate_plan(const skygpu_plan* plan, int d) {
    if (!plan) return;
    if (plan->strategy < 0 || plan->strategy > 3) invalid("unknown strategy");
    if (plan->partitions < 1) invalid("partitions must be >= 1");
    (void)d;
}

// local-skyline pruning for one call: the pipeline flag SKYGPU_SKY_PARTS, or
// SKYGPU_LOCAL_PRUNE=1 for every call of the process (the C++ drop-in's
// parallel_skyline has no flags)
bool local_prune_env() {
    static const bool on = [] {
        const char* e = getenv("SKYGPU_LOCAL_PRUNE");
        return e && e[0] == '1';
    }();
    return on;
}

struct LocalPruneScope {
    Ctx& c;
    LocalPruneScope(Ctx& cx, bool on) : c(cx) { c.local_prune = on || local_prune_env(); }
    ~LocalPruneScope() { c.local_prune = false; }
};

template <class F>
int guarded(char* err, size_t errlen, F&& f) {
    try {
        f();
        write_err(err, errlen, "");
        return SKYGPU_OK;
    } catch (const Error& e) {
        write_err(err, errlen, e.what());
        return e.code;
    } catch (const std::bad_alloc&) {
        write_err(err, errlen, "host allocation failed");
        return SKYGPU_ENOMEM;
    } catch (const std::exception& e) {
        write_err(err, errlen, e.what());
        return SKYGPU_ERUNTIME;
    }
}

void begin_stats(Ctx& c, skygpu_stats* st) {
    c.st = st ? st : &c.scratch_stats;
    memset(c.st, 0, sizeof(skygpu_stats));
    c.launches = 0;
    // per-call flags start clear: an earlier call on this device may have
    // thrown mid-pipeline (after fetching its counters, with a speculative
    // gres launch pending, or mid-round)
    c.chist_zeroed = false;
    c.counters_fetched = false;
    c.gres_spec = false;
    c.gres_timing_pending = false;
    c.nspans = 0;
    c.ntrace = 0;
    trace_mark(c, "begin");
    reset_tests(c);
}

// the call's final synchronisation: test counters and event spans
// queue the read of the test counters with a call's outputs (before its
// final synchronisation), so end_stats needs no round trip of its own
void fetch_test_counters(Ctx& c) {
    SKY_CUDA(cudaMemcpyAsync(c.h_slots + S_TESTS_SKY, c.d_slots + S_TESTS_SKY,
                             3 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, c.stream));
    c.counters_fetched = true;
}

void end_stats(Ctx& c) {
    if (c.counters_fetched) {  // read with the outputs: only the timing events
        c.counters_fetched = false;  // recorded since then are left to complete
        SKY_CUDA(cudaStreamSynchronize(c.stream));
    } else {
        read_slots(c, S_TESTS_SKY, 3);
    }
    c.st->skyline_tests = c.h_slots[S_TESTS_SKY];
    c.st->gres_tests = c.h_slots[S_TESTS_GRES];
    c.st->sky_units = c.h_slots[S_UNITS_SKY];
    for (int i = 0; i < c.nspans; ++i) {
        float ms = 0;
        SKY_CUDA(cudaEventElapsedTime(&ms, c.ev[c.spans[i].a], c.ev[c.spans[i].a + 1]));
        *c.spans[i].dst = ms;
    }
    c.nspans = 0;
    if (c.gres_timing_pending) {
        float ms = 0;
        SKY_CUDA(cudaEventElapsedTime(&ms, c.ev[10], c.ev[11]));
        c.st->ms_gres_kernel += ms;
        c.gres_timing_pending = false;
    }
    c.st->kernel_launches = c.launches;
    if (c.trace && c.ntrace > 1) {
        for (int i = 1; i < c.ntrace; ++i) {
            float ms = 0;
            SKY_CUDA(cudaEventElapsedTime(&ms, c.tev[i - 1], c.tev[i]));
            fprintf(stderr, "[skygpu trace] %8.1f us  (host issue %8.1f us)  %s\n", ms * 1e3,
                    c.thost[i] - c.thost[i - 1], c.tlabel[i]);
        }
        for (int ch = 0; ch < c.trace_chunks; ++ch) {  // streamed input: chunk arrivals
            float at = 0;
            SKY_CUDA(cudaEventElapsedTime(&at, c.tev[0], c.xev[ch]));
            fprintf(stderr, "[skygpu trace] chunk %d on the device at %8.1f us\n", ch, at * 1e3);
        }
        c.trace_chunks = 0;
        float tot = 0;
        SKY_CUDA(cudaEventElapsedTime(&tot, c.tev[0], c.tev[c.ntrace - 1]));
        fprintf(stderr, "[skygpu trace] %8.1f us  TOTAL (%llu launches)\n", tot * 1e3,
                (unsigned long long)c.launches);
    }
    c.ntrace = 0;
}

// ---- partition.cpp:13-83 plan sizing (host) ----
constexpr long long kMaxPartitions = 1LL << 20;
long long ipow_cap(long long b, int e) {
    long long v = 1;
    for (int i = 0; i < e; ++i) {
        v *= b;
        if (v > kMaxPartitions) return kMaxPartitions + 1;
    }
    return v;
}
int closest_slices(long long target, int e) {
    int m = 2;
    while (ipow_cap(m + 1, e) <= target) ++m;
    long long lo = ipow_cap(m, e), hi = ipow_cap(m + 1, e);
    return (target - lo <= hi - target) ? m : m + 1;
}

}  // namespace

void issue_late_ids(Ctx& c) {
    if (!c.ids_host) return;
    SKY_CUDA(cudaEventRecord(c.xev[5], c.stream));
    SKY_CUDA(cudaStreamWaitEvent(c.copy, c.xev[5], 0));
    SKY_CUDA(cudaMemcpyAsync(c.ids_dev, c.ids_host, c.ids_n * sizeof(int64_t),
                             cudaMemcpyHostToDevice, c.copy));
    SKY_CUDA(cudaEventRecord(c.xev[6], c.copy));
    c.ids_ready = c.xev[6];
    c.ids_host = nullptr;
}

namespace {
__global__ void k_clear_slot(unsigned long long* slots, int i) {
    pdl_wait();
    slots[i] = 0;
}

// skyline_bnl's set (core.cpp:25-46) from the SFS engine's result K (in (sum,
// id) order): BNL keeps exactly the tuples no tuple dominates, SFS those no
// PREDECESSOR dominates.  They differ only for t in K dominated by a later
// tuple of EQUAL float64 sum — and then by one inside K (the dominance-maximal
// such tuple has no dominator of smaller or equal sum), which sits right
// behind t in K's order.  keep[j] = 0 for those.
__global__ void k_bnl_refine(const double* __restrict__ v, int d, const uint32_t* __restrict__ K,
                             uint64_t S, uint8_t* __restrict__ keep) {
    pdl_wait();
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < S;
         j += (uint64_t)gridDim.x * blockDim.x) {
        const double* t = v + (uint64_t)K[j] * d;
        double st = 0.0;
        for (int k = 0; k < d; ++k) st = __dadd_rn(st, t[k]);
        bool dominated = false;
        for (uint64_t q = j + 1; q < S && !dominated; ++q) {
            const double* w = v + (uint64_t)K[q] * d;
            double sw = 0.0;
            for (int k = 0; k < d; ++k) sw = __dadd_rn(sw, w[k]);
            if (!(sw == st)) break;  // sums ascend along K: the equal-sum run ended
            dominated = dom_f64_dyn(w, t, d);
        }
        keep[j] = !dominated;
    }
}

__global__ void k_widen(const uint32_t* __restrict__ a, uint64_t* __restrict__ b, uint64_t n) {
    pdl_wait();
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        b[i] = a[i];
}
}  // namespace

namespace {
__global__ void k_iota64(int64_t* __restrict__ a, uint64_t n) {
    pdl_wait();
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        a[i] = (int64_t)i;
}
__global__ void k_fill_i32(int32_t* __restrict__ a, uint64_t n, int32_t v) {
    pdl_wait();
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        a[i] = v;
}
__global__ void k_mark_i32(int32_t* __restrict__ a, const uint32_t* __restrict__ at, uint64_t n,
                           int32_t v) {
    pdl_wait();
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        a[at[i]] = v;
}
}  // namespace

// ---- NCCL, loaded at run time (dlopen: the process's copy when torch has
// already loaded one — same soname — else the system's libnccl.so.2)
namespace nccl {
typedef struct {
    char internal[128];
} UniqueId;
typedef void* Comm;
enum { kUint8 = 1, kInt32 = 2 };  // ncclDataType_t (nccl.h)
enum { kMax = 2 };                // ncclRedOp_t
struct Api {
    int (*get_unique_id)(UniqueId*) = nullptr;
    int (*comm_init_rank)(Comm*, int, UniqueId, int) = nullptr;
    int (*all_reduce)(const void*, void*, size_t, int, int, Comm, cudaStream_t) = nullptr;
    int (*comm_destroy)(Comm) = nullptr;
    const char* (*error_string)(int) = nullptr;
    bool ok = false;
    std::string why;
};
Api& api() {
    static Api a = [] {
        Api x;
        // the copy already in the process first (torch's, when torch was
        // imported: a second NCCL of the same soname would be bound by
        // torch's own references), then SKYGPU_NCCL_LIB, then the system's;
        // loaded RTLD_LOCAL so it never shadows another copy's symbols
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h && getenv("SKYGPU_NCCL_LIB")) h = dlopen(getenv("SKYGPU_NCCL_LIB"), RTLD_NOW | RTLD_LOCAL);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
        if (!h) {
            x.why = std::string("libnccl.so.2 not loadable: ") + dlerror();
            return x;
        }
        x.get_unique_id = (int (*)(UniqueId*))dlsym(h, "ncclGetUniqueId");
        x.comm_init_rank = (int (*)(Comm*, int, UniqueId, int))dlsym(h, "ncclCommInitRank");
        x.all_reduce = (int (*)(const void*, void*, size_t, int, int, Comm, cudaStream_t))dlsym(
            h, "ncclAllReduce");
        x.comm_destroy = (int (*)(Comm))dlsym(h, "ncclCommDestroy");
        x.error_string = (const char* (*)(int))dlsym(h, "ncclGetErrorString");
        x.ok = x.get_unique_id && x.comm_init_rank && x.all_reduce && x.comm_destroy;
        if (!x.ok) x.why = "libnccl.so.2 lacks the expected symbols";
        return x;
    }();
    return a;
}
void check(int rc, const char* what) {
    if (rc != 0)
        throw Error(SKYGPU_ERUNTIME, std::string(what) + " failed: " +
                                         (api().error_string ? api().error_string(rc) : "?"));
}
}  // namespace nccl

void shard_allreduce_max(Ctx& c, void* dev_ptr, uint64_t count, int elem_bytes) {
    if (c.shard_world <= 1 || count == 0) return;
    if (c.nccl) {  // stream-ordered, in place; no host synchronisation
        if (c.nccl_world != c.shard_world || c.nccl_rank != c.shard_rank)
            invalid("sharded pipeline: shard rank/world differ from the NCCL group's");
        nccl::check(nccl::api().all_reduce(dev_ptr, dev_ptr, count,
                                           elem_bytes == 1 ? nccl::kUint8 : nccl::kInt32,
                                           nccl::kMax, (nccl::Comm)c.nccl, c.stream),
                    "ncclAllReduce");
        return;
    }
    if (!c.coll) return;
    SKY_CUDA(cudaStreamSynchronize(c.stream));  // the reduced data is complete
    const int rc = c.coll(dev_ptr, count, elem_bytes, (void*)c.stream, c.coll_user);
    if (rc != 0)
        throw Error(SKYGPU_ERUNTIME, "sharded pipeline: the installed collective failed (" +
                                         std::to_string(rc) + ")");
}

void iota64(Ctx& c, int64_t* a, uint64_t n) {
    pdl_launch(k_iota64, grid_for(n, 256), 256, 0, c.stream, a, n);
    SKY_LAUNCH_CHECK();
    note_launch(c);
}

void widen_u32_u64(Ctx& c, const uint32_t* a, uint64_t* b, uint64_t n) {
    pdl_launch(k_widen, grid_for(n, 256), 256, 0, c.stream, a, b, n);
    SKY_LAUNCH_CHECK();
    note_launch(c);
}

void aos_to_soa(Ctx& c, const double* d_aos, uint64_t n, int d, double* d_soa) {
    if (n == 0) return;
    pdl_launch(k_aos_to_soa, grid_for(n * d, 256), 256, 0, c.stream, d_aos, n, d, d_soa);
    SKY_LAUNCH_CHECK();
    note_launch(c);
}

}  // namespace skygpu

using namespace skygpu;

// internal pipeline flag: inputs already on the device, outputs to the host
static constexpr unsigned kInputsOnDevice = 1u << 30;

extern "C" {

int skygpu_version(void) { return 10; }

int skygpu_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
    return n;
}

int skygpu_set_device(int device, char* err, size_t errlen) {
    return guarded(err, errlen, [&] { SKY_CUDA(cudaSetDevice(device)); });
}

int skygpu_set_stream(void* stream, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        int dev = 0;
        SKY_CUDA(cudaGetDevice(&dev));
        g_user_stream[dev] = static_cast<cudaStream_t>(stream);
        g_user_stream_set[dev] = stream != nullptr;
    });
}

int skygpu_release(void) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return SKYGPU_ECUDA;
    if (g_ctx[dev]) {
        cudaStreamSynchronize(g_ctx[dev]->stream);
        for (auto& b : g_ctx[dev]->buf) b.release();
        for (int i = 0; i < 4; ++i) {
            if (g_ctx[dev]->hbuf[i]) cudaFreeHost(g_ctx[dev]->hbuf[i]);
            g_ctx[dev]->hbuf[i] = nullptr;
            g_ctx[dev]->hcap[i] = 0;
        }
    }
    return SKYGPU_OK;
}

int skygpu_host_buffer(uint64_t bytes, int slot, void** out, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        if (slot < 0 || slot > 3) invalid("host_buffer: slot must be in [0, 3]");
        if (!out) invalid("host_buffer: out is NULL");
        Ctx& c = ctx();
        if (bytes > c.hcap[slot]) {
            if (c.hbuf[slot]) {
                SKY_CUDA(cudaStreamSynchronize(c.stream));  // (a copy may still read it)
                SKY_CUDA(cudaFreeHost(c.hbuf[slot]));
                c.hbuf[slot] = nullptr;
                c.hcap[slot] = 0;
            }
            const size_t want = bytes + bytes / 8 + 4096;
            SKY_CUDA(cudaHostAlloc(&c.hbuf[slot], want, cudaHostAllocPortable));
            c.hcap[slot] = want;
        }
        *out = c.hbuf[slot];
    });
}

int skygpu_make_plan(int strategy, long long target, int dims, skygpu_plan* out, char* err,
                     size_t errlen) {
    return guarded(err, errlen, [&] {
        if (dims < 1) invalid("make_plan: dims must be >= 1");
        if (target < 1 || target > kMaxPartitions)
            invalid("make_plan: target partition count must be in [1, " +
                    std::to_string(kMaxPartitions) + "]");
        skygpu_plan p{strategy, 1, 1, dims};
        switch (strategy) {
            case SKYGPU_NONE: break;
            case SKYGPU_GRID:
                p.slices = closest_slices(target, dims);
                p.partitions = ipow_cap(p.slices, dims);
                break;
            case SKYGPU_ANGULAR:
                if (dims < 2) invalid("make_plan: angular partitioning needs dims >= 2");
                p.slices = closest_slices(target, dims - 1);
                p.partitions = ipow_cap(p.slices, dims - 1);
                break;
            case SKYGPU_SLICED: p.partitions = target; break;
            default: invalid("unknown strategy");
        }
        if (p.partitions > kMaxPartitions)
            invalid("make_plan: partition count exceeds " + std::to_string(kMaxPartitions));
        *out = p;
    });
}

int skygpu_assign_partitions(const double* vals, const int64_t* ids, uint64_t n, int d,
                             const skygpu_plan* plan, int64_t* out_pid, char* err,
                             size_t errlen) {
    return guarded(err, errlen, [&] {
        if (!plan) invalid("assign_partitions: plan is required");
        if (d < 1 || d > kMaxDims) invalid("assign_partitions: dims must be in [1, 32]");
        validate_plan(plan, d);
        const skygpu_plan pl = *plan;
        if ((pl.strategy == SKYGPU_GRID || pl.strategy == SKYGPU_ANGULAR) && pl.slices < 1)
            invalid(pl.strategy == SKYGPU_GRID ? "grid_cell: slices must be >= 1"
                                               : "assign_angular: slices must be >= 1");
        if (!plan_ids_in_range(pl, d) || pl.partitions > (1LL << 30))
            invalid("assign_partitions: plan inconsistent with dims (partition ids would exceed "
                    "the plan's partition count)");
        if (n == 0) return;
        if (n >= 0xFFFFFFFFull) invalid("assign_partitions: more than 2^32-1 tuples");
        bool sorted = true;
        for (uint64_t i = 0; ids && i + 1 < n && sorted; ++i) sorted = ids[i] < ids[i + 1];
        Ctx& c = ctx();
        double* dv = c.buf[B_IN_VALS].as<double>(n * d);
        int64_t* di = c.buf[B_IN_IDS].as<int64_t>(n);
        int32_t* pid = c.buf[B_PPID].as<int32_t>(n);
        SKY_CUDA(cudaMemcpyAsync(dv, vals, n * d * sizeof(double), cudaMemcpyHostToDevice,
                                 c.stream));
        if (ids)
            SKY_CUDA(cudaMemcpyAsync(di, ids, n * sizeof(int64_t), cudaMemcpyHostToDevice,
                                     c.stream));
        if (pl.strategy == SKYGPU_ANGULAR && d < 2) {
            // to_hyperspherical throws for the first tuple that is not the origin
            for (uint64_t i = 0; i < n; ++i)
                if (vals[i] != 0.0) invalid("to_hyperspherical: needs at least 2 dimensions");
        }
        zero_slots(c);
        assign_partitions_device(c, dv, ids ? di : nullptr, sorted, n, d, pl, pid);
        std::vector<int32_t> h(n);
        SKY_CUDA(cudaMemcpyAsync(h.data(), pid, n * sizeof(int32_t), cudaMemcpyDeviceToHost,
                                 c.stream));
        read_slots(c, S_GRIDBAD, 1);
        if (pl.strategy == SKYGPU_GRID && c.h_slots[S_GRIDBAD] != ~0ULL) {
            const uint64_t flat = c.h_slots[S_GRIDBAD];
            invalid("grid_cell: value " + std::to_string(vals[flat]) + " in attribute " +
                    std::to_string(flat % d + 1) + " outside [0,1]; normalize the data first");
        }
        for (uint64_t i = 0; i < n; ++i) out_pid[i] = h[i];
    });
}

int skygpu_parallel_skyline(const double* vals, const int64_t* ids, uint64_t n, int d,
                            const skygpu_plan* plan, const double* rep_vals,
                            const int64_t* rep_ids, uint64_t n_reps, int cores,
                            uint64_t* out_pos, uint64_t* out_n, skygpu_stats* stats, char* err,
                            size_t errlen) {
    (void)rep_ids;
    return guarded(err, errlen, [&] {
        if (cores < 1) invalid("parallel_skyline: cores must be >= 1");
        if (d < 1 || d > kMaxDims) invalid("parallel_skyline: dims must be in [1, 32]");
        validate_plan(plan, d);
        skygpu_plan pl = plan ? *plan : skygpu_plan{SKYGPU_NONE, 1, 1, d};
        Ctx& c = ctx();
        begin_stats(c, stats);
        *out_n = 0;
        if (n == 0) {
            end_stats(c);
            return;
        }
        Timer all(c, 0);
        double* dv = c.buf[B_IN_VALS].as<double>(n * d);
        int64_t* di = c.buf[B_IN_IDS].as<int64_t>(n);
        double* dr = nullptr;
        SKY_CUDA(cudaMemcpyAsync(dv, vals, n * d * sizeof(double), cudaMemcpyHostToDevice,
                                 c.stream));
        SKY_CUDA(cudaMemcpyAsync(di, ids, n * sizeof(int64_t), cudaMemcpyHostToDevice, c.stream));
        if (n_reps) {
            dr = c.buf[B_REPS].as<double>(n_reps * d);
            SKY_CUDA(cudaMemcpyAsync(dr, rep_vals, n_reps * d * sizeof(double),
                                     cudaMemcpyHostToDevice, c.stream));
        }
        LocalPruneScope lps(c, false);
        SkylineOut so = skyline_device(c, dv, di, n, d, pl, dr, n_reps);
        if (so.S)
            SKY_CUDA(cudaMemcpyAsync(out_pos, so.d_pos64, so.S * sizeof(uint64_t),
                                     cudaMemcpyDeviceToHost, c.stream));
        all.stop(&c.st->ms_total);
        end_stats(c);  // final synchronisation
        *out_n = so.S;
    });
}

int skygpu_skyline_bnl(const double* vals, const int64_t* ids, uint64_t n, int d,
                       uint64_t* out_pos, uint64_t* out_n, skygpu_stats* stats, char* err,
                       size_t errlen) {
    return guarded(err, errlen, [&] {
        if (d < 1 || d > kMaxDims) invalid("skyline_bnl: dims must be in [1, 32]");
        Ctx& c = ctx();
        begin_stats(c, stats);
        *out_n = 0;
        if (n == 0) {
            end_stats(c);
            return;
        }
        Timer all(c, 0);
        double* dv = c.buf[B_IN_VALS].as<double>(n * d);
        int64_t* di = c.buf[B_IN_IDS].as<int64_t>(n);
        SKY_CUDA(cudaMemcpyAsync(dv, vals, n * d * sizeof(double), cudaMemcpyHostToDevice,
                                 c.stream));
        if (ids) {
            SKY_CUDA(cudaMemcpyAsync(di, ids, n * sizeof(int64_t), cudaMemcpyHostToDevice,
                                     c.stream));
        } else {
            pdl_launch(k_iota64, grid_for(n, 256), 256, 0, c.stream, di, n);
            SKY_LAUNCH_CHECK();
            note_launch(c);
        }
        const skygpu_plan none{SKYGPU_NONE, 1, 1, d};
        LocalPruneScope lps(c, false);
        SkylineOut so = skyline_device(c, dv, di, n, d, none, nullptr, 0);
        std::vector<uint64_t> pos(so.S);
        std::vector<uint8_t> keep(so.S);
        if (so.S) {
            uint8_t* dk = c.buf[B_PFLAGS].as<uint8_t>(so.S);
            pdl_launch(k_bnl_refine, grid_for(so.S, 256), 256, 0, c.stream, (const double*)dv, d,
                       (const uint32_t*)so.d_inpos, so.S, dk);
            SKY_LAUNCH_CHECK();
            note_launch(c);
            SKY_CUDA(cudaMemcpyAsync(pos.data(), so.d_pos64, so.S * sizeof(uint64_t),
                                     cudaMemcpyDeviceToHost, c.stream));
            SKY_CUDA(cudaMemcpyAsync(keep.data(), dk, so.S, cudaMemcpyDeviceToHost, c.stream));
        }
        all.stop(&c.st->ms_total);
        end_stats(c);  // final synchronisation
        uint64_t m = 0;
        for (uint64_t j = 0; j < so.S; ++j)
            if (keep[j]) out_pos[m++] = pos[j];
        *out_n = m;
        c.st->skyline_size = m;
    });
}

int skygpu_grid_resistance(const double* sky_vals, const int64_t* sky_ids, uint64_t s, int d,
                           const skygpu_plan* plan, uint64_t rep_count, int cores, int cap,
                           int check_skyline, int32_t* out_den, int* out_g_max,
                           skygpu_stats* stats, char* err, size_t errlen) {
    (void)rep_count;
    return guarded(err, errlen, [&] {
        if (cores < 1) invalid("grid_resistance: cores must be >= 1");
        if (d < 1 || d > kMaxDims) invalid("grid_resistance: dims must be in [1, 32]");
        validate_plan(plan, d);
        Ctx& c = ctx();
        begin_stats(c, stats);
        *out_g_max = 1;
        if (s == 0) {
            end_stats(c);
            return;
        }
        Timer all(c, 0);
        double* dv = c.buf[B_IN_VALS].as<double>(s * d);
        double* soa = c.buf[B_SKYV].as<double>(s * d);
        int64_t* di = c.buf[B_IN_IDS].as<int64_t>(s);
        int32_t* den = c.buf[B_DEN].as<int32_t>(s);
        SKY_CUDA(cudaMemcpyAsync(dv, sky_vals, s * d * sizeof(double), cudaMemcpyHostToDevice,
                                 c.stream));
        SKY_CUDA(cudaMemcpyAsync(di, sky_ids, s * sizeof(int64_t), cudaMemcpyHostToDevice,
                                 c.stream));
        zero_slots(c);
        pdl_launch(k_check_values, grid_for(s * d, 256), 256, 0, c.stream, dv, s * d, c.d_slots);
        SKY_LAUNCH_CHECK();
        note_launch(c);
        read_slots(c, S_BAD, 1);
        if (c.h_slots[S_BAD] != ~0ULL)
            invalid("grid_resistance: tuple at position " + std::to_string(c.h_slots[S_BAD] / d) +
                    " has a negative or NaN value (Relation::add contract, core.cpp:14-17)");
        aos_to_soa(c, dv, s, d, soa);
        GresOut go = gres_device(c, soa, di, s, d, cap, SKYGPU_GRES_AUTO, 0, 1,
                                 check_skyline != 0, den);
        if (plan && plan->strategy == SKYGPU_GRID && go.g_max >= 2)
            check_grid_projection(c, soa, s, d, go.g_max);
        SKY_CUDA(cudaMemcpyAsync(out_den, den, s * sizeof(int32_t), cudaMemcpyDeviceToHost,
                                 c.stream));
        all.stop(&c.st->ms_total);
        *out_g_max = go.g_max;
        end_stats(c);
    });
}

int skygpu_snap_relation(const double* vals, uint64_t count, int intervals, double* out,
                         char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        if (intervals < 1) invalid("snap_to_grid: intervals must be >= 1");
        if (count == 0) return;
        Ctx& c = ctx();
        double* dv = c.buf[B_IN_VALS].as<double>(count);
        double* dq = c.buf[B_PROJ].as<double>(count);
        SKY_CUDA(cudaMemcpyAsync(dv, vals, count * sizeof(double), cudaMemcpyHostToDevice,
                                 c.stream));
        pdl_launch(k_snap, grid_for(count, 256), 256, 0, c.stream, dv, count, intervals, dq);
        SKY_LAUNCH_CHECK();
        SKY_CUDA(cudaMemcpyAsync(out, dq, count * sizeof(double), cudaMemcpyDeviceToHost,
                                 c.stream));
        SKY_CUDA(cudaStreamSynchronize(c.stream));
    });
}

int skygpu_max_grid_intervals(const double* vals, uint64_t n, int d, int cap, int* out,
                              char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        if (d < 1) invalid("max_grid_intervals: dims must be >= 1");
        Ctx& c = ctx();
        skygpu_stats tmp;
        begin_stats(c, &tmp);
        double gap = 0, maxv = 0;
        bool has = false;
        if (n > 0) {
            double* dv = c.buf[B_IN_VALS].as<double>(n * d);
            double* soa = c.buf[B_SKYV].as<double>(n * d);
            SKY_CUDA(cudaMemcpyAsync(dv, vals, n * d * sizeof(double), cudaMemcpyHostToDevice,
                                     c.stream));
            aos_to_soa(c, dv, n, d, soa);
            has = min_positive_gap_device(c, soa, n, d, &gap, &maxv);
        }
        if (!has)
            invalid("max_grid_intervals: undefined, all tuples are identical on every attribute");
        if (cap > 0 && 1.0 / gap >= static_cast<double>(cap)) {
            *out = cap;
            return;
        }
        double bound = std::floor(1.0 / gap);
        if (bound > 2147483647.0)
            invalid("max_grid_intervals: bound overflows the integer range; set a cap");
        *out = static_cast<int>(bound);
    });
}

int skygpu_pipeline(const double* vals, const int64_t* ids, uint64_t n, int d,
                    const skygpu_plan* plan, int cap, int gres_engine, int shard_rank,
                    int shard_world, unsigned flags, uint64_t* out_pos, int32_t* out_den,
                    uint64_t* out_s, int* out_g_max, skygpu_stats* stats, char* err,
                    size_t errlen) {
    return guarded(err, errlen, [&] {
        if (d < 1 || d > kMaxDims) invalid("pipeline: dims must be in [1, 32]");
        validate_plan(plan, d);
        if (shard_world < 1 || shard_rank < 0 || shard_rank >= shard_world)
            invalid("pipeline: bad shard");
        skygpu_plan pl = plan ? *plan : skygpu_plan{SKYGPU_NONE, 1, 1, d};
        Ctx& c = ctx();
        begin_stats(c, stats);
        // kInputsOnDevice (internal): device inputs, host outputs (the CSV path)
        const bool dev_in = flags & (SKYGPU_DEVICE_PTRS | kInputsOnDevice);
        const bool dev = flags & SKYGPU_DEVICE_PTRS;
        *out_s = 0;
        *out_g_max = 1;
        if (n == 0) {
            end_stats(c);
            return;
        }
        Timer all(c, 0);
        const double* dv = vals;
        const int64_t* di = ids;
        TailFeed feed;
        // host inputs of a large relation stream in (copy stream, 4 chunks):
        // the skyline stage decides the first chunk while the rest is in
        // flight (SKYGPU_OVERLAP=0 disables)
        static const bool overlap_env = [] {
            const char* e = getenv("SKYGPU_OVERLAP");
            return !(e && e[0] == '0');
        }();
        // (worth it only when the tail's copy outlasts the head's decision,
        // ~0.5 ms: from ~48 MB of input on)
        static const uint64_t stream_min = [] {  // SKYGPU_STREAM_MIN_MB: tuning override
            const char* e = getenv("SKYGPU_STREAM_MIN_MB");
            return (uint64_t)(e ? atoll(e) : 48) << 20;
        }();
        const bool streamed = !dev_in && overlap_env && !(flags & SKYGPU_NORMALIZE) &&
                              n * (uint64_t)(d + 1) * 8 >= stream_min &&
                              d <= 8 && pl.strategy != SKYGPU_GRID && !(flags & SKYGPU_SKY_GRID) &&
                              !(flags & SKYGPU_SKY_PARTS) && !local_prune_env();
        LocalPruneScope lps(c, (flags & SKYGPU_SKY_PARTS) != 0);
        // host ids travel behind the values and are only waited for at the
        // end of the skyline (speculating they are strictly increasing, the
        // usual row-order ids; otherwise the call re-runs once they are in)
        static const bool ids_late_env = [] {
            const char* e = getenv("SKYGPU_IDS_LATE");
            return !(e && e[0] == '0');
        }();
        const bool ids_late = !dev_in && ids_late_env && n >= (1u << 16) &&
                              !(flags & SKYGPU_NORMALIZE);
        struct IdsScope {  // the ids event never outlives the call
            Ctx& c;
            ~IdsScope() {
                c.ids_ready = nullptr;
                c.ids_host = nullptr;
            }
        } ids_scope{c};
        if (!dev_in) {
            Timer h2d(c, 2);
            double* bv = c.buf[B_IN_VALS].as<double>(n * d);
            int64_t* bi = c.buf[B_IN_IDS].as<int64_t>(n);
            if (streamed) {
                if (!c.copy) {
                    SKY_CUDA(cudaStreamCreateWithFlags(&c.copy, cudaStreamNonBlocking));
                    for (auto& e : c.xev)
                        SKY_CUDA(cudaEventCreateWithFlags(
                            &e, c.trace ? cudaEventDefault : cudaEventDisableTiming));
                }
                feed.nchunks = 4;
                c.trace_chunks = feed.nchunks;
                for (int ch = 0; ch <= feed.nchunks; ++ch) feed.bound[ch] = n * ch / feed.nchunks;
                if (ids_late) pdl_launch(k_clear_slot, 1, 1, 0, c.stream, c.d_slots, S_IDSBAD);
                SKY_LAUNCH_CHECK();
                // the copies follow the stream's earlier work on these buffers
                SKY_CUDA(cudaEventRecord(c.xev[9], c.stream));
                SKY_CUDA(cudaStreamWaitEvent(c.copy, c.xev[9], 0));
                for (int ch = 0; ch < feed.nchunks; ++ch) {
                    const uint64_t lo = feed.bound[ch], cnt = feed.bound[ch + 1] - lo;
                    SKY_CUDA(cudaMemcpyAsync(bv + lo * d, vals + lo * d, cnt * d * sizeof(double),
                                             cudaMemcpyHostToDevice, c.copy));
                    if (!ids_late)
                        SKY_CUDA(cudaMemcpyAsync(bi + lo, ids + lo, cnt * sizeof(int64_t),
                                                 cudaMemcpyHostToDevice, c.copy));
                    SKY_CUDA(cudaEventRecord(c.xev[ch], c.copy));
                    feed.ready[ch] = c.xev[ch];
                }
                if (ids_late) {  // every value first; the ids when the skyline asks
                    c.ids_host = ids;  // (issue_late_ids: behind the values, or at
                    c.ids_dev = bi;    //  the rank-grid kernel's start)
                    c.ids_n = n;
                }
            } else if (ids_late) {
                // values first (the skyline starts as soon as they land), the
                // ids behind them on the copy stream, overlapping the skyline
                if (!c.copy) {
                    SKY_CUDA(cudaStreamCreateWithFlags(&c.copy, cudaStreamNonBlocking));
                    for (auto& e : c.xev)
                        SKY_CUDA(cudaEventCreateWithFlags(
                            &e, c.trace ? cudaEventDefault : cudaEventDisableTiming));
                }
                pdl_launch(k_clear_slot, 1, 1, 0, c.stream, c.d_slots, S_IDSBAD);
                SKY_LAUNCH_CHECK();
                SKY_CUDA(cudaMemcpyAsync(bv, vals, n * d * sizeof(double), cudaMemcpyHostToDevice,
                                         c.stream));
                c.ids_host = ids;  // copied when K5 starts (issue_late_ids)
                c.ids_dev = bi;
                c.ids_n = n;
            } else {
                SKY_CUDA(cudaMemcpyAsync(bv, vals, n * d * sizeof(double), cudaMemcpyHostToDevice,
                                         c.stream));
                SKY_CUDA(cudaMemcpyAsync(bi, ids, n * sizeof(int64_t), cudaMemcpyHostToDevice,
                                         c.stream));
            }
            h2d.stop(&c.st->ms_h2d);
            dv = bv;
            di = bi;
        }
        if (flags & SKYGPU_NORMALIZE) {  // run_experiment's --normalize, on the device
            double* nv = c.buf[B_NORM].as<double>(n * d);
            normalize_device(c, dv, n, d, nv);
            dv = nv;
        }
        Timer tsky(c, 4);
        // sharded call with a collective: the rank-grid skyline is split by
        // grid row and the denominators are reduced here (skygpu.h)
        struct ShardScope {
            Ctx& c;
            ShardScope(Ctx& cc, int r, int w) : c(cc) {
                const bool coll = c.coll || c.nccl;
                c.shard_rank = coll ? r : 0;
                c.shard_world = coll ? w : 1;
            }
            ~ShardScope() {
                c.shard_rank = 0;
                c.shard_world = 1;
            }
        } shard_scope(c, shard_rank, shard_world);
        SkylineOut so = skyline_device(c, dv, di, n, d, pl, nullptr, 0,
                                       flags & (SKYGPU_SKY_ROUNDS | SKYGPU_SKY_GRID),
                                       streamed ? &feed : nullptr);
        if (streamed)  // the copy stream is idle again before the call returns
            SKY_CUDA(cudaStreamWaitEvent(c.stream, c.xev[feed.nchunks - 1], 0));
        tsky.stop(&c.st->ms_skyline);
        int32_t* den = c.buf[B_DEN].as<int32_t>(so.S ? so.S : 1);
        GresOut go;
        if (!(flags & SKYGPU_SKIP_GRES)) {
            Timer tg(c, 6);
            go = gres_device(c, so.d_skyv, so.d_ids, so.S, d, cap, gres_engine, shard_rank,
                             shard_world, (flags & SKYGPU_CHECK_SKYLINE) != 0, den,
                             /*allow_spec=*/true);
            if (c.shard_world > 1) shard_allreduce_max(c, den, so.S, 4);  // the full map
            tg.stop(&c.st->ms_gres);
        }
        trace_mark(c, "gres: finalize");
        Timer d2h(c, 12);
        auto copy_den = [&] {
            if (!(flags & SKYGPU_SKIP_GRES))
                SKY_CUDA(cudaMemcpyAsync(out_den, den, so.S * sizeof(int32_t),
                                         dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                                         c.stream));
        };
        if (dev) {
            // outputs stay on the device; positions widened to u64
            if (so.S) {
                copy_den();
                widen_u32_u64(c, so.d_inpos, out_pos, so.S);
            }
        } else if (so.S) {
            // positions widened on the device, copied straight into the
            // caller's buffer (no host-side staging or conversion loop)
            // (widened by the skyline's emit kernel, SkylineOut::d_pos64)
            SKY_CUDA(cudaMemcpyAsync(out_pos, so.d_pos64, so.S * sizeof(uint64_t),
                                     cudaMemcpyDeviceToHost, c.stream));
            copy_den();
        }
        gres_spec_fetch(c);
        if (ids_late)
            SKY_CUDA(cudaMemcpyAsync(c.h_slots + S_IDSBAD, c.d_slots + S_IDSBAD,
                                     sizeof(unsigned long long), cudaMemcpyDeviceToHost, c.stream));
        fetch_test_counters(c);
        SKY_CUDA(cudaStreamSynchronize(c.stream));
        if (ids_late && c.h_slots[S_IDSBAD]) {
            c.counters_fetched = false;  // (the redo adds tests)
            // the ids are not strictly increasing: (sum, id) ties may order
            // differently from positions — the whole call again, ids resident
            trace_mark(c, "ids not in position order: re-run");
            c.ids_ready = nullptr;
            c.gres_spec = false;
            so = skyline_device(c, dv, di, n, d, pl, nullptr, 0,
                                flags & (SKYGPU_SKY_ROUNDS | SKYGPU_SKY_GRID), nullptr);
            den = c.buf[B_DEN].as<int32_t>(so.S ? so.S : 1);
            if (!(flags & SKYGPU_SKIP_GRES)) {
                go = gres_device(c, so.d_skyv, so.d_ids, so.S, d, cap, gres_engine, shard_rank,
                                 shard_world, (flags & SKYGPU_CHECK_SKYLINE) != 0, den);
                if (c.shard_world > 1) shard_allreduce_max(c, den, so.S, 4);
            }
            if (so.S) {
                SKY_CUDA(cudaMemcpyAsync(out_pos, so.d_pos64, so.S * sizeof(uint64_t),
                                         cudaMemcpyDeviceToHost, c.stream));
                copy_den();
            }
            SKY_CUDA(cudaStreamSynchronize(c.stream));
        }
        if (gres_spec_failed(c)) {  // the speculative gres launch did not apply: redo
            c.counters_fetched = false;  // (the redo adds tests)
            trace_mark(c, "gres: speculation missed, exact path");
            go = gres_device(c, so.d_skyv, so.d_ids, so.S, d, cap, gres_engine, shard_rank,
                             shard_world, false, den);
            copy_den();
            SKY_CUDA(cudaStreamSynchronize(c.stream));
        }
        d2h.stop(&c.st->ms_d2h);
        all.stop(&c.st->ms_total);
        *out_s = so.S;
        *out_g_max = go.g_max;
        end_stats(c);
    });
}

// the CSV bytes parsed on the device (harness.cpp:93-134); throws the
// reference's runtime_error texts; returns the device values (rows x dims)
static double* csv_to_device(Ctx& c, const char* bytes, uint64_t len, const std::string& nm,
                             uint64_t* rows_out, int* dims_out) {
    // header (harness.cpp:94-100): the first getline; its width fixes dims
    if (len == 0) throw Error(SKYGPU_ERUNTIME, nm + ": empty file, expected a header line");
    uint64_t h = 0;
    int commas = 0;
    bool content = false;
    for (; h < len && bytes[h] != '\n'; ++h) {
        commas += bytes[h] == ',';
        content |= bytes[h] != ',' && bytes[h] != '\r';
    }
    if (commas == 0 && !content) throw Error(SKYGPU_ERUNTIME, nm + ": header line has no columns");
    const int dims = commas + 1;
    *dims_out = dims;
    char* db = c.buf[B_CSV].as<char>(len);
    SKY_CUDA(cudaMemcpyAsync(db, bytes, len, cudaMemcpyHostToDevice, c.stream));
    const uint64_t cap = (len + 1) / 2 + 1;
    double* dv = c.buf[B_CSVVAL].as<double>(cap);
    uint64_t rows = 0, eline = 0;
    int ecol = 0, ekind = 0, internal = 0;
    const int rc = csv_parse_device(c, db, len, dims, &rows, dv, cap, &eline, &ecol, &ekind,
                                    &internal);
    *rows_out = rows;
    if (internal) throw Error(SKYGPU_ERUNTIME, nm + ": a field exceeds the device parser's limits");
    if (rc == 2) {
        // the reference's message, from the offending line's bytes
        uint64_t s = 0, line = 1;
        while (line < eline && s < len) {
            if (bytes[s] == '\n') ++line;
            ++s;
        }
        uint64_t e = s;
        while (e < len && bytes[e] != '\n') ++e;
        const std::string where = nm + ": line " + std::to_string(eline);
        if (ekind == 1) {
            int k = 1;
            for (uint64_t i = s; i < e; ++i) k += bytes[i] == ',';
            throw Error(SKYGPU_ERUNTIME, where + ": expected " + std::to_string(dims) +
                                             " fields, got " + std::to_string(k));
        }
        std::string field;
        int col = 1;
        for (uint64_t i = s; i < e; ++i) {
            if (bytes[i] == ',') {
                if (col == ecol) break;
                ++col;
                field.clear();
            } else if (bytes[i] != '\r') {
                field += bytes[i];
            }
        }
        const std::string at = where + ", column " + std::to_string(ecol);
        if (ekind == 2) throw Error(SKYGPU_ERUNTIME, at + ": not a number: '" + field + "'");
        throw Error(SKYGPU_ERUNTIME, at + ": negative value " + field);
    }
    return dv;
}

int skygpu_read_csv(const char* bytes, uint64_t len, const char* name, double* out_vals,
                    uint64_t out_cap, uint64_t* out_rows, int* out_dims, char* err,
                    size_t errlen) {
    return guarded(err, errlen, [&] {
        *out_rows = 0;
        *out_dims = 0;
        Ctx& c = ctx();
        begin_stats(c, nullptr);
        uint64_t rows = 0;
        int dims = 0;
        const double* dv = csv_to_device(c, bytes, len, name ? name : "", &rows, &dims);
        *out_rows = rows;
        *out_dims = dims;
        if (rows * (uint64_t)dims > out_cap)
            invalid("read_csv: output buffer holds " + std::to_string(out_cap) +
                    " values, need " + std::to_string(rows * (uint64_t)dims));
        if (rows)
            SKY_CUDA(cudaMemcpyAsync(out_vals, dv, rows * dims * sizeof(double),
                                     cudaMemcpyDeviceToHost, c.stream));
        end_stats(c);
    });
}

int skygpu_pipeline_csv(const char* bytes, uint64_t len, const char* name, int strategy,
                        long long target_partitions, int cap, int gres_engine, unsigned flags,
                        uint64_t* out_pos, int32_t* out_den, uint64_t out_cap, uint64_t* out_s,
                        int* out_g_max, uint64_t* out_rows, int* out_dims, skygpu_stats* stats,
                        char* err, size_t errlen) {
    uint64_t rows = 0;
    int dims = 0;
    double* dv = nullptr;
    int64_t* di = nullptr;
    skygpu_plan plan{};
    const int rc = guarded(err, errlen, [&] {
        *out_s = 0;
        *out_g_max = 1;
        Ctx& c = ctx();
        begin_stats(c, nullptr);
        dv = csv_to_device(c, bytes, len, name ? name : "", &rows, &dims);
        *out_rows = rows;
        *out_dims = dims;
        if (rows > out_cap)
            invalid("pipeline_csv: output buffers hold " + std::to_string(out_cap) +
                    " tuples, need " + std::to_string(rows));
        di = c.buf[B_IN_IDS].as<int64_t>(rows ? rows : 1);  // ids = row order
        if (rows) iota64(c, di, rows);
        char perr[512];
        if (skygpu_make_plan(strategy, target_partitions, dims, &plan, perr, sizeof perr) !=
            SKYGPU_OK)
            invalid(perr);
        end_stats(c);
    });
    if (rc != SKYGPU_OK) return rc;
    // the rest of run_experiment on the device-resident relation; results to
    // the caller's host buffers
    return skygpu_pipeline(dv, di, rows, dims, &plan, cap, gres_engine, 0, 1,
                           (flags & ~SKYGPU_DEVICE_PTRS) | kInputsOnDevice, out_pos, out_den,
                           out_s, out_g_max, stats, err, errlen);
}

int skygpu_normalize(const double* vals, uint64_t n, int d, double* out, char* err,
                     size_t errlen) {
    return guarded(err, errlen, [&] {
        if (d < 1 || d > kMaxDims) invalid("normalize: dims must be in [1, 32]");
        if (n == 0) return;
        Ctx& c = ctx();
        begin_stats(c, nullptr);
        double* dv = c.buf[B_IN_VALS].as<double>(n * d);
        double* dout = c.buf[B_PROJ].as<double>(n * d);
        SKY_CUDA(cudaMemcpyAsync(dv, vals, n * d * sizeof(double), cudaMemcpyHostToDevice,
                                 c.stream));
        normalize_device(c, dv, n, d, dout);
        SKY_CUDA(cudaMemcpyAsync(out, dout, n * d * sizeof(double), cudaMemcpyDeviceToHost,
                                 c.stream));
        end_stats(c);
    });
}

int skygpu_select_representatives(const double* vals, const int64_t* ids, uint64_t n, int d,
                                  uint64_t k, uint64_t* out_pos, uint64_t* out_n,
                                  uint64_t* tests, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        if (d < 1 || d > kMaxDims) invalid("select_representatives: dims must be in [1, 32]");
        *out_n = 0;
        *tests = 0;
        if (n == 0 || k == 0) return;
        if (n >= 0xFFFFFFFFull) invalid("select_representatives: more than 2^32-1 tuples");
        Ctx& c = ctx();
        begin_stats(c, nullptr);
        double* dv = c.buf[B_IN_VALS].as<double>(n * d);
        int64_t* di = c.buf[B_IN_IDS].as<int64_t>(n);
        SKY_CUDA(cudaMemcpyAsync(dv, vals, n * d * sizeof(double), cudaMemcpyHostToDevice,
                                 c.stream));
        SKY_CUDA(cudaMemcpyAsync(di, ids, n * sizeof(int64_t), cudaMemcpyHostToDevice, c.stream));
        const uint64_t kk = k < n ? k : n;
        uint32_t* picks = c.buf[B_ACC8].as<uint32_t>(kk);
        auto* t = c.buf[B_ACC9].as<unsigned long long>(1);
        SKY_CUDA(cudaMemsetAsync(t, 0, sizeof(unsigned long long), c.stream));
        const uint64_t m = select_representatives_device(c, dv, di, n, d, kk, picks, t);
        std::vector<uint32_t> h(m);
        unsigned long long ht = 0;
        if (m)
            SKY_CUDA(cudaMemcpyAsync(h.data(), picks, m * sizeof(uint32_t), cudaMemcpyDeviceToHost,
                                     c.stream));
        SKY_CUDA(cudaMemcpyAsync(&ht, t, sizeof(ht), cudaMemcpyDeviceToHost, c.stream));
        SKY_CUDA(cudaStreamSynchronize(c.stream));
        for (uint64_t i = 0; i < m; ++i) out_pos[i] = h[i];
        *out_n = m;
        *tests = ht;
        end_stats(c);
    });
}

int skygpu_nccl_unique_id(void* out_id128, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        if (!out_id128) invalid("nccl_unique_id: out is NULL");
        if (!nccl::api().ok) throw Error(SKYGPU_ERUNTIME, nccl::api().why);
        nccl::UniqueId id;
        nccl::check(nccl::api().get_unique_id(&id), "ncclGetUniqueId");
        memcpy(out_id128, &id, sizeof(id));
    });
}

int skygpu_nccl_init(const void* id128, int nranks, int rank, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        if (!id128) invalid("nccl_init: id is NULL");
        if (nranks < 1 || rank < 0 || rank >= nranks) invalid("nccl_init: bad rank / nranks");
        if (!nccl::api().ok) throw Error(SKYGPU_ERUNTIME, nccl::api().why);
        Ctx& c = ctx();
        if (c.nccl) {
            nccl::api().comm_destroy((nccl::Comm)c.nccl);
            c.nccl = nullptr;
        }
        nccl::UniqueId id;
        memcpy(&id, id128, sizeof(id));
        nccl::Comm comm = nullptr;
        nccl::check(nccl::api().comm_init_rank(&comm, nranks, id, rank), "ncclCommInitRank");
        c.nccl = comm;
        c.nccl_rank = rank;
        c.nccl_world = nranks;
    });
}

int skygpu_nccl_release(void) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return SKYGPU_ECUDA;
    if (g_ctx[dev] && g_ctx[dev]->nccl) {
        cudaStreamSynchronize(g_ctx[dev]->stream);
        nccl::api().comm_destroy((nccl::Comm)g_ctx[dev]->nccl);
        g_ctx[dev]->nccl = nullptr;
        g_ctx[dev]->nccl_rank = 0;
        g_ctx[dev]->nccl_world = 1;
    }
    return SKYGPU_OK;
}

int skygpu_cells_step_plan(const double* col_max, int d, int g_max, uint64_t s, int rank,
                           int world, int* out_steps, int* out_n, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        if (d < 1 || d > kMaxDims) invalid("cells_step_plan: dims must be in [1, 32]");
        if (world < 1 || rank < 0 || rank >= world) invalid("cells_step_plan: bad rank / world");
        const std::vector<double> amax(col_max, col_max + d);
        const std::vector<int> st = cells_step_plan(amax, d, g_max, s, rank, world);
        for (size_t i = 0; i < st.size(); ++i) out_steps[i] = st[i];
        *out_n = (int)st.size();
    });
}

int skygpu_set_collective(skygpu_allreduce_max_fn fn, void* user, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        Ctx& c = ctx();
        c.coll = fn;
        c.coll_user = user;
    });
}

int skygpu_sfs_accounting(const double* vals, const int64_t* ids, uint64_t n, int d,
                          const int64_t* pid, long long p, const double* rep_vals,
                          uint64_t n_reps, uint64_t* per_part, uint64_t* final_tests,
                          uint64_t* into_final, uint64_t* out_pos, uint64_t* out_n, char* err,
                          size_t errlen) {
    return guarded(err, errlen, [&] {
        if (d < 1 || d > kMaxDims) invalid("sfs_accounting: dims must be in [1, 32]");
        if (p < 1 || p > (1LL << 20)) invalid("sfs_accounting: partitions must be in [1, 2^20]");
        if (n >= 0xFFFFFFFFull) invalid("sfs_accounting: more than 2^32-1 tuples");
        Ctx& c = ctx();
        begin_stats(c, nullptr);
        for (long long k = 0; k < p; ++k) per_part[k] = 0;
        *final_tests = 0;
        *into_final = 0;
        *out_n = 0;
        if (n == 0) {
            end_stats(c);
            return;
        }
        std::vector<int32_t> gid(n);
        for (uint64_t i = 0; i < n; ++i) {
            if (pid[i] >= p) invalid("sfs_accounting: partition id out of range");
            gid[i] = pid[i] < 0 ? -1 : (int32_t)pid[i];
        }
        double* dv = c.buf[B_IN_VALS].as<double>(n * d);
        int64_t* di = c.buf[B_IN_IDS].as<int64_t>(n);
        int32_t* dg = c.buf[B_ACC12].as<int32_t>(n);
        int32_t* dg2 = c.buf[B_ACC13].as<int32_t>(n);
        uint32_t* kept1 = c.buf[B_ACC14].as<uint32_t>(n);
        uint32_t* kept2 = c.buf[B_ACC15].as<uint32_t>(n);
        auto* cnt = c.buf[B_ACC16].as<unsigned long long>((uint64_t)p + 1);
        double* dr = n_reps ? c.buf[B_REPS].as<double>(n_reps * d) : nullptr;
        SKY_CUDA(cudaMemcpyAsync(dv, vals, n * d * sizeof(double), cudaMemcpyHostToDevice, c.stream));
        SKY_CUDA(cudaMemcpyAsync(di, ids, n * sizeof(int64_t), cudaMemcpyHostToDevice, c.stream));
        SKY_CUDA(cudaMemcpyAsync(dg, gid.data(), n * sizeof(int32_t), cudaMemcpyHostToDevice,
                                 c.stream));
        if (n_reps)
            SKY_CUDA(cudaMemcpyAsync(dr, rep_vals, n_reps * d * sizeof(double),
                                     cudaMemcpyHostToDevice, c.stream));
        SKY_CUDA(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long) * ((uint64_t)p + 1), c.stream));
        // phase 1: representative filter + local SFS per partition
        const uint64_t nk = sfs_accounting_device(c, dv, di, n, d, dg, (uint32_t)p, dr,
                                                  (uint32_t)n_reps, cnt, kept1);
        std::vector<unsigned long long> h(p + 1);
        SKY_CUDA(cudaMemcpyAsync(h.data(), cnt, sizeof(unsigned long long) * p,
                                 cudaMemcpyDeviceToHost, c.stream));
        // phase 2: one SFS over the union of the local skylines
        pdl_launch(k_fill_i32, grid_for(n, 256), 256, 0, c.stream, dg2, n, -1);
        if (nk) pdl_launch(k_mark_i32, grid_for(nk, 256), 256, 0, c.stream, dg2, kept1, nk, 0);
        SKY_LAUNCH_CHECK();
        note_launch(c, 2);
        SKY_CUDA(cudaMemsetAsync(cnt + p, 0, sizeof(unsigned long long), c.stream));
        const uint64_t nf = sfs_accounting_device(c, dv, di, n, d, dg2, 1, nullptr, 0, cnt + p,
                                                  kept2);
        SKY_CUDA(cudaMemcpyAsync(h.data() + p, cnt + p, sizeof(unsigned long long),
                                 cudaMemcpyDeviceToHost, c.stream));
        std::vector<uint32_t> pos(nf);
        if (nf)
            SKY_CUDA(cudaMemcpyAsync(pos.data(), kept2, nf * sizeof(uint32_t),
                                     cudaMemcpyDeviceToHost, c.stream));
        SKY_CUDA(cudaStreamSynchronize(c.stream));
        for (long long k = 0; k < p; ++k) per_part[k] = h[k];
        *final_tests = h[p];
        *into_final = nk;
        for (uint64_t k = 0; k < nf; ++k) out_pos[k] = pos[k];
        *out_n = nf;
        end_stats(c);
    });
}

}  // extern "C"

