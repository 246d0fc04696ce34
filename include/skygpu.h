/*
 * skygpu.h — C-ABI of the B200-native grid-resistance engine (libskygpu.so).
 *
 * The reference (arXiv 2412.02274 `skypar`, /root/reference/proj) has no FFI:
 * its hot path is a set of C++ free functions in namespace skypar.  Each entry
 * point below is the flat, exception-free form of one of them; the C++ drop-in
 * adapter (paper_2412_02274_b200/adapter/skypar_gpu.cpp) re-wraps them into the
 * exact reference signatures and re-throws the same exception type and text.
 *
 *   skygpu_parallel_skyline    <- skypar::parallel_skyline   include/skypar/parallel.hpp:46-47
 *   skygpu_grid_resistance     <- skypar::grid_resistance    include/skypar/gres.hpp:73-75
 *   skygpu_skyline_bnl         <- skypar::skyline_bnl        include/skypar/core.hpp:78
 *   skygpu_snap_relation       <- skypar::snap_relation      include/skypar/gres.hpp:28
 *                                 (and snap_to_grid, gres.hpp:26 = a 1-tuple relation)
 *   skygpu_max_grid_intervals  <- skypar::max_grid_intervals include/skypar/gres.hpp:35
 *   skygpu_make_plan           <- skypar::make_plan          include/skypar/partition.hpp:43
 *   skygpu_assign_partitions   <- skypar::assign_partitions  include/skypar/partition.hpp:90
 *                                 (partition.cpp:183-213)
 *   skygpu_pipeline            <- the composition run_experiment performs
 *                                 (proj/src/harness.cpp:208 then :229-231)
 *   skygpu_sfs_accounting      <- the DominanceCounter totals inside
 *                                 parallel_skyline (parallel.cpp:59-93)
 *   skygpu_read_csv            <- skypar::read_dataset_csv     include/skypar/harness.hpp
 *   skygpu_pipeline_csv        <- run_experiment with --dataset (harness.cpp:191-231)
 *   skygpu_normalize           <- skypar::normalize            include/skypar/harness.hpp
 *   skygpu_select_representatives <- skypar::select_representatives partition.hpp
 *   skygpu_set_collective      <- (no reference counterpart: the reference is
 *                                 one process; this installs the multi-GPU
 *                                 exchange)
 *
 * Conventions
 *  - Values are float64, row-major n x d (tuple i = vals[i*d .. i*d+d-1]),
 *    smaller is better, non-negative (Relation::add, core.cpp:8-19); NaN is
 *    rejected.  Ids are int64 and must be unique.
 *  - Buffers are caller-owned.  Unless a function says otherwise pointers are
 *    HOST pointers (pinned memory makes the copies faster); skygpu_pipeline
 *    also accepts device pointers (flag SKYGPU_DEVICE_PTRS).
 *  - Every function returns a status; on failure a NUL-terminated message is
 *    written into err[0..errlen) (err may be NULL).  No exception crosses the ABI.
 *  - Calls are not re-entrant per device; one host thread drives a device.
 *  - There is NO CPU fallback: without a usable sm_100 device every compute
 *    entry point fails with SKYGPU_ECUDA.
 */
#ifndef SKYGPU_H
#define SKYGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
#define SKYGPU_OK 0
#define SKYGPU_EINVAL 1   /* the reference throws std::invalid_argument */
#define SKYGPU_ERUNTIME 2 /* the reference throws std::runtime_error */
#define SKYGPU_ECUDA 3    /* CUDA error or no usable device */
#define SKYGPU_ENOMEM 4   /* device allocation failed */

/* strategies, numbered as skypar::Strategy (partition.hpp:21) */
#define SKYGPU_NONE 0
#define SKYGPU_GRID 1
#define SKYGPU_ANGULAR 2
#define SKYGPU_SLICED 3

/* gres engines */
#define SKYGPU_GRES_AUTO 0  /* the small-grid cell kernel when it applies (d <= 4, codes <= 31),
                               else pairs unless the per-step cell engine is far cheaper */
#define SKYGPU_GRES_PAIRS 1 /* (tuple, comparator, step) dominance tests, early exit */
#define SKYGPU_GRES_CELLS 2 /* occupancy prefix-OR over the code grid: every step in one
                               shared-memory launch for small grids, per step in HBM otherwise
                               (stats: gres_cells = 0 for the former) */

/* skygpu_pipeline flags */
#define SKYGPU_DEVICE_PTRS 1u   /* vals/ids/outputs are device pointers */
#define SKYGPU_CHECK_SKYLINE 2u /* O(S^2) "input is a skyline" check (gres.cpp:70-80, !NDEBUG) */
#define SKYGPU_SKIP_GRES 4u     /* skyline only (harness mode "skyline") */
#define SKYGPU_SKY_ROUNDS 8u    /* force the prefix-round skyline engine */
#define SKYGPU_SKY_GRID 16u     /* force the one-pass rank-grid skyline engine (d <= 8) */
#define SKYGPU_NORMALIZE 32u    /* min-max normalise on the device first (harness.cpp:161-177) */
#define SKYGPU_SKY_PARTS 64u    /* the plan's partitions as local-skyline pruning before the
                                   merge (parallel.cpp:59-73 recast; partition.cu): the tuples
                                   dominated inside their own partition are dropped first */

/* mirrors skypar::PartitionPlan (partition.hpp:27-32) */
typedef struct skygpu_plan {
    int strategy;
    int slices;
    long long partitions;
    int dims;
} skygpu_plan;

/* counters and device-event timings of one call */
typedef struct skygpu_stats {
    uint64_t tuples_in;            /* n */
    uint64_t tuples_into_parallel; /* after grid-cell pruning / rep filtering */
    uint64_t tuples_into_final;    /* candidates entering the merge */
    uint64_t skyline_size;         /* S */
    uint64_t skyline_tests;        /* dominance tests executed by the skyline kernels */
    uint64_t gres_tests;           /* (candidate, comparator, g) code tests executed */
    uint64_t gres_cells;           /* per-step cell engine: algorithmic bytes (3 grid sweeps + 2 value
                                      reads per step); 0 for the shared-memory small-grid kernel */
    int g_max;                     /* ResistanceMetrics::g_max (gres.hpp:46) */
    int gres_steps;                /* interval counts scanned (g_max-1 or fewer) */
    int gres_engine;               /* engine actually used */
    int code_bits;                 /* 8 = packed u8 codes, 64 = float64 projections */
    int sfs_rounds;                /* block-SFS rounds */
    int sky_engine;                /* skyline engine used: 8 = prefix rounds, 16 = rank grid */
    double ms_total;               /* device time of the whole call (events) */
    double ms_h2d, ms_skyline, ms_gres, ms_d2h;
    double ms_gres_kernel;         /* summed time of the dominant gres kernel launches */
    double ms_sky_kernel;          /* summed time of the dominant skyline kernel launches */
    uint64_t gres_kernel_launches;
    uint64_t sky_kernel_launches;
    uint64_t kernel_launches;      /* all of libskygpu's kernel launches in the call */
    uint64_t sky_units;            /* rank-grid decide kernel: (comparator, 128-candidate item)
                                      bitset tests — the unit of its shared-memory roofline */
} skygpu_stats;

/* library / device */
int skygpu_version(void);
int skygpu_device_count(void);
int skygpu_set_device(int device, char* err, size_t errlen);
/* bind subsequent calls on the current device to a caller stream (NULL = the
 * library's own non-blocking stream) */
int skygpu_set_stream(void* cuda_stream, char* err, size_t errlen);
/* release cached device buffers of the current device */
int skygpu_release(void);
/* a page-locked host staging buffer of at least `bytes`, owned by the
 * current device's context (grow-only; `slot` 0..3 are independent buffers,
 * valid until the next call with the same slot and a larger size or
 * skygpu_release).  A caller that flattens its relation into it gets DMA-rate
 * host->device copies (the C++ drop-in's Relation flattening: the reference
 * API has no device pointers, parallel.hpp:46-47). */
int skygpu_host_buffer(uint64_t bytes, int slot, void** out, char* err, size_t errlen);

/* partition.hpp:43 make_plan */
int skygpu_make_plan(int strategy, long long target_partitions, int dims, skygpu_plan* out,
                     char* err, size_t errlen);

/* partition.hpp:90 assign_partitions (partition.cpp:183-213) on the device:
 * out_pid[i] = the partition of tuple i under `plan` — grid cells
 * (grid_cell + cell_partition_id, :85-109), hyperspherical slices
 * (assign_angular, :139-174), or equal-count slices of the (attribute 0, id)
 * order (assign_sliced, :176-181); 0 for SKYGPU_NONE.  Grid and sliced ids
 * are the reference's bit for bit; angular ids use the device atan2 and may
 * differ from glibc's only where an angle lies within an ulp of a slice
 * boundary.  Errors: the reference's grid_cell text for a Grid value outside
 * [0,1]; EINVAL for a plan whose ids would exceed its partition count.
 * ids may be NULL (position order).  Host pointers. */
int skygpu_assign_partitions(const double* vals, const int64_t* ids, uint64_t n, int d,
                             const skygpu_plan* plan, int64_t* out_pid, char* err,
                             size_t errlen);

/* parallel.hpp:46-47 parallel_skyline.
 * out_pos[0..*out_n) receives the INPUT POSITIONS of the skyline tuples in the
 * reference's output order ((sum, id) ascending); out_pos must hold n entries.
 * rep_vals/rep_ids: the RepresentativeSet tuples (may be NULL when n_reps = 0). */
int skygpu_parallel_skyline(const double* vals, const int64_t* ids, uint64_t n, int d,
                            const skygpu_plan* plan, const double* rep_vals,
                            const int64_t* rep_ids, uint64_t n_reps, int cores,
                            uint64_t* out_pos, uint64_t* out_n, skygpu_stats* stats, char* err,
                            size_t errlen);

/* core.hpp:78 skyline_bnl (core.cpp:25-46): the tuples of (vals, ids) that no
 * tuple dominates — the brute-force skyline's set (it differs from
 * parallel_skyline's only where a tuple is dominated by one of EQUAL float64
 * sum and larger id).  out_pos[0..*out_n) = their
 * input positions in (sum, id) order (BNL's own window order is an artefact of
 * its sequential swap-remove; the reference's callers compare sets,
 * test_util.hpp:22-36).  out_pos sized n; ids may be NULL (positions).
 * Host pointers. */
int skygpu_skyline_bnl(const double* vals, const int64_t* ids, uint64_t n, int d,
                       uint64_t* out_pos, uint64_t* out_n, skygpu_stats* stats, char* err,
                       size_t errlen);

/* gres.hpp:73-75 grid_resistance over a skyline of s tuples.
 * out_den[i] = resistance denominator of input tuple i (1 or g in [2, g_max]);
 * cap <= 0 means no cap (std::nullopt).  check_skyline != 0 runs the O(S^2)
 * precondition check of gres.cpp:70-80. */
int skygpu_grid_resistance(const double* sky_vals, const int64_t* sky_ids, uint64_t s, int d,
                           const skygpu_plan* plan, uint64_t rep_count, int cores, int cap,
                           int check_skyline, int32_t* out_den, int* out_g_max,
                           skygpu_stats* stats, char* err, size_t errlen);

/* gres.hpp:28 snap_relation on `count` values: out = floor(v*g)/g */
int skygpu_snap_relation(const double* vals, uint64_t count, int intervals, double* out,
                         char* err, size_t errlen);

/* gres.hpp:35 max_grid_intervals; cap <= 0 means no cap */
int skygpu_max_grid_intervals(const double* vals, uint64_t n, int d, int cap, int* out,
                              char* err, size_t errlen);

/* The whole hot path in one call: skyline of (vals, ids), then the
 * grid-resistance scan of that skyline (harness.cpp:208, :229-231).
 * Outputs: out_pos[0..*out_s) skyline input positions in (sum, id) order and
 * out_den[k] the denominator of skyline tuple out_pos[k]; both sized n.
 * shard_world > 1 computes denominators only for this shard's skyline tuples
 * (interleaved chunks) and writes 0 for the others,
 * so a max-reduction over ranks yields the full map. */
int skygpu_pipeline(const double* vals, const int64_t* ids, uint64_t n, int d,
                    const skygpu_plan* plan, int cap, int gres_engine, int shard_rank,
                    int shard_world, unsigned flags, uint64_t* out_pos, int32_t* out_den,
                    uint64_t* out_s, int* out_g_max, skygpu_stats* stats, char* err,
                    size_t errlen);

/* The exchange step of sharded pipeline calls (shard_world > 1): an
 * element-wise MAX all-reduce, across the shard group, of `count` elements of
 * `elem_bytes` bytes (1 = uint8, 4 = int32) at the DEVICE pointer dev_ptr;
 * work queued on `cuda_stream` before the call must be complete in the
 * reduction, and the result must be in place when the function returns.
 * Returns 0 on success.  With a collective installed, skygpu_pipeline shards
 * the rank-grid skyline engine by grid row (keep flags MAX-reduced) and
 * returns the FULL denominator map on every rank (den MAX-reduced); without
 * one, only the gres stage is sharded and the caller reduces the map. */
typedef int (*skygpu_allreduce_max_fn)(void* dev_ptr, uint64_t count, int elem_bytes,
                                       void* cuda_stream, void* user);
int skygpu_set_collective(skygpu_allreduce_max_fn fn, void* user, char* err, size_t errlen);

/* The library's OWN NCCL path for the same exchange steps (preferred over
 * skygpu_set_collective): one process per GPU; rank 0 makes a 128-byte
 * unique id, the caller ships it to every rank (any out-of-band channel —
 * torch.distributed's broadcast in dist.py), and every rank joins the
 * communicator on the current device.  Sharded pipeline calls then queue
 * ncclAllReduce(ncclMax) in place on the library's stream — no host
 * synchronisation around the exchange.  libnccl.so.2 is loaded at run time
 * (the copy already in the process, e.g. torch's, when there is one).
 * The group's world size and rank must match the shard_world / shard_rank
 * of the calls. */
int skygpu_nccl_unique_id(void* out_id128, char* err, size_t errlen);
int skygpu_nccl_init(const void* id128, int nranks, int rank, char* err, size_t errlen);
int skygpu_nccl_release(void);

/* The step split of the cell-occupancy resistance engine (host only, no
 * device): the steps of g_max .. 2 that shard `rank` of `world` runs, in
 * descending order — longest-processing-time over the per-step cost model of
 * cells.cu (grid rows from the per-attribute maxima col_max[d] of the
 * skyline, plus the S-tuple mark and query).  out_steps holds g_max - 1. */
int skygpu_cells_step_plan(const double* col_max, int d, int g_max, uint64_t s, int rank,
                           int world, int* out_steps, int* out_n, char* err, size_t errlen);

/* Exact reference accounting of parallel_skyline — "metrics-parity" mode,
 * not the hot path.  Returns the DominanceCounter
 * totals the reference's CPU algorithm executes (core.hpp:46-67): per
 * partition the representative filter (partition.cpp:287-302) + the local
 * SFS (core.cpp:48-73), and the merge-phase SFS (parallel.cpp:83-86).
 * pid[i] = partition of tuple i in [0, p), or -1 for a tuple dropped before
 * phase 1 (Grid dominated cells, parallel.cpp:32-42); the caller assigns
 * partitions with the reference's own assign_partitions (partition.cpp:183).
 * rep_vals: the representative tuples (n_reps x d, may be NULL when 0).
 * Outputs: per_part[0..p) tests per partition, *final_tests merge tests,
 * *into_final = tuples entering the merge, out_pos[0..*out_n) = skyline
 * input positions in (sum, id) order (out_pos sized n). */
int skygpu_sfs_accounting(const double* vals, const int64_t* ids, uint64_t n, int d,
                          const int64_t* pid, long long p, const double* rep_vals,
                          uint64_t n_reps, uint64_t* per_part, uint64_t* final_tests,
                          uint64_t* into_final, uint64_t* out_pos, uint64_t* out_n, char* err,
                          size_t errlen);

/* harness.cpp:161-177 normalize on the device: per attribute (v - min) /
 * (max - min), 0 for a constant attribute; bit-identical to the reference.
 * Host pointers; out may alias vals. */
int skygpu_normalize(const double* vals, uint64_t n, int d, double* out, char* err,
                     size_t errlen);

/* partition.cpp:249-271 select_representatives(r, k, sum_score, c) on the
 * device: out_pos[0..*out_n) = input positions of the kept picks in (sum, id)
 * order (out_pos sized min(k, n)); *tests = the pruning's DominanceCounter
 * total.  Host pointers. */
int skygpu_select_representatives(const double* vals, const int64_t* ids, uint64_t n, int d,
                                  uint64_t k, uint64_t* out_pos, uint64_t* out_n,
                                  uint64_t* tests, char* err, size_t errlen);

/* harness.cpp:93-134 read_dataset_csv on the device: `bytes` = the whole file
 * (len bytes), `name` = the path used in error texts.  The header line fixes
 * the width; empty lines are skipped; ids are row order.  On success
 * out_vals[0 .. rows*dims) holds the relation (row-major) — out_vals must hold
 * `out_cap` doubles ((len + 1) / 2 always suffices) — and *out_rows/*out_dims
 * are set.  Format errors return SKYGPU_ERUNTIME with the reference's exact
 * text (runtime_error); a too-small buffer returns SKYGPU_EINVAL with
 * *out_rows/*out_dims set. */
int skygpu_read_csv(const char* bytes, uint64_t len, const char* name, double* out_vals,
                    uint64_t out_cap, uint64_t* out_rows, int* out_dims, char* err,
                    size_t errlen);

/* run_experiment with --dataset (harness.cpp:191-208, :229-231) on the device:
 * the CSV parsed by skygpu_read_csv's parser without leaving the GPU, the
 * plan sized for the file's width (make_plan(strategy, target, dims)), then
 * the skyline + grid-resistance pipeline (flags as skygpu_pipeline, incl.
 * SKYGPU_NORMALIZE for --normalize; outputs are HOST buffers of out_cap
 * tuples).  *out_rows / *out_dims give the relation's shape. */
int skygpu_pipeline_csv(const char* bytes, uint64_t len, const char* name, int strategy,
                        long long target_partitions, int cap, int gres_engine, unsigned flags,
                        uint64_t* out_pos, int32_t* out_den, uint64_t out_cap, uint64_t* out_s,
                        int* out_g_max, uint64_t* out_rows, int* out_dims, skygpu_stats* stats,
                        char* err, size_t errlen);

/* Product-side seeded generators (bit-exact with proj/src/datagen.cpp:41-94;
 * kind 0 uni, 1 ant, 2 corr = BASELINE C3, 3 lattice = test_util.hpp:38-54).
 * Host-side input preparation, not part of the timed path. */
int skygpu_generate(int kind, uint64_t n, int d, uint64_t seed, double* out, char* err,
                    size_t errlen);

#ifdef __cplusplus
}
#endif
#endif /* SKYGPU_H */
