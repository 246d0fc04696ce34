"""Python host mirror of the reference's hot-path API over libskygpu's C-ABI.

Same names, argument meaning and error behaviour as the reference C++ API
(/root/reference/proj/include/skypar/*.hpp); ``std::invalid_argument``
becomes ``ValueError``, ``std::runtime_error`` becomes ``RuntimeError``:

    make_plan(strategy, target_partitions, dims)            partition.hpp:43
    parallel_skyline(values, ids, plan, reps, cores)        parallel.hpp:46-47
    grid_resistance(sky_values, sky_ids, plan, rep_count,   gres.hpp:73-75
                    cores, cap)
    snap_to_grid(values, intervals) / snap_relation(...)    gres.hpp:26-28
    max_grid_intervals(values, cap)                         gres.hpp:35

A relation is a float64 array of shape (n, d) plus an int64 id vector
(default: row index, the reference's generator/CSV convention).  There is
no CPU fallback: if libskygpu.so is missing or no sm_100 device is present,
every call raises.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
from dataclasses import dataclass, field

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
# (SKYGPU_LIB_PATH: an alternative in-tree build, for A/B measurements)
LIB_PATH = os.environ.get("SKYGPU_LIB_PATH") or os.path.join(_PKG, "_lib", "libskygpu.so")

SKYGPU_OK, SKYGPU_EINVAL, SKYGPU_ERUNTIME, SKYGPU_ECUDA, SKYGPU_ENOMEM = range(5)
GRES_AUTO, GRES_PAIRS, GRES_CELLS = 0, 1, 2
DEVICE_PTRS, CHECK_SKYLINE, SKIP_GRES = 1, 2, 4
SKY_AUTO, SKY_ROUNDS, SKY_GRID = 0, 8, 16  # skyline engine flags
NORMALIZE = 32  # pipeline flag: min-max normalise on the device first
SKY_PARTS = 64  # pipeline flag: the plan's partitions as local-skyline pruning before the merge


class SkyGpuError(RuntimeError):
    """CUDA / device failure inside libskygpu (no CPU fallback exists)."""


class Strategy(enum.IntEnum):
    NONE = 0
    GRID = 1
    ANGULAR = 2
    SLICED = 3

    @classmethod
    def from_name(cls, name: str) -> "Strategy":  # partition.cpp:43-49
        table = {"none": cls.NONE, "grid": cls.GRID, "angular": cls.ANGULAR, "sliced": cls.SLICED}
        if name not in table:
            raise ValueError("unknown strategy: " + name)
        return table[name]


class _Plan(C.Structure):
    _fields_ = [("strategy", C.c_int), ("slices", C.c_int), ("partitions", C.c_longlong),
                ("dims", C.c_int)]


class Stats(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in ("tuples_in", "tuples_into_parallel", "tuples_into_final",
                                           "skyline_size", "skyline_tests", "gres_tests",
                                           "gres_cells")] + \
               [(n, C.c_int) for n in ("g_max", "gres_steps", "gres_engine", "code_bits",
                                        "sfs_rounds", "sky_engine")] + \
               [(n, C.c_double) for n in ("ms_total", "ms_h2d", "ms_skyline", "ms_gres", "ms_d2h",
                                           "ms_gres_kernel", "ms_sky_kernel")] + \
               [(n, C.c_uint64) for n in ("gres_kernel_launches", "sky_kernel_launches",
                                           "kernel_launches", "sky_units")]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


@dataclass
class PartitionPlan:  # partition.hpp:27-32
    strategy: Strategy = Strategy.NONE
    slices: int = 1
    partitions: int = 1
    dims: int = 0

    def _c(self) -> _Plan:
        return _Plan(int(self.strategy), self.slices, self.partitions, self.dims)


_lib = None


def lib() -> C.CDLL:
    """Load the in-tree libskygpu.so (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2412_02274_b200.build` "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        vp, u64, i32, i64, sz, cp = C.c_void_p, C.c_uint64, C.c_int, C.c_longlong, C.c_size_t, C.c_char_p
        L.skygpu_version.restype = i32
        L.skygpu_device_count.restype = i32
        L.skygpu_set_device.argtypes = [i32, cp, sz]
        L.skygpu_set_stream.argtypes = [vp, cp, sz]
        L.skygpu_make_plan.argtypes = [i32, i64, i32, C.POINTER(_Plan), cp, sz]
        L.skygpu_assign_partitions.argtypes = [vp, vp, u64, i32, C.POINTER(_Plan), vp, cp, sz]
        L.skygpu_skyline_bnl.argtypes = [vp, vp, u64, i32, vp, vp, vp, cp, sz]
        L.skygpu_parallel_skyline.argtypes = [vp, vp, u64, i32, C.POINTER(_Plan), vp, vp, u64, i32,
                                              vp, vp, C.POINTER(Stats), cp, sz]
        L.skygpu_grid_resistance.argtypes = [vp, vp, u64, i32, C.POINTER(_Plan), u64, i32, i32, i32,
                                             vp, vp, C.POINTER(Stats), cp, sz]
        L.skygpu_snap_relation.argtypes = [vp, u64, i32, vp, cp, sz]
        L.skygpu_max_grid_intervals.argtypes = [vp, u64, i32, i32, vp, cp, sz]
        L.skygpu_pipeline.argtypes = [vp, vp, u64, i32, C.POINTER(_Plan), i32, i32, i32, i32,
                                      C.c_uint, vp, vp, vp, vp, C.POINTER(Stats), cp, sz]
        L.skygpu_generate.argtypes = [i32, u64, i32, u64, vp, cp, sz]
        L.skygpu_sfs_accounting.argtypes = [vp, vp, u64, i32, vp, i64, vp, u64, vp, vp, vp, vp, vp,
                                            cp, sz]
        L.skygpu_set_collective.argtypes = [vp, vp, cp, sz]
        L.skygpu_normalize.argtypes = [vp, u64, i32, vp, cp, sz]
        L.skygpu_read_csv.argtypes = [cp, u64, cp, vp, u64, vp, vp, cp, sz]
        L.skygpu_pipeline_csv.argtypes = [cp, u64, cp, i32, i64, i32, i32, C.c_uint, vp, vp, u64,
                                          vp, vp, vp, vp, C.POINTER(Stats), cp, sz]
        L.skygpu_select_representatives.argtypes = [vp, vp, u64, i32, u64, vp, vp, vp, cp, sz]
        _lib = L
    return _lib


EXPORTED_SYMBOLS = ("skygpu_version", "skygpu_device_count", "skygpu_set_device", "skygpu_set_stream",
                    "skygpu_release", "skygpu_make_plan", "skygpu_parallel_skyline",
                    "skygpu_grid_resistance", "skygpu_snap_relation", "skygpu_max_grid_intervals",
                    "skygpu_pipeline", "skygpu_generate", "skygpu_sfs_accounting",
                    "skygpu_set_collective", "skygpu_normalize", "skygpu_select_representatives",
                    "skygpu_read_csv", "skygpu_pipeline_csv", "skygpu_host_buffer",
                    "skygpu_nccl_unique_id", "skygpu_nccl_init", "skygpu_nccl_release",
                    "skygpu_cells_step_plan", "skygpu_assign_partitions", "skygpu_skyline_bnl")


def _check(rc: int, err: C.Array) -> None:
    if rc == SKYGPU_OK:
        return
    msg = err.value.decode(errors="replace")
    if rc == SKYGPU_EINVAL:
        raise ValueError(msg)
    if rc == SKYGPU_ERUNTIME:
        raise RuntimeError(msg)
    if rc == SKYGPU_ENOMEM:
        raise MemoryError(msg)
    raise SkyGpuError(msg)


def _errbuf():
    return C.create_string_buffer(1024)


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _relation(values, ids):
    v = np.ascontiguousarray(values, dtype=np.float64)
    if v.ndim != 2:
        raise ValueError("a relation is an (n, d) float64 array")
    n = v.shape[0]
    i = np.arange(n, dtype=np.int64) if ids is None else np.ascontiguousarray(ids, dtype=np.int64)
    if i.shape != (n,):
        raise ValueError("ids must have one entry per tuple")
    return v, i


# ------------------------------------------------------------------ API
def make_plan(strategy, target_partitions: int, dims: int) -> PartitionPlan:
    s = Strategy.from_name(strategy) if isinstance(strategy, str) else Strategy(strategy)
    out = _Plan()
    err = _errbuf()
    _check(lib().skygpu_make_plan(int(s), int(target_partitions), int(dims), C.byref(out), err, 1024), err)
    return PartitionPlan(Strategy(out.strategy), out.slices, out.partitions, out.dims)


def assign_partitions(values, plan: PartitionPlan, ids=None) -> np.ndarray:
    """partition.hpp:90 (partition.cpp:183-213) on the device: the partition of
    every tuple under ``plan`` (int64, one per tuple)."""
    v, i = _relation(values, ids)
    n, d = v.shape
    out = np.zeros(max(n, 1), dtype=np.int64)
    err = _errbuf()
    _check(lib().skygpu_assign_partitions(_p(v), _p(i), n, d, C.byref(plan._c()), _p(out), err,
                                          1024), err)
    return out[:n]


@dataclass
class SkylineResult:
    positions: np.ndarray  # input positions, (sum, id) order
    ids: np.ndarray
    values: np.ndarray
    stats: dict = field(default_factory=dict)


def parallel_skyline(values, ids=None, plan: PartitionPlan | None = None, reps=None,
                     cores: int = 1) -> SkylineResult:
    """parallel.hpp:46-47.  ``reps`` = (rep_values (k, d), rep_ids) or None."""
    v, i = _relation(values, ids)
    n, d = v.shape
    plan = plan or PartitionPlan(Strategy.NONE, 1, 1, d)
    if reps is not None and len(reps[0]):
        rv = np.ascontiguousarray(reps[0], dtype=np.float64).reshape(-1, d)
        ri = np.ascontiguousarray(reps[1], dtype=np.int64)
    else:
        rv = np.zeros((0, d)); ri = np.zeros(0, dtype=np.int64)
    out = np.empty(max(n, 1), dtype=np.uint64)
    cnt = np.zeros(1, dtype=np.uint64)
    st = Stats()
    err = _errbuf()
    _check(lib().skygpu_parallel_skyline(_p(v), _p(i), n, d, C.byref(plan._c()), _p(rv), _p(ri),
                                         rv.shape[0], int(cores), _p(out), _p(cnt), C.byref(st),
                                         err, 1024), err)
    pos = out[: int(cnt[0])].astype(np.int64)
    return SkylineResult(pos, i[pos], v[pos], st.as_dict())


def skyline_bnl(values, ids=None) -> SkylineResult:
    """core.hpp:78 skyline_bnl: the tuples no tuple dominates (a set; returned
    in (sum, id) order)."""
    v, i = _relation(values, ids)
    n, d = v.shape
    out = np.empty(max(n, 1), dtype=np.uint64)
    cnt = np.zeros(1, dtype=np.uint64)
    st = Stats()
    err = _errbuf()
    _check(lib().skygpu_skyline_bnl(_p(v), _p(i), n, d, _p(out), _p(cnt), C.byref(st), err, 1024),
           err)
    pos = out[: int(cnt[0])].astype(np.int64)
    return SkylineResult(pos, i[pos], v[pos], st.as_dict())


@dataclass
class GridResistanceResult:  # gres.hpp:56-64
    ids: np.ndarray
    den: np.ndarray  # denominator per input skyline tuple
    g_max: int
    stats: dict = field(default_factory=dict)

    @property
    def denominators(self) -> dict:
        return {int(k): int(v) for k, v in zip(self.ids, self.den)}


def grid_resistance(sky_values, sky_ids=None, plan: PartitionPlan | None = None, rep_count: int = 0,
                    cores: int = 1, cap: int | None = 25, check_skyline: bool = False
                    ) -> GridResistanceResult:
    """gres.hpp:73-75.  ``cap=None`` = std::nullopt."""
    v, i = _relation(sky_values, sky_ids)
    s, d = v.shape
    plan = plan or PartitionPlan(Strategy.NONE, 1, 1, d)
    den = np.zeros(max(s, 1), dtype=np.int32)
    gm = np.zeros(1, dtype=np.int32)
    st = Stats()
    err = _errbuf()
    _check(lib().skygpu_grid_resistance(_p(v), _p(i), s, d, C.byref(plan._c()), int(rep_count),
                                        int(cores), 0 if cap is None else int(cap),
                                        1 if check_skyline else 0, _p(den), _p(gm), C.byref(st),
                                        err, 1024), err)
    return GridResistanceResult(i, den[:s], int(gm[0]), st.as_dict())


def snap_relation(values, intervals: int) -> np.ndarray:
    v = np.ascontiguousarray(values, dtype=np.float64)
    out = np.empty_like(v)
    err = _errbuf()
    _check(lib().skygpu_snap_relation(_p(v), v.size, int(intervals), _p(out), err, 1024), err)
    return out


def snap_to_grid(values, intervals: int) -> np.ndarray:
    return snap_relation(np.asarray(values, dtype=np.float64).reshape(1, -1), intervals)[0]


def max_grid_intervals(values, cap: int | None) -> int:
    v = np.ascontiguousarray(values, dtype=np.float64)
    if v.ndim != 2:
        raise ValueError("a relation is an (n, d) float64 array")
    out = np.zeros(1, dtype=np.int32)
    err = _errbuf()
    _check(lib().skygpu_max_grid_intervals(_p(v), v.shape[0], v.shape[1], 0 if cap is None else int(cap),
                                           _p(out), err, 1024), err)
    return int(out[0])


@dataclass
class PipelineResult:
    positions: np.ndarray
    den: np.ndarray
    g_max: int
    stats: dict


def pipeline(values, ids=None, plan: PartitionPlan | None = None, cap: int | None = 25,
             engine: int = GRES_AUTO, shard_rank: int = 0, shard_world: int = 1,
             check_skyline: bool = False, skip_gres: bool = False,
             sky_engine: int = SKY_AUTO, normalize: bool = False,
             local_prune: bool = False) -> PipelineResult:
    """Skyline + grid resistance in one call (harness.cpp:208, :229-231).
    ``sky_engine`` forces the prefix-round (SKY_ROUNDS) or one-pass rank-grid
    (SKY_GRID) skyline engine; the default picks by the first round's yield.
    ``local_prune`` runs the plan's partitions as local-skyline pruning before
    the merge (SKY_PARTS, parallel.cpp:59-73 recast)."""
    v, i = _relation(values, ids)
    n, d = v.shape
    plan = plan or PartitionPlan(Strategy.NONE, 1, 1, d)
    pos = np.empty(max(n, 1), dtype=np.uint64)
    den = np.zeros(max(n, 1), dtype=np.int32)
    s = np.zeros(1, dtype=np.uint64)
    gm = np.zeros(1, dtype=np.int32)
    st = Stats()
    err = _errbuf()
    flags = (CHECK_SKYLINE if check_skyline else 0) | (SKIP_GRES if skip_gres else 0) | int(sky_engine)
    flags |= NORMALIZE if normalize else 0
    flags |= SKY_PARTS if local_prune else 0
    _check(lib().skygpu_pipeline(_p(v), _p(i), n, d, C.byref(plan._c()), 0 if cap is None else int(cap),
                                 int(engine), int(shard_rank), int(shard_world), flags, _p(pos), _p(den),
                                 _p(s), _p(gm), C.byref(st), err, 1024), err)
    S = int(s[0])
    return PipelineResult(pos[:S].astype(np.int64), den[:S].copy(), int(gm[0]), st.as_dict())


def pipeline_raw(vals_ptr: int, ids_ptr: int, n: int, d: int, plan: PartitionPlan, cap: int | None,
                 engine: int, shard_rank: int, shard_world: int, flags: int, out_pos_ptr: int,
                 out_den_ptr: int):
    """Pointer-level call (host pinned or device pointers per ``flags``) used by bench.py."""
    s = np.zeros(1, dtype=np.uint64)
    gm = np.zeros(1, dtype=np.int32)
    st = Stats()
    err = _errbuf()
    _check(lib().skygpu_pipeline(C.c_void_p(vals_ptr), C.c_void_p(ids_ptr), n, d, C.byref(plan._c()),
                                 0 if cap is None else int(cap), int(engine), int(shard_rank),
                                 int(shard_world), int(flags), C.c_void_p(out_pos_ptr),
                                 C.c_void_p(out_den_ptr), _p(s), _p(gm), C.byref(st), err, 1024), err)
    return int(s[0]), int(gm[0]), st.as_dict()


_DEVICE = 0  # the device the library's calls run on (set_device)


def set_device(device: int) -> None:
    global _DEVICE
    err = _errbuf()
    _check(lib().skygpu_set_device(int(device), err, 1024), err)
    _DEVICE = int(device)


def current_device() -> int:
    """The device set with set_device (the library's buffers live there)."""
    return _DEVICE


def set_stream(stream_ptr: int | None) -> None:
    err = _errbuf()
    _check(lib().skygpu_set_stream(C.c_void_p(stream_ptr or 0), err, 1024), err)


def device_count() -> int:
    return int(lib().skygpu_device_count())


GEN_KINDS = {"uni": 0, "ant": 1, "corr": 2, "lattice": 3}


def generate(kind: str, n: int, d: int, seed: int) -> np.ndarray:
    """Seeded input (datagen.cpp recipes; 'corr' = BASELINE C3)."""
    out = np.empty((n, d), dtype=np.float64)
    err = _errbuf()
    _check(lib().skygpu_generate(GEN_KINDS[kind], n, d, seed, _p(out), err, 1024), err)
    return out


@dataclass
class Accounting:
    """The reference's DominanceCounter totals of one parallel_skyline run
    (parallel.cpp:59-93): per-partition tests (rep filter + local SFS), the
    merge-phase tests, the merge input size and the skyline positions."""
    per_partition: np.ndarray
    final_tests: int
    into_final: int
    positions: np.ndarray


def sfs_accounting(values, ids, pids, partitions: int, reps=None) -> Accounting:
    """Exact reference accounting (metrics-parity mode; skygpu_sfs_accounting).
    ``pids[i]`` = partition of tuple i (the reference's assign_partitions), -1
    = dropped before phase 1; ``reps`` = representative tuples (k x d)."""
    v, i = _relation(values, ids)
    n, d = v.shape
    pid = np.ascontiguousarray(pids, dtype=np.int64)
    if pid.shape != (n,):
        raise ValueError("pids must hold one partition id per tuple")
    r = np.ascontiguousarray(np.zeros((0, d)) if reps is None else reps, dtype=np.float64)
    per = np.zeros(max(int(partitions), 1), dtype=np.uint64)
    fin = np.zeros(1, dtype=np.uint64)
    into = np.zeros(1, dtype=np.uint64)
    pos = np.empty(max(n, 1), dtype=np.uint64)
    cnt = np.zeros(1, dtype=np.uint64)
    err = _errbuf()
    _check(lib().skygpu_sfs_accounting(_p(v), _p(i), n, d, _p(pid), int(partitions), _p(r), len(r),
                                       _p(per), _p(fin), _p(into), _p(pos), _p(cnt), err, 1024), err)
    return Accounting(per[:int(partitions)].copy(), int(fin[0]), int(into[0]),
                      pos[:int(cnt[0])].astype(np.int64))


def cells_step_plan(col_max, g_max: int, s: int, rank: int, world: int) -> list:
    """Steps of the cell engine's scan that shard `rank` of `world` runs
    (host only; the split of a sharded pipeline call)."""
    cm = np.ascontiguousarray(col_max, dtype=np.float64)
    out = np.zeros(max(int(g_max), 1), dtype=np.int32)
    n = np.zeros(1, dtype=np.int32)
    err = _errbuf()
    _check(lib().skygpu_cells_step_plan(_p(cm), len(cm), int(g_max), int(s), int(rank), int(world),
                                        _p(out), _p(n), err, 1024), err)
    return out[:int(n[0])].tolist()


def _share_torch_nccl() -> None:
    """Load torch (and with it torch's libnccl.so.2) before the library
    loads NCCL, so the process holds ONE NCCL copy: libskygpu then binds the
    copy already present (RTLD_NOLOAD) instead of the system's older one,
    which torch's own NCCL references would otherwise resolve to."""
    try:
        import torch  # noqa: F401
        torch.cuda.is_available()
    except Exception:
        pass


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id (skygpu_nccl_unique_id) — made on one rank,
    shipped to the others out of band."""
    _share_torch_nccl()
    buf = C.create_string_buffer(128)
    err = _errbuf()
    _check(lib().skygpu_nccl_unique_id(buf, err, 1024), err)
    return buf.raw


def nccl_init(uid: bytes, nranks: int, rank: int) -> None:
    """Join the library's own NCCL group on the current device: sharded
    pipeline calls then MAX-all-reduce in place on the library's stream."""
    if len(uid) != 128:
        raise ValueError("nccl_init: the unique id is 128 bytes")
    _share_torch_nccl()
    err = _errbuf()
    _check(lib().skygpu_nccl_init(C.create_string_buffer(uid, 128), int(nranks), int(rank), err,
                                  1024), err)


def nccl_release() -> None:
    lib().skygpu_nccl_release()


# skygpu_allreduce_max_fn(dev_ptr, count, elem_bytes, cuda_stream, user) -> int
COLLECTIVE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_uint64, C.c_int, C.c_void_p, C.c_void_p)
_collective_ref = None  # keeps the installed callback alive


def set_collective(fn=None) -> None:
    """Install the exchange step of sharded pipeline calls (skygpu.h:
    skygpu_set_collective): ``fn(dev_ptr, count, elem_bytes, stream)`` must
    MAX-all-reduce the device buffer in place across the shard group and
    return 0.  ``None`` uninstalls it."""
    global _collective_ref
    err = _errbuf()
    if fn is None:
        _collective_ref = None
        _check(lib().skygpu_set_collective(None, None, err, 1024), err)
        return

    def tramp(ptr, count, elem_bytes, stream, user):
        try:
            return int(fn(int(ptr or 0), int(count), int(elem_bytes), int(stream or 0)) or 0)
        except Exception:  # an exception must not unwind through C
            import traceback
            traceback.print_exc()
            return 1

    _collective_ref = COLLECTIVE_FN(tramp)
    _check(lib().skygpu_set_collective(C.cast(_collective_ref, C.c_void_p), None, err, 1024), err)


def normalize(values) -> np.ndarray:
    """harness.cpp:161-177 normalize on the device (bit-identical)."""
    v = np.ascontiguousarray(values, dtype=np.float64)
    n, d = v.shape
    out = np.empty_like(v)
    err = _errbuf()
    _check(lib().skygpu_normalize(_p(v), n, d, _p(out), err, 1024), err)
    return out


def select_representatives(values, ids=None, k: int = 1):
    """partition.cpp:249-271 with sum_score on the device: (positions of the
    kept picks in (sum, id) order, the pruning's dominance-test count)."""
    v, i = _relation(values, ids)
    n, d = v.shape
    pos = np.empty(max(min(int(k), n), 1), dtype=np.uint64)
    cnt = np.zeros(1, dtype=np.uint64)
    tests = np.zeros(1, dtype=np.uint64)
    err = _errbuf()
    _check(lib().skygpu_select_representatives(_p(v), _p(i), n, d, int(k), _p(pos), _p(cnt),
                                                _p(tests), err, 1024), err)
    return pos[:int(cnt[0])].astype(np.int64), int(tests[0])


def read_csv_bytes(data: bytes, name: str = ""):
    """harness.cpp:93-134 read_dataset_csv on the device: (values rows x dims,
    ids).  Format errors raise RuntimeError with the reference's text (the
    `name` it reports is the path the reference would print)."""
    cap = (len(data) + 1) // 2 + 1
    out = np.empty(cap, dtype=np.float64)
    rows = np.zeros(1, dtype=np.uint64)
    dims = np.zeros(1, dtype=np.int32)
    err = C.create_string_buffer(4096)  # the reference's texts quote the field
    _check(lib().skygpu_read_csv(data, len(data), name.encode(), _p(out), cap, _p(rows), _p(dims),
                                 err, 4096), err)
    r, d = int(rows[0]), int(dims[0])
    return out[:r * d].reshape(r, d).copy(), np.arange(r, dtype=np.int64)


def load_dataset_csv(path: str):
    """harness.cpp:127-131 load_dataset_csv (the file read on the host, parsed
    on the device)."""
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError:
        raise RuntimeError("cannot open dataset file: " + path) from None
    return read_csv_bytes(data, path)


def pipeline_csv(data: bytes, name: str = "", strategy: str = "none", target_partitions: int = 1,
                 cap: int | None = 25, engine: int = GRES_AUTO, normalize: bool = False):
    """run_experiment with --dataset on the device: the CSV bytes parsed on the
    GPU (optionally normalised there) and fed to the pipeline without a host
    round trip.  Returns (PipelineResult, (rows, dims))."""
    cap_t = (len(data) + 1) // 2 + 1
    pos = np.empty(cap_t, dtype=np.uint64)
    den = np.zeros(cap_t, dtype=np.int32)
    s = np.zeros(1, dtype=np.uint64)
    gm = np.zeros(1, dtype=np.int32)
    rows = np.zeros(1, dtype=np.uint64)
    dims = np.zeros(1, dtype=np.int32)
    st = Stats()
    err = C.create_string_buffer(4096)
    _check(lib().skygpu_pipeline_csv(data, len(data), name.encode(), int(Strategy.from_name(strategy)),
                                     int(target_partitions), 0 if cap is None else int(cap),
                                     int(engine), NORMALIZE if normalize else 0, _p(pos), _p(den),
                                     cap_t, _p(s), _p(gm), _p(rows), _p(dims), C.byref(st), err,
                                     4096), err)
    S = int(s[0])
    res = PipelineResult(pos[:S].astype(np.int64), den[:S].copy(), int(gm[0]), st.as_dict())
    return res, (int(rows[0]), int(dims[0]))
