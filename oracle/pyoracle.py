"""ctypes view of oracle/skyoracle.c — TEST INFRASTRUCTURE ONLY.

Only tests/, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline leg
may import this module, and only as the checker.  The product package
(``paper_2412_02274_b200``) never imports it.

Every function here forwards to the C restatement of the reference path; the
reference file:line each one follows is cited in skyoracle.c.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
BUILD = os.path.join(HERE, "_build")
LIB_PATH = os.path.join(BUILD, "libskyoracle.so")
SRC = os.path.join(HERE, "skyoracle.c")
REF_DIR = os.path.join(HERE, "_ref")

GEN_KINDS = {"uni": 0, "ant": 1, "corr": 2, "lattice": 3}
STRATEGIES = {"none": 0, "grid": 1, "angular": 2, "sliced": 3}


def build(force: bool = False) -> str:
    """Compile skyoracle.c with the reference's FP rules (no contraction)."""
    os.makedirs(BUILD, exist_ok=True)
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(SRC):
        cc = os.environ.get("SKY_CC", "/usr/bin/gcc")
        subprocess.check_call([cc, "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math",
                               "-fPIC", "-shared", SRC, "-o", LIB_PATH, "-lm"])
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB_PATH)
        u64, i32, i64, dp = C.c_uint64, C.c_int, C.c_longlong, C.c_void_p
        L.so_mt64_nth.restype = u64
        L.so_mt64_nth.argtypes = [u64, u64]
        L.so_generate.argtypes = [i32, u64, i32, u64, dp]
        L.so_skyline_sfs.argtypes = [dp, dp, u64, i32, dp, dp, dp]
        L.so_skyline_bruteforce.argtypes = [dp, u64, i32, dp, dp]
        L.so_min_positive_gap.argtypes = [dp, u64, i32, dp]
        L.so_intervals_from_gap.argtypes = [C.c_double, i32, dp]
        L.so_max_grid_intervals.argtypes = [dp, u64, i32, i32, dp]
        L.so_snap.argtypes = [dp, u64, i32, dp]
        L.so_grid_resistance.argtypes = [dp, dp, u64, i32, i32, dp, dp, dp]
        L.so_gres_bruteforce.argtypes = [dp, dp, u64, i32, i32]
        L.so_gres_cells.argtypes = [dp, u64, i32, i32, dp]
        L.so_gres_cells_steps.argtypes = [dp, u64, i32, dp, i32, dp]
        L.so_make_plan.argtypes = [i32, i64, i32, dp, dp]
        L.so_assign_partitions.argtypes = [dp, dp, u64, i32, i32, i32, i64, dp]
        L.so_assign_partitions.restype = i64
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def mt64_nth(seed: int, n: int) -> int:
    return int(lib().so_mt64_nth(seed, n))


def generate(kind: str, n: int, d: int, seed: int) -> np.ndarray:
    out = np.empty((n, d), dtype=np.float64)
    rc = lib().so_generate(GEN_KINDS[kind], n, d, seed, _p(out))
    if rc:
        raise ValueError(f"so_generate rc={rc}")
    return out


def skyline_sfs(vals: np.ndarray, ids: np.ndarray | None = None):
    """-> (positions in (sum,id) output order, tests executed)"""
    vals = np.ascontiguousarray(vals, dtype=np.float64)
    n, d = vals.shape
    ids = np.arange(n, dtype=np.int64) if ids is None else np.ascontiguousarray(ids, dtype=np.int64)
    pos = np.empty(max(n, 1), dtype=np.uint64)
    cnt = np.zeros(1, dtype=np.uint64)
    tests = np.zeros(1, dtype=np.uint64)
    lib().so_skyline_sfs(_p(vals), _p(ids), n, d, _p(pos), _p(cnt), _p(tests))
    return pos[: int(cnt[0])].astype(np.int64), int(tests[0])


def skyline_bruteforce(vals: np.ndarray) -> np.ndarray:
    vals = np.ascontiguousarray(vals, dtype=np.float64)
    n, d = vals.shape
    pos = np.empty(max(n, 1), dtype=np.uint64)
    cnt = np.zeros(1, dtype=np.uint64)
    lib().so_skyline_bruteforce(_p(vals), n, d, _p(pos), _p(cnt))
    return pos[: int(cnt[0])].astype(np.int64)


def min_positive_gap(vals: np.ndarray):
    vals = np.ascontiguousarray(vals, dtype=np.float64)
    n, d = vals.shape
    g = np.zeros(1)
    ok = lib().so_min_positive_gap(_p(vals), n, d, _p(g))
    return float(g[0]) if ok else None


def max_grid_intervals(vals: np.ndarray, cap: int | None) -> int:
    vals = np.ascontiguousarray(vals, dtype=np.float64)
    n, d = vals.shape
    out = np.zeros(1, dtype=np.int32)
    rc = lib().so_max_grid_intervals(_p(vals), n, d, cap or 0, _p(out))
    if rc == -4:
        raise ValueError("max_grid_intervals: undefined, all tuples are identical on every attribute")
    if rc == -3:
        raise ValueError("max_grid_intervals: bound overflows the integer range; set a cap")
    return int(out[0])


def snap(vals: np.ndarray, g: int) -> np.ndarray:
    vals = np.ascontiguousarray(vals, dtype=np.float64)
    out = np.empty_like(vals)
    lib().so_snap(_p(vals), vals.size, g, _p(out))
    return out


def grid_resistance(sky: np.ndarray, ids: np.ndarray | None, cap: int | None):
    """-> (den per sky tuple in input order, g_max, tests)"""
    sky = np.ascontiguousarray(sky, dtype=np.float64)
    s, d = sky.shape
    ids = np.arange(s, dtype=np.int64) if ids is None else np.ascontiguousarray(ids, dtype=np.int64)
    den = np.zeros(max(s, 1), dtype=np.int32)
    gm = np.zeros(1, dtype=np.int32)
    tests = np.zeros(1, dtype=np.uint64)
    rc = lib().so_grid_resistance(_p(sky), _p(ids), s, d, cap or 0, _p(den), _p(gm), _p(tests))
    if rc == -3:
        raise ValueError("max_grid_intervals: bound overflows the integer range; set a cap")
    return den[:s], int(gm[0]), int(tests[0])


def gres_bruteforce(t: np.ndarray, r: np.ndarray, cap: int | None) -> int:
    t = np.ascontiguousarray(t, dtype=np.float64)
    r = np.ascontiguousarray(r, dtype=np.float64)
    n, d = r.shape
    rc = lib().so_gres_bruteforce(_p(t), _p(r), n, d, cap or 0)
    if rc < 0:
        raise ValueError("grid_resistance_bruteforce: uncapped interval bound too large")
    return int(rc)


def gres_cells(sky: np.ndarray, g_max: int) -> np.ndarray:
    sky = np.ascontiguousarray(sky, dtype=np.float64)
    s, d = sky.shape
    den = np.zeros(max(s, 1), dtype=np.int32)
    rc = lib().so_gres_cells(_p(sky), s, d, g_max, _p(den))
    if rc:
        raise ValueError(f"so_gres_cells unsupported input (rc={rc})")
    return den[:s]


def gres_cells_steps(sky: np.ndarray, steps) -> np.ndarray:
    """The cell scan over a subset of the steps (a shard of the step split)."""
    sky = np.ascontiguousarray(sky, dtype=np.float64)
    s, d = sky.shape
    st = np.ascontiguousarray(sorted(steps, reverse=True), dtype=np.int32)
    den = np.zeros(max(s, 1), dtype=np.int32)
    rc = lib().so_gres_cells_steps(_p(sky), s, d, _p(st), len(st), _p(den))
    if rc:
        raise ValueError(f"so_gres_cells_steps unsupported input (rc={rc})")
    return den[:s]


def make_plan(strategy: str, target: int, dims: int):
    sl = np.zeros(1, dtype=np.int32)
    pa = np.zeros(1, dtype=np.int64)
    rc = lib().so_make_plan(STRATEGIES[strategy], target, dims, _p(sl), _p(pa))
    if rc:
        raise ValueError("make_plan: invalid argument")
    return int(sl[0]), int(pa[0])


def assign_partitions(vals: np.ndarray, ids, strategy: str, slices: int, parts: int) -> np.ndarray:
    """partition.cpp:183-213 restated (so_assign_partitions)."""
    v = np.ascontiguousarray(vals, dtype=np.float64)
    n, d = v.shape
    i = None if ids is None else np.ascontiguousarray(ids, dtype=np.int64)
    out = np.zeros(max(n, 1), dtype=np.int64)
    rc = lib().so_assign_partitions(_p(v), None if i is None else _p(i), n, d,
                                    STRATEGIES[strategy], slices, parts, _p(out))
    if rc:
        raise ValueError(f"grid_cell: value outside [0,1] at flat index {rc - 1}")
    return out[:n]


def refdrive_path(release: bool = True) -> str | None:
    """Path to the compiled reference driver (oracle/_ref), if it was built."""
    p = os.path.join(REF_DIR, "refdrive" if release else "refdrive_chk")
    return p if os.path.exists(p) else None
