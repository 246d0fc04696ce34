#!/usr/bin/env python
"""Benchmark of the grid-resistance hot path (skyline + descending-g scan).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C5]
                    [--impl ours|reference] [--scaling weak|strong]

One STEP = one pass of the hot path over one seeded synthetic relation:
parallel_skyline of the n tuples, then grid_resistance of every skyline tuple
(proj/src/harness.cpp:208, :229-231).  Default workload C5, the LARGEST
BASELINE.json configuration that fits one GPU (configs[4]: anti-correlated
n=10,000,000, d=7, seed 1, cap 25, angular p=64; 560 MB of float64).
--gpus N without torchrun's WORLD_SIZE re-launches itself under
torch.distributed.run with N ranks (127.0.0.1); N > 1 defaults to strong
scaling (one C5 instance sharded over the ranks).

value  = skyline tuples whose resistance was computed per second, whole job,
         inputs resident in HBM (device-event timed, max over ranks).
e2e    = the same metric through the public C-ABI call with pinned HOST
         buffers: H2D of the relation + ids and D2H of positions + denominators
         inside the timed region (host clock around the synchronous call).
--impl reference times the unmodified reference library (oracle/_ref,
compiled from /root/reference by oracle/build_ref.sh) on all host cores.
Timing: W untimed warm-up steps, then K steps, each bracketed by CUDA events
on the stream the kernels run on; L2 is flushed (256 MiB write) before every
timed step because the C2 relation (32 MB) fits in the 126 MB L2.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (generator, n, d, seed, strategy, target partitions, cap)
    "C1": ("uni", 100_000, 4, 1, "sliced", 16, 25),
    "C2": ("ant", 1_000_000, 3, 1, "angular", 16, 25),
    "C3": ("corr", 1_000_000, 6, 1, "sliced", 16, 25),
    "C4": ("uni", 10_000_000, 5, 1, "angular", 64, 25),
    "C5p10k": ("ant", 10_000, 7, 1, "angular", 64, 25),
    "C5p20k": ("ant", 20_000, 7, 1, "angular", 64, 25),
    "C5": ("ant", 10_000_000, 7, 1, "angular", 64, 25),
}
# the CPU reference cannot finish these in a bench run (C5: days; its SFS merge
# is quadratic in the skyline, S ~ 0.65 n); it is timed on the leading prefix
# of the same seeded stream instead (the generator is per-tuple sequential, so
# a prefix IS the first tuples of the full relation), and the line says so
CPU_SAMPLE_N = {"C5": 20_000}
# timed repetitions of the reference arm when one sampled step is long (the
# C5 20k prefix is ~20-40 s of CPU per step): the arm stays within minutes
REF_MAX_STEPS = {"C5": 4}
DEFAULT_WORKLOAD = "C5"
METRIC = "grid-resistance skyline tuples/sec"
UNIT = "skyline tuples/s"


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ------------------------------------------------------------- reference arm
def run_reference_cpu(wl, repeat, cores=0):
    """Time the unmodified reference (oracle/_ref/refdrive, release build) —
    the CPU baseline.  Falls back to the C oracle port when it was not built."""
    from oracle import pyoracle as po
    gen, n, d, seed, strat, p, cap = WORKLOADS[wl]
    n = CPU_SAMPLE_N.get(wl, n)
    exe = po.refdrive_path(release=True)
    ncores = os.cpu_count() or 1
    if exe:
        cmd = [exe, "--mode", "bench", "--gen", gen, "--n", str(n), "--d", str(d), "--seed",
               str(seed), "--strategy", strat, "--p", str(p), "--cap", str(cap), "--cores",
               str(cores or ncores), "--repeat", str(repeat)]
        r = json.loads(subprocess.check_output(cmd, text=True))
        step_ms = r["skyline_ms_mean"] + r["gres_ms_mean"]
        return {"kind": "reference", "cores": r["cores"], "step_ms": step_ms, "S": r["skyline_size"],
                "detail": r, "n": n}
    v = po.generate(gen, n, d, seed)
    t0 = time.perf_counter()
    for _ in range(repeat):
        pos, _ = po.skyline_sfs(v)
        po.grid_resistance(v[pos], pos, cap)
    step_ms = (time.perf_counter() - t0) * 1e3 / repeat
    return {"kind": "port", "cores": 1, "step_ms": step_ms, "S": len(pos), "detail": {}, "n": n}


def sample_text(wl, r, repeat):
    n_full = WORKLOADS[wl][1]
    if r.get("n", n_full) != n_full:
        return (f"leading {r['n']}-tuple prefix of the {wl} stream (same seed; the generator is "
                f"per-tuple sequential) x{repeat}: the full n={n_full} is not computable by the "
                f"CPU reference within a bench run (its SFS merge is quadratic in the skyline)")
    return f"full {wl} workload x{repeat}"


def reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    wl = args.workload
    # warm-up runs are discarded (one is enough on a CPU); K timed runs (one
    # step = one full pass over the sample), at most REF_MAX_STEPS[wl]
    steps = max(1, min(args.steps, REF_MAX_STEPS.get(wl, args.steps)))
    if args.warmup:
        run_reference_cpu(wl, 1)
    r = run_reference_cpu(wl, steps)
    value = r["S"] / (r["step_ms"] / 1e3)
    gen, n, d, seed, strat, p, cap = WORKLOADS[wl]
    sampled = r["n"] != n
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": r["step_ms"],
        "steps_timed": steps,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference generator, seeded)",
        "config": {"workload": f"{wl}: {gen} n={n} d={d} seed={seed}, {strat} p={p}, cap={cap}"
                               + (f" [reference timed on the leading {r['n']}-tuple prefix]"
                                  if sampled else ""),
                   "cores": r["cores"], "cpu": cpu_model()},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": r["cores"], "kind": r["kind"],
                         "sample": sample_text(wl, r, steps)},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "reference_detail": r["detail"],
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------- clocks
class ClockSampler:
    def __init__(self, device_index):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._t = None
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.ok = False

    def _run(self):
        nv = self.nv
        names = {
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
            "hw_power_brake_slowdown": getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in names.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(0.01)

    def start(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()

    def stop(self):
        if self._t:
            self._stop.set()
            self._t.join()
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "samples": len(self.samples),
                "reasons": sorted(self.reasons)}


# ------------------------------------------------------------------ our arm
def our_arm(args):
    import torch
    import torch.distributed as dist

    import paper_2412_02274_b200 as sk
    from paper_2412_02274_b200 import skypar

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    skypar.set_device(local)
    stream = torch.cuda.current_stream(dev)
    skypar.set_stream(stream.cuda_stream)

    gen, n, d, seed, strat, p, cap = WORKLOADS[args.workload]
    strong = args.scaling == "strong"
    my_seed = seed if (strong or world == 1) else seed + rank  # weak: one instance per rank
    host = sk.generate(gen, n, d, my_seed)
    ids_host = np.arange(n, dtype=np.int64)
    plan = sk.make_plan(strat, p, d)
    vals_d = torch.from_numpy(host).to(dev)
    ids_d = torch.from_numpy(ids_host).to(dev)
    pos_d = torch.empty(n, dtype=torch.int64, device=dev)
    den_d = torch.empty(n, dtype=torch.int32, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    shard_rank, shard_world = (rank, world) if strong else (0, 1)
    sky_flag = {"auto": skypar.SKY_AUTO, "rounds": skypar.SKY_ROUNDS, "grid": skypar.SKY_GRID}[args.sky_engine]
    if args.local_prune:  # the plan's partitions as local-skyline pruning before the merge
        sky_flag |= skypar.SKY_PARTS

    if strong and world > 1:
        # the library's own NCCL group (unique id shipped over
        # torch.distributed): its exchange steps (rank-grid keep flags,
        # denominators) are ncclAllReduce(MAX) on the library's stream
        from paper_2412_02274_b200 import dist as skydist
        skydist.init_library_nccl()

    def step_device():
        return skypar.pipeline_raw(vals_d.data_ptr(), ids_d.data_ptr(), n, d, plan, cap,
                                   args.engine, shard_rank, shard_world,
                                   skypar.DEVICE_PTRS | sky_flag, pos_d.data_ptr(),
                                   den_d.data_ptr())

    for _ in range(args.warmup):
        step_device()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    clocks = ClockSampler(local)
    clocks.start()
    times, stats = [], []
    S = gm = 0
    for _ in range(args.steps):
        flush.zero_()  # L2 flush outside the timed region
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        S, gm, st = step_device()
        e1.record(stream)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
        stats.append(st)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk = clocks.stop()

    total_ms = sum(times)
    units = S if strong else S * 1  # per rank
    t = torch.tensor([total_ms, float(units)], dtype=torch.float64, device=dev)
    if world > 1:
        tmax = t.clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        tsum = t.clone()
        dist.all_reduce(tsum, op=dist.ReduceOp.SUM)
        total_ms = float(tmax[0])
        units_all = float(t[1]) if strong else float(tsum[1])
    else:
        units_all = float(units)
    ms_per_step = total_ms / args.steps
    value = units_all / (ms_per_step / 1e3)

    # ---- e2e through the public API with pinned host buffers
    skypar.set_stream(None)
    pin_vals = torch.from_numpy(host).pin_memory()
    pin_ids = torch.from_numpy(ids_host).pin_memory()
    out_pos = torch.empty(n, dtype=torch.int64).pin_memory()
    out_den = torch.empty(n, dtype=torch.int32).pin_memory()

    def step_e2e():
        S2, _, _ = skypar.pipeline_raw(pin_vals.data_ptr(), pin_ids.data_ptr(), n, d, plan, cap,
                                       args.engine, shard_rank, shard_world, sky_flag,
                                       out_pos.data_ptr(), out_den.data_ptr())
        return S2

    for _ in range(max(1, args.warmup)):
        step_e2e()
    e2e_times = []
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        step_e2e()
        e2e_times.append((time.perf_counter() - t0) * 1e3)
    e2e_ms = sum(e2e_times) / len(e2e_times)
    if world > 1:
        te = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e_ms = float(te[0])
    e2e_value = units_all / (e2e_ms / 1e3)

    # ---- roofline of the dominant kernel (live CUDA-event launch times)
    sky_ms = sum(s["ms_sky_kernel"] for s in stats) / len(stats)
    gres_ms = sum(s["ms_gres_kernel"] for s in stats) / len(stats)
    st0 = stats[-1]
    roof = roofline(st0, sky_ms, gres_ms, d, clk, args.workload)

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong" if strong else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded reference generators, bit-exact)",
        "config": {"workload": f"{args.workload}: {gen} n={n} d={d} seed={seed}"
                               f"{'' if strong or world == 1 else '+rank'}, {strat} p={p}, cap={cap}",
                   "skyline_size": S, "g_max": gm, "l2": "flushed (256 MiB write) before each step",
                   "parallelism": f"{'one instance sharded: rank-grid rows, cell-engine steps (or gres tuples), libskygpu NCCL MAX all-reduces' if strong else 'independent instance'}"
                                  f" per GPU x{world}",
                   "gres_engine": {0: "auto", 1: "pairs", 2: "cells"}[args.engine],
                   "skyline_engine": {8: "prefix rounds", 16: "rank grid"}.get(stats[-1]["sky_engine"], "?")
                                     + (" after local-skyline pruning per partition" if args.local_prune else ""),
                   "tuples_into_final": stats[-1]["tuples_into_final"]},
        "e2e": {"value": e2e_value, "unit": UNIT, "ms_per_step": e2e_ms,
                # (the spread of the host-timed steps: host noise shows here)
                "ms_min": min(e2e_times), "ms_median": sorted(e2e_times)[len(e2e_times) // 2],
                "h2d_bytes_per_step": n * d * 8 + n * 8,
                "d2h_bytes_per_step": S * 8 + S * 4},  # u64 positions + i32 denominators
        "gpu_launches": int(sum(s["kernel_launches"] for s in stats)),
        "roofline": roof,
        "clocks": clk,
        "stage_ms": {"skyline": st0["ms_skyline"], "gres": st0["ms_gres"],
                     "sky_kernels": sky_ms, "gres_kernels": gres_ms},
        "tests": {"skyline": st0["skyline_tests"], "gres": st0["gres_tests"],
                  "sfs_rounds": st0["sfs_rounds"], "gres_steps": st0["gres_steps"],
                  "code_bits": st0["code_bits"]},
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            # ~10-30 s of CPU work: one pass over the C5 prefix, 3 elsewhere
            rep = args.cpu_repeat or (1 if args.workload == "C5" else 3)
            r = run_reference_cpu(args.workload, rep)
            line["cpu_baseline"] = {"value": r["S"] / (r["step_ms"] / 1e3), "unit": UNIT,
                                    "cores": r["cores"], "kind": r["kind"],
                                    "sample": sample_text(args.workload, r, rep)
                                              + f" ({r['step_ms']:.1f} ms/step, {cpu_model()})"}
        except Exception as e:  # pragma: no cover
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 0, "kind": "port",
                                    "sample": f"unavailable: {e}"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


TRAFFIC_FILE = os.path.join(ROOT, "profiles", "traffic.json")


def _hbm_peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except (OSError, ValueError, KeyError):
        return 6650.0  # B200_PROFILING.md fallback ("of fallback")


HBM_PEAK_GBS = _hbm_peak()


def kernel_traffic(workload, kernel):
    """DRAM bytes per launch of `kernel` from the committed ncu capture
    (profiles/traffic.json, written by scripts/ncu_summary.py), else None."""
    try:
        t = json.load(open(TRAFFIC_FILE))
        return t.get(workload, {}).get(kernel)
    except (OSError, ValueError):
        return None


def roofline(st, sky_ms, gres_ms, d, clk, workload="C2"):
    """Compare roofline of the dominant dominance kernel family (SURVEY.md
    §8(d)): R = N_SM * f_clk * L_pipe / I_test.  float64 dominance kernels:
    I_test = 2d DSETP on the FP64 pipe (64 lanes/clk/SM); SWAR code kernels
    (gres): 4 ALU ops per test for u32 code words (d <= 4), 8 for u64, on the
    ALU pipe (64 lanes/clk/SM).  f_clk = median SM clock sampled during the
    timed region (else the 1965 MHz max)."""
    f = (clk.get("sm_mhz") or 1965.0) * 1e6

    def one(kind):
        if kind == "gres" and st["gres_engine"] == 2 and st["gres_cells"] == 0:
            # small-grid cell engine: all steps in one launch, grids in shared
            # memory — no HBM sweeps, no pair tests: launch-latency bound
            return {"bound": "latency", "kernel": "k_cells_smem", "achieved": None,
                    "peak": None, "unit": None, "frac": None, "traffic": None,
                    "kernel_ms_per_step": gres_ms,
                    "launches_per_step": st["gres_kernel_launches"]}
        if kind == "gres" and st["gres_engine"] == 2:  # cell-occupancy engine: HBM sweeps
            ms = gres_ms
            byts = st["gres_cells"]
            achieved = byts / (ms / 1e3) if ms > 0 else 0.0
            peak = HBM_PEAK_GBS * 1e9
            tr = kernel_traffic(workload, "cells_engine_per_call")
            return {"bound": "hbm", "kernel": "min-grid cell engine (k_mg_*, k_cells_codes)",
                    "achieved": achieved / 1e9, "peak": peak / 1e9, "unit": "GB/s",
                    "frac": achieved / peak, "traffic": tr,
                    "traffic_unit": "B/call, all cell-engine kernels (ncu dram read+write, profiles/r02_launches_C5_v6.md)",
                    "algorithmic_bytes_per_step": byts, "kernel_ms_per_step": ms,
                    "launches_per_step": st["gres_kernel_launches"],
                    "bytes_model": "codes: S*d*8 B read + S*8 B per scanned step written; per step: the "
                                   "byte grid written once, read + written once by an ideal fused "
                                   "prefix minimum (3 x grid bytes), the S code words read twice"}
        if kind == "skyline" and st["sky_engine"] == 16 and st.get("sky_units"):
            # rank-grid engine, TMA bitset decide kernel (skyline_grid.cu K6): one
            # unit = one staged comparator tested against a 128-candidate item =
            # D 16-byte candidate-bitset table reads; the shared-memory pipe
            # (128 B/clk/SM) bounds it: peak = 148 * f * 128 / (16 D) units/s
            units, ms, launches = st["sky_units"], sky_ms, st["sky_kernel_launches"]
            peak = 148 * f * 128.0 / (16.0 * d)
            achieved = units / (ms / 1e3) if ms > 0 else 0.0
            return {"bound": "shared-memory pipe", "kernel": "k_grid_decide_tma",
                    "achieved": achieved / 1e9, "peak": peak / 1e9, "unit": "G comparator-item tests/s",
                    "frac": achieved / peak, "traffic": kernel_traffic(workload, "k_grid_decide"),
                    "traffic_unit": "B/launch (ncu dram read+write)", "units_per_step": units,
                    "tests_per_step": st["skyline_tests"], "kernel_ms_per_step": ms,
                    "launches_per_step": launches, "bytes_smem_per_unit": 16 * d,
                    "smem_bytes_per_clk_sm": 128, "f_clk_mhz": f / 1e6,
                    "dominance_tests_per_s": st["skyline_tests"] / (ms / 1e3) / 1e9 if ms > 0 else 0.0,
                    # the (live candidate, comparator) decisions against what a
                    # per-pair SWAR kernel could do at best (3 ALU ops per test
                    # on the 64-lane ALU pipe, the round-1 k_grid_decide model)
                    "compare_roofline_equiv": {
                        "peak_gtests_s": 148 * f * 64 / 3.0 / 1e9,
                        "frac": (st["skyline_tests"] / (ms / 1e3)) / (148 * f * 64 / 3.0) if ms > 0 else 0.0}}
        if kind == "skyline" and st["sky_engine"] == 16:  # rank-grid engine (skyline_grid.cu)
            tests, ms, launches = st["skyline_tests"], sky_ms, st["sky_kernel_launches"]
            i_test, l_pipe = 3, 64  # IADD3 + LOP3 + VIMNMX on the ALU pipe (+ IMAD.X, FMA pipe)
            peak = 148 * f * l_pipe / i_test
            achieved = tests / (ms / 1e3) if ms > 0 else 0.0
            return {"bound": "compare", "kernel": "k_grid_decide", "achieved": achieved / 1e9,
                    "peak": peak / 1e9, "unit": "Gtests/s", "frac": achieved / peak,
                    "traffic": kernel_traffic(workload, "k_grid_decide"),
                    "traffic_unit": "B/launch (ncu dram read+write)",
                    "tests_per_step": tests, "kernel_ms_per_step": ms, "launches_per_step": launches,
                    "I_test": i_test, "L_pipe": l_pipe, "pipe": "alu", "f_clk_mhz": f / 1e6}
        if kind == "gres":
            # gres.cu: the resident pair kernel up to 2^21 skyline tuples, tiled beyond
            kern = ("k_gres_pairs_resident" if st["skyline_size"] <= (1 << 21) else
                    "k_gres_pairs_tiled") if st["code_bits"] == 8 else "k_gres_pairs_f64"
            tests, ms, launches = st["gres_tests"], gres_ms, st["gres_kernel_launches"]
            if st["code_bits"] == 8:
                i_test, pipe = (4 if d <= 4 else 8), "alu"
            else:
                i_test, pipe = 2 * d, "fp64"
        elif d <= 8:
            # 16-bit quantised SWAR prefilter (one u64 word per 4 attributes):
            # IADD3, IADD3.X, 2 LOP3, 2 ISETP per word on the ALU pipe; the
            # exact float64 test runs only on a code pass
            kern = "k_sfs_intra_smem+k_sfs_filter_q"
            tests, ms, launches = st["skyline_tests"], sky_ms, st["sky_kernel_launches"]
            i_test, pipe = 6 * (1 if d <= 4 else 2), "alu"
        else:
            kern = "k_sfs_intra_sorted+k_sfs_filter_cells"
            tests, ms, launches = st["skyline_tests"], sky_ms, st["sky_kernel_launches"]
            i_test, pipe = 2 * d, "fp64"
        l_pipe = 64
        peak = 148 * f * l_pipe / i_test
        achieved = tests / (ms / 1e3) if ms > 0 else 0.0
        traffic = None
        if launches:
            tr = [kernel_traffic(workload, k) for k in kern.split("+")]
            if all(t is not None for t in tr):
                traffic = sum(tr)
        return {"bound": "compare", "kernel": kern, "achieved": achieved / 1e9,
                "peak": peak / 1e9, "unit": "Gtests/s", "frac": achieved / peak if peak else None,
                "traffic": traffic, "traffic_unit": "B/launch (ncu dram read+write)",
                "tests_per_step": tests, "kernel_ms_per_step": ms, "launches_per_step": launches,
                "I_test": i_test, "L_pipe": l_pipe, "pipe": pipe, "f_clk_mhz": f / 1e6}

    dominant = "gres" if gres_ms > sky_ms else "skyline"
    r = one(dominant)
    r["other"] = one("skyline" if dominant == "gres" else "gres")
    return r


def spawn_ranks(n):
    """bench.py --gpus N run without torchrun: re-launch under
    torch.distributed.run, one rank per GPU, rendezvous on 127.0.0.1; rank 0's
    JSON line is relayed as this process's output."""
    import socket

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default=DEFAULT_WORKLOAD, choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scaling", default=None, choices=["weak", "strong"],
                    help="default: strong for N > 1 (one instance sharded over the ranks)")
    ap.add_argument("--engine", type=int, default=0, help="gres engine: 0 auto, 1 pairs, 2 cells")
    ap.add_argument("--sky-engine", default="auto", choices=["auto", "rounds", "grid"],
                    help="skyline engine (default: chosen after the first prefix round)")
    ap.add_argument("--strategy", default=None, choices=["none", "grid", "angular", "sliced"],
                    help="override the workload's partitioning plan (both arms)")
    ap.add_argument("--partitions", type=int, default=None, help="override the target partitions")
    ap.add_argument("--local-prune", action="store_true",
                    help="the plan's partitions as local-skyline pruning before the merge")
    ap.add_argument("--cpu-repeat", type=int, default=0, help="0: 1 for C5, else 3")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.scaling is None:
        args.scaling = "strong" if args.gpus > 1 else "weak"
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args.gpus)
    if args.strategy or args.partitions:
        gen, n, d, seed, strat, p, cap = WORKLOADS[args.workload]
        WORKLOADS[args.workload] = (gen, n, d, seed, args.strategy or strat, args.partitions or p, cap)
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        return reference_arm(args)
    return our_arm(args)


if __name__ == "__main__":
    sys.exit(main())
