"""Generate the golden fixtures in tests/golden/ by running the UNMODIFIED
reference library (oracle/_ref/refdrive*, built by oracle/build_ref.sh from
/root/reference/proj/src).  Run in the dev container (the reference tree does
not exist on the GPU box):

    oracle/build_ref.sh && python tests/golden/make_golden.py

Each fixture records the input spec (generator + seed, or the literal values)
and the reference outputs: sorted skyline ids, the skyline in the reference's
output order, g_max, the denominators map, and (small cases) the brute-force
skyline / resistance of proj/src/oracle.cpp.
"""
from __future__ import annotations

import gzip
import json
import os
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF_CHK = os.path.join(ROOT, "oracle", "_ref", "refdrive_chk")
REF_REL = os.path.join(ROOT, "oracle", "_ref", "refdrive")


def run(args, release=False):
    exe = REF_REL if release else REF_CHK
    r = subprocess.run([exe] + [str(a) for a in args], capture_output=True, text=True)
    if r.returncode not in (0, 3):
        raise RuntimeError(r.stdout + r.stderr)
    return json.loads(r.stdout)


def save(name, spec, res):
    obj = {"name": name, "spec": spec}
    if "error" in res:
        obj["error"] = res["error"]
    else:
        ids = res["skyline_ids"]
        obj["skyline_ids"] = ids
        obj["skyline_order"] = res["skyline_order"]
        if "gres_error" in res:
            obj["gres_error"] = res["gres_error"]
        if "g_max" in res:
            den = dict((int(a), int(b)) for a, b in res["den"])
            obj["g_max"] = res["g_max"]
            obj["den"] = [den[i] for i in ids]
            obj["rows"] = res["rows"]
        if "bruteforce_ids" in res:
            obj["bruteforce_ids"] = res["bruteforce_ids"]
        if "bruteforce_den" in res:
            bd = dict((int(a), int(b)) for a, b in res["bruteforce_den"])
            obj["bruteforce_den"] = [bd[i] for i in ids]
    path = os.path.join(HERE, name + ".json.gz")
    with gzip.open(path, "wt") as f:
        json.dump(obj, f, separators=(",", ":"))
    print(f"{name}: S={len(obj.get('skyline_ids', []))} g_max={obj.get('g_max')} "
          f"{'ERROR ' + obj['error'] if 'error' in obj else ''}", flush=True)


def literal_case(name, rows, strategy="none", p=1, cap=25, brute=True, cores=1):
    vals = np.asarray(rows, dtype=np.float64)
    n, d = vals.shape
    with tempfile.NamedTemporaryFile(suffix=".bin", delete=False) as f:
        f.write(vals.tobytes())
        path = f.name
    spec = {"kind": "literal", "values": [[float(x) for x in r] for r in vals], "n": n, "d": d,
            "strategy": strategy, "p": p, "cap": cap, "reps": 0}
    args = ["--input", path, "--n", n, "--d", d, "--strategy", strategy, "--p", p, "--cap", cap,
            "--cores", cores]
    if brute:
        args.append("--brute")
    try:
        save(name, spec, run(args))
    finally:
        os.unlink(path)


def gen_case(name, gen, n, d, seed, strategy="none", p=1, cap=25, reps=0, brute=False,
             release=False, cores=4):
    spec = {"kind": "gen", "gen": gen, "n": n, "d": d, "seed": seed, "strategy": strategy, "p": p,
            "cap": cap, "reps": reps}
    args = ["--gen", gen, "--n", n, "--d", d, "--seed", seed, "--strategy", strategy, "--p", p,
            "--cap", cap, "--reps", reps, "--cores", cores]
    if brute:
        args.append("--brute")
    save(name, spec, run(args, release=release))


def main(which):
    if which in ("all", "small"):
        # known-answer tests of the reference's own suites
        literal_case("kat_three_tuple", [[1, 2], [2, 3], [2, 1]])            # test_core.cpp:61-68
        literal_case("kat_two_tuple", [[0.30, 0.62], [0.32, 0.58]])         # test_gres.cpp:99-106
        literal_case("kat_singleton", [[0.5, 0.5]])                          # test_gres.cpp:91-97
        literal_case("kat_collide_uncapped", [[0.30, 0.40], [0.40, 0.30]], cap=0)  # :163-170
        literal_case("kat_identical", [[1, 1], [1, 1]])                      # test_core.cpp:84-90
        literal_case("kat_fp_tie", [[2e-20, 1.0], [1e-20, 1.0]])
        literal_case("kat_negzero", [[-0.0, 0.5], [0.0, 0.5], [0.25, -0.0], [0.5, 0.25],
                                     [-0.0, -0.0], [0.0, 0.0]])
        rng = np.random.default_rng(11)
        lit = np.vstack([[0.0, 0.0], 0.01 + 0.9 * rng.random((40, 2))])     # test_core.cpp:70-82
        literal_case("kat_origin", lit.tolist())
        # unnormalised values: f64 projection path (codes > 127)
        big = (np.floor(rng.random((300, 3)) * 4000) / 16.0)
        literal_case("big_values_f64", big.tolist(), cap=25)
        # huge values: projected sums tie -> exact (psum, id) order path
        base = 1e15
        huge = base + np.floor(rng.random((60, 3)) * 40) * 0.125
        literal_case("huge_values_ties", huge.tolist(), cap=25, strategy="sliced", p=4)
        # Grid on data outside [0,1] -> the reference's invalid_argument text
        literal_case("grid_out_of_range", [[0.2, 0.3], [0.4, 1.5], [2.0, 0.1]], strategy="grid",
                     p=4, brute=False)
        # seeded random relations across strategies (acceptance-style)
        k = 0
        for gen in ("uni", "ant", "lattice"):
            for d in (2, 3, 4, 5, 7):
                for n in (50, 400, 1500):
                    strat = ["none", "grid", "angular", "sliced"][k % 4]
                    p = [4, 16][k % 2]
                    gen_case(f"rand_{gen}_n{n}_d{d}_{strat}", gen, n, d, 100 + k, strategy=strat,
                             p=p, brute=(n <= 400), cores=2)
                    k += 1
        for gen, d in (("lattice", 2), ("lattice", 3)):
            gen_case(f"uncapped_{gen}_d{d}", gen, 300, d, 77, cap=0, brute=True)
        gen_case("reps10_ant_d3", "ant", 2000, 3, 5, strategy="angular", p=16, reps=10)
        gen_case("reps1_uni_d4", "uni", 2000, 4, 6, strategy="grid", p=16, reps=1)
    if which in ("all", "configs"):
        gen_case("C1_uni_100k_d4", "uni", 100000, 4, 1, release=True, cores=8)
        gen_case("C1_uni_100k_d4_sliced16", "uni", 100000, 4, 1, strategy="sliced", p=16,
                 release=True, cores=8)
        gen_case("C2_ant_1M_d3", "ant", 1000000, 3, 1, strategy="angular", p=16, release=True,
                 cores=8)
        gen_case("C3_corr_1M_d6", "corr", 1000000, 6, 1, release=True, cores=8)
        gen_case("C5_prefix_2k_d7", "ant", 2000, 7, 1, strategy="angular", p=64, release=True,
                 cores=8)
        gen_case("C5_prefix_10k_d7", "ant", 10000, 7, 1, strategy="angular", p=64, release=True,
                 cores=8)
    if which in ("all", "big"):
        gen_case("C4_uni_10M_d5", "uni", 10000000, 5, 1, strategy="angular", p=64, release=True,
                 cores=8)
    if which in ("all", "big", "big2"):
        # config 4 names all three plans at target 64 (grid -> m=2, p=32;
        # sliced -> 64; angular above); the reference's plan invariance
        # (acceptance_main.cpp:145-184) says the answers agree — pinned here
        # through the reference itself for each plan
        gen_case("C4_uni_10M_d5_grid64", "uni", 10000000, 5, 1, strategy="grid", p=64,
                 release=True, cores=8)
        gen_case("C4_uni_10M_d5_sliced64", "uni", 10000000, 5, 1, strategy="sliced", p=64,
                 release=True, cores=8)
        # the C5 stream's 20k prefix (the reference arm's bench sample)
        gen_case("C5_prefix_20k_d7", "ant", 20000, 7, 1, strategy="angular", p=64, release=True,
                 cores=8)
    if which in ("all", "pids"):
        # the reference's own assign_partitions (partition.cpp:183-213) on
        # seeded inputs: golden ids for the device assign_partitions and the
        # oracle's restatement (one file, all cases)
        cases = []
        for gen, n, d, strat, p, seed in (
                ("uni", 3000, 2, "grid", 16, 21), ("uni", 3000, 5, "grid", 64, 22),
                ("ant", 3000, 7, "grid", 64, 23), ("lattice", 3000, 3, "grid", 64, 24),
                ("uni", 3000, 2, "angular", 16, 31), ("ant", 3000, 3, "angular", 16, 32),
                ("uni", 3000, 5, "angular", 64, 33), ("ant", 3000, 7, "angular", 64, 34),
                ("lattice", 3000, 4, "angular", 81, 35),
                ("uni", 3000, 3, "sliced", 16, 41), ("ant", 3000, 7, "sliced", 64, 42),
                ("lattice", 3000, 2, "sliced", 7, 43), ("lattice", 3000, 5, "sliced", 100, 44),
                ("uni", 2999, 4, "none", 1, 51)):
            r = run(["--mode", "pids", "--gen", gen, "--n", n, "--d", d, "--seed", seed,
                     "--strategy", strat, "--p", p])
            cases.append(r)
            print(f"pids {gen} n={n} d={d} {strat} p={p}: partitions={r['partitions']} "
                  f"distinct={len(set(r.get('pids', [])))}", flush=True)
        with gzip.open(os.path.join(HERE, "partition", "pids_cases.json.gz"), "wt") as f:
            json.dump({"name": "pids_cases", "cases": cases}, f, separators=(",", ":"))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "all")
