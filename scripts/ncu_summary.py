#!/usr/bin/env python
"""Summarise ncu output for profiles/: the launch list (per-kernel share of a
step) and full captures (duration, DRAM traffic, throughput, occupancy,
stall reasons).

    python scripts/ncu_summary.py [--traffic C2] gpurun_out/launches_C2.csv gpurun_out/prof_C2_*.ncu-rep > profiles/rNN_ncu_C2.md

--traffic W merges the captures' DRAM bytes per kernel into profiles/traffic.json
(read by bench.py for roofline.traffic).
"""
import collections
import csv
import io
import subprocess
import sys


def launch_list(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h, data = rows[hi], rows[hi + 1:]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    names = [r[ki] for r in data]
    # one step = the launches between the last two k_score launches of the
    # device-timed phase (bench runs warm-up + steps, then the e2e phase)
    starts = [i for i, n in enumerate(names) if "k_score" in n]
    s, e = (starts[-3], starts[-2]) if len(starts) >= 3 else (0, len(names))
    agg = collections.OrderedDict()
    tot = 0.0
    for r in data[s:e]:
        n = r[ki].split("(")[0].replace("void ", "")
        n = n.replace("skygpu::", "").replace("<unnamed>::", "")[:70]
        v = float(r[vi].replace(",", "")) / 1e3
        a = agg.setdefault(n, [0, 0.0])
        a[0] += 1
        a[1] += v
        tot += v
    out = ["| kernel | launches/step | us/step (ncu, serialised) | share |", "|---|---|---|---|"]
    for n, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"| `{n}` | {c} | {v:.1f} | {100 * v / tot:.1f}% |")
    out.append(f"| **total** | {sum(c for c, _ in agg.values())} | {tot:.1f} | 100% |")
    return "\n".join(out)


WANT = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "memory throughput %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("sm__inst_executed.sum", "warp instructions"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
]


def full_capture(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    if len(rows) < 3:
        return f"(no data in {path})"
    h, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "")
        name = name.replace("skygpu::", "").replace("<unnamed>::", "")
        out.append(f"#### `{name}`  ({path.split('/')[-1]})\n")
        out.append("| metric | value |\n|---|---|")
        for key, label in WANT:
            if key in h:
                i = h.index(key)
                out.append(f"| {label} (`{key}`) | {r[i]} {units[i]} |")
        stalls = [(h[i], r[i]) for i in range(len(h))
                  if h[i].startswith("smsp__average_warp_latency_issue_stalled_")
                  or h[i].startswith("smsp__pcsamp_warps_issue_stalled_")]
        vals = []
        for k, v in stalls:
            try:
                vals.append((float(v.replace(",", "")), k))
            except ValueError:
                pass
        vals.sort(reverse=True)
        if vals:
            out.append("\nTop stall reasons: " + ", ".join(
                f"{k.split('stalled_')[-1]}={v:g}" for v, k in vals[:6]))
        out.append("")
    return "\n".join(out)


def traffic(path):
    """{kernel base name: dram read+write bytes} of a full capture"""
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    out = {}
    if len(rows) < 3:
        return out
    h, units = rows[0], rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for r in rows[2:]:
        name = r[h.index("Kernel Name")].split("(")[0].split("<")[0].split("::")[-1]
        tot = 0.0
        for key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = h.index(key)
            tot += float(r[i].replace(",", "")) * scale.get(units[i], 1)
        out[name] = tot
    return out


def main():
    import json
    import os
    parts = []
    args = sys.argv[1:]
    workload = None
    if args and args[0] == "--traffic":
        workload, args = args[1], args[2:]
    if workload:
        tf = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                          "traffic.json")
        data = json.load(open(tf)) if os.path.exists(tf) else {}
        for p in args:
            if p.endswith(".ncu-rep"):
                data.setdefault(workload, {}).update(traffic(p))
        json.dump(data, open(tf, "w"), indent=1, sort_keys=True)
    for p in args:
        if p.endswith(".csv"):
            parts.append("### Launch list (one step)\n\n" + launch_list(p) + "\n")
        elif p.endswith(".ncu-rep"):
            parts.append(full_capture(p))
    print("\n".join(parts))


if __name__ == "__main__":
    main()
