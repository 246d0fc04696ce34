"""Instructions per dominance test from scripts/gpu_itest.sh output:
python scripts/itest_summary.py gpurun_out/itest/*.csv"""
import collections
import csv
import io
import json
import sys

for path in sys.argv[1:]:
    txt = open(path).read()
    stats = [json.loads(l) for l in txt.splitlines() if l.startswith("{")]
    body = "\n".join(l for l in txt.splitlines() if l.startswith('"'))
    rows = list(csv.reader(io.StringIO(body)))
    h, data = rows[0], rows[1:]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per = collections.OrderedDict()
    for r in data:
        k = (r[ii], r[ki].split("(")[0].replace("void ", ""))
        per.setdefault(k, {})[r[mi]] = float(r[vi].replace(",", ""))
    st = stats[-1] if stats else {}
    print(f"## {path.split('/')[-1]}  {json.dumps(st)}")
    agg = collections.OrderedDict()
    for (i, k), m in per.items():
        a = agg.setdefault(k, collections.Counter())
        for n, v in m.items():
            a[n] += v
        a["launches"] += 1
    for k, m in agg.items():
        print(f"  {k}: launches={m['launches']:.0f} time_us={m['gpu__time_duration.sum']/1e3:.1f}"
              f" inst={m['smsp__inst_executed.sum']:.4g} alu={m['smsp__inst_executed_pipe_alu.sum']:.4g}"
              f" fma={m['smsp__inst_executed_pipe_fma.sum']:.4g} fp64={m['smsp__inst_executed_pipe_fp64.sum']:.4g}"
              f" lsu={m['smsp__inst_executed_pipe_lsu.sum']:.4g} shared_wavefronts={m['l1tex__data_pipe_lsu_wavefronts_mem_shared.sum']:.4g}"
              f" alu_busy%={m['sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active']/m['launches']:.1f}"
              f" issue%={m['smsp__issue_active.avg.pct_of_peak_sustained_active']/m['launches']:.1f}"
              f" dram_MB={(m['dram__bytes_read.sum']+m['dram__bytes_write.sum'])/1e6:.1f}")
    print()
