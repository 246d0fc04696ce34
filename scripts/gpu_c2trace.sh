timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pt_all.log 2>&1; echo "pt rc=$?"
for w in C2 C5 C4; do timeout 600 python bench.py --no-cpu-baseline --workload $w > gpurun_out/b_$w.log 2>&1; done
W=C5 bash scripts/gpu_trace.sh
