timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pt_all.log 2>&1; echo "pt rc=$?"
for w in C2 C1 C3 C4; do timeout 300 python bench.py --no-cpu-baseline --workload $w > gpurun_out/b_$w.log 2>&1; done
