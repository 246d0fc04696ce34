timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pt_parity.log 2>&1; echo "pt rc=$?"
for w in C2 C4 C1 C3; do timeout 600 python bench.py --no-cpu-baseline --workload $w > gpurun_out/b_$w.log 2>&1; done
