timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pt_all.log 2>&1; echo "pytest rc=$?"
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/b_c2.log 2>&1; echo "bench rc=$?"
timeout 300 python bench.py --no-cpu-baseline --workload C1 > gpurun_out/b_c1.log 2>&1; echo "bench c1 rc=$?"
SKYGPU_TRACE=1 timeout 300 python scripts/e2e_trace.py ant 1000000 3 > gpurun_out/tr_c2_plain.log 2>&1
