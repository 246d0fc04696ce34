timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pt_all.log 2>&1; echo "pt rc=$?"
for i in 1 2; do
timeout 300 python bench.py --no-cpu-baseline --workload C2 > gpurun_out/b_C2_$i.log 2>&1
SKYGPU_IDS_LATE=0 timeout 300 python bench.py --no-cpu-baseline --workload C2 > gpurun_out/b_C2_noids_$i.log 2>&1
done
timeout 300 python bench.py --no-cpu-baseline --workload C1 > gpurun_out/b_C1.log 2>&1
timeout 300 python bench.py --no-cpu-baseline --workload C3 > gpurun_out/b_C3.log 2>&1
SKYGPU_TRACE=1 timeout 300 python scripts/e2e_trace.py ant 1000000 3 > gpurun_out/tr_c2_plain.log 2>&1
