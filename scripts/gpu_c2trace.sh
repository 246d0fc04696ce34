timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pt_all.log 2>&1; echo "pt rc=$?"
for w in C2 C4 C5 C3; do timeout 600 python bench.py --no-cpu-baseline --workload $w > gpurun_out/b_$w.log 2>&1; done
SKYGPU_IDS_LATE=0 timeout 600 python bench.py --no-cpu-baseline --workload C4 > gpurun_out/b_C4_noids.log 2>&1
SKYGPU_IDS_LATE=0 timeout 600 python bench.py --no-cpu-baseline --workload C5 > gpurun_out/b_C5_noids.log 2>&1
