timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pt_all.log 2>&1; echo "pt rc=$?"
for w in C3 C2 C1 C4; do timeout 600 python bench.py --no-cpu-baseline --workload $w > gpurun_out/b_$w.log 2>&1; done
SKYGPU_TRACE=1 timeout 300 python bench.py --steps 2 --warmup 3 --workload C3 --no-cpu-baseline > gpurun_out/trc3_new.log 2>&1
