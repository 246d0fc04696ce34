SKYGPU_TRACE=1 timeout 300 python bench.py --steps 2 --warmup 3 --workload C2 --no-cpu-baseline > gpurun_out/trc2_dev.log 2>&1
