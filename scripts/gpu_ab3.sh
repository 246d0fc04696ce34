SKYGPU_TRACE=1 timeout 300 python bench.py --steps 2 --warmup 3 --workload C3 --no-cpu-baseline > gpurun_out/trc3_new.log 2>&1
SKYGPU_LIB_PATH=$PWD/ab/libskygpu_head.so SKYGPU_TRACE=1 timeout 300 python bench.py --steps 2 --warmup 3 --workload C3 --no-cpu-baseline > gpurun_out/trc3_head.log 2>&1
