for i in 1 2 3; do
timeout 300 python bench.py --no-cpu-baseline --workload C2 > gpurun_out/b_spec_$i.log 2>&1
SKYGPU_NO_SPEC_FINAL=1 timeout 300 python bench.py --no-cpu-baseline --workload C2 > gpurun_out/b_nospec_$i.log 2>&1
done
