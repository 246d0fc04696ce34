W=${W:-C2}
SKYGPU_TRACE=1 python bench.py --steps 2 --warmup 3 --workload $W --no-cpu-baseline > gpurun_out/trace_$W.log 2>&1
echo rc=$?
