W=${W:-C5}
CMD="python bench.py --steps 2 --warmup 3 --workload $W --no-cpu-baseline"
$CMD > gpurun_out/prof_plain_$W.log 2>&1; echo "plain rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -c ${NLAUNCH:-3000} --csv --log-file gpurun_out/launches_$W.csv $CMD > gpurun_out/ncu_launch_$W.log 2>&1
echo "launch list rc=$?"
