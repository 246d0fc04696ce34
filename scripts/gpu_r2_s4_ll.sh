CMD="python bench.py --steps 2 --warmup 3 --workload C5 --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_C5_final.csv $CMD > gpurun_out/ncu_launch_C5.log 2>&1; echo "launch list rc=$?"
