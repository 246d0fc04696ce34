# round 2 final: the full GPU suite, one bench line per workload + the reference arm, the C5 launch list
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 2400 python -m pytest tests -m gpu -q -x --durations=12 > gpurun_out/r2final_pytest_gpu.log 2>&1; echo "suite rc=$?"; tail -18 gpurun_out/r2final_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2final_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2final_smoke.log
timeout 900 python bench.py > gpurun_out/r2final_bench_C5.log 2>&1; echo "bench C5 (default, with cpu baseline) rc=$?"; tail -1 gpurun_out/r2final_bench_C5.log | cut -c1-400
WORKLOADS="C1 C2 C3 C4 C5p10k C5p20k" BENCH_ARGS="--no-cpu-baseline" bash scripts/gpu_bench_all.sh
CMD="python bench.py --steps 2 --warmup 3 --workload C5 --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_C5_final.csv $CMD > gpurun_out/ncu_launch_C5.log 2>&1; echo "launch list rc=$?"
