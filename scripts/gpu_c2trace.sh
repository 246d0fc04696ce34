timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pt_parity.log 2>&1; echo "pt rc=$?"
timeout 300 python bench.py --no-cpu-baseline --workload C2 > gpurun_out/b_C2.log 2>&1
timeout 300 python bench.py --no-cpu-baseline --workload C1 > gpurun_out/b_C1.log 2>&1
ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,sm__cycles_active.max --clock-control none -k regex:k_sfs_intra_smem -c 4 --csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/k4_ncu.csv 2>&1
