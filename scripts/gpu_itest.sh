# executed instructions per dominance test of the compare kernels (I_test
# evidence): ncu instruction/pipe counters of one launch + the test count
# the same call reported; SASS of the inner loops is extracted on the CPU
# side (scripts/sass_excerpt.py)
M=smsp__inst_executed.sum,smsp__inst_executed_pipe_alu.sum,smsp__inst_executed_pipe_fma.sum,smsp__inst_executed_pipe_fp64.sum,smsp__inst_executed_pipe_lsu.sum,smsp__inst_executed_pipe_uniform.sum,smsp__inst_executed_pipe_adu.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg
mkdir -p gpurun_out/itest
probe() {  # label workload kernel-regex [engine]
    ncu --metrics $M --clock-control none -k regex:$3 -c 3 --csv python scripts/itest_probe.py $2 $4 > gpurun_out/itest/$1.csv 2> gpurun_out/itest/$1.err
    echo "$1 rc=$?"; grep '^{' gpurun_out/itest/$1.csv | tail -1
}
probe C5_k6 C5 'k_grid_decide' 
probe C2_k5 C2 'k_sfs_(filter_q|intra_smem)'
probe C4_k5 C4 'k_sfs_(filter_q|intra_smem|intra_chunked)'
probe C5p10k_pairs C5p10k 'k_gres_pairs' 1
probe C5p20k_pairs C5p20k 'k_gres_pairs' 1
