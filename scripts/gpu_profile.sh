# launch list + full capture of the top kernels for one workload
W=${W:-C2}
CMD="python bench.py --steps 2 --warmup 3 --workload $W --no-cpu-baseline"
$CMD > gpurun_out/prof_plain_$W.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c ${NLAUNCH:-2000} --csv --log-file gpurun_out/launches_$W.csv $CMD > gpurun_out/ncu_launch_$W.log 2>&1
echo "launch list rc=$?"
for K in ${KERNELS:-k_sfs_filter_warp k_gres_pairs_tiled}; do
  ncu --set full --clock-control none --import-source on -k regex:$K -s ${SKIP:-3} -c 1 -o gpurun_out/prof_${W}_$K -f $CMD > gpurun_out/ncu_full_${W}_$K.log 2>&1
  echo "full $K rc=$?"
done
ls -la gpurun_out/
