# full ncu captures of the min-grid cell engine's step-0 (g = 25) kernels on C5
for K in k_mg_slabcol k_mg_pair k_mg_mark k_mg_query k_mg_fill; do
  ncu --set full --import-source on --clock-control none -k regex:$K -c 1 -o gpurun_out/prof_C5_$K -f python scripts/itest_probe.py C5 > gpurun_out/ncu_full_$K.log 2>&1
  echo "$K rc=$?"
done
