# full ncu capture of K6 on C5 (source-level sampling: read here with scripts/ncu_lines.py)
python scripts/c5_sky_dump.py /tmp/x.npy > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_grid_decide_tma -s 1 -c 1 -o gpurun_out/prof_C5_k6 -f python scripts/c5_sky_dump.py /tmp/x.npy > gpurun_out/ncu_k6.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/ncu_k6.log; ls -la gpurun_out/prof_C5_k6.ncu-rep
