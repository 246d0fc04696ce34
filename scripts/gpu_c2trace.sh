for i in 1 2; do
timeout 300 python scripts/e2e_trace.py ant 1000000 3 > gpurun_out/t_c2_plain_$i.log 2>&1
SKYGPU_STREAM_MIN_MB=8 timeout 300 python scripts/e2e_trace.py ant 1000000 3 > gpurun_out/t_c2_stream_$i.log 2>&1
done
SKYGPU_STREAM_MIN_MB=8 SKYGPU_TRACE=1 timeout 300 python scripts/e2e_trace.py ant 1000000 3 > gpurun_out/tr_c2_stream.log 2>&1
timeout 300 python scripts/e2e_trace.py uni 100000 4 > gpurun_out/t_c1_plain.log 2>&1
timeout 300 python scripts/e2e_trace.py corr 1000000 6 > gpurun_out/t_c3_plain.log 2>&1
SKYGPU_STREAM_MIN_MB=1000 timeout 300 python scripts/e2e_trace.py corr 1000000 6 > gpurun_out/t_c3_nostream.log 2>&1
