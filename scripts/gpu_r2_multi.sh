timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "step_sharded or nccl or shards or sharded" > gpurun_out/multi_tests.log 2>&1; echo "multi rc=$?"; tail -5 gpurun_out/multi_tests.log
timeout 2000 python -m pytest tests/test_dropin_gpu.py -q -x > gpurun_out/dropin2.log 2>&1; echo "dropin rc=$?"; tail -3 gpurun_out/dropin2.log
