# A/B: the working tree's libskygpu vs ab/libskygpu_head.so (HEAD build)
for w in ${WS:-C3 C2}; do for i in 1 2; do
timeout 600 python bench.py --no-cpu-baseline --workload $w > gpurun_out/ab_new_${w}_$i.log 2>&1
SKYGPU_LIB_PATH=$PWD/ab/libskygpu_head.so timeout 600 python bench.py --no-cpu-baseline --workload $w > gpurun_out/ab_head_${w}_$i.log 2>&1
done; done
