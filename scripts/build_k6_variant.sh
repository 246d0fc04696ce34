#!/bin/bash
# build a variant of the rank-grid TU beside the in-tree library, e.g. the K6 watchdog build
# (scripts/build_k6_variant.sh dbg -DSKYGPU_K6_WATCHDOG: a wait that never completes prints its
# site and traps); run with SKYGPU_LIB_PATH=.../_lib_v/NAME/libskygpu.so
# -> paper_2412_02274_b200/_lib_v/NAME/libskygpu.so (the other objects are the in-tree build's)
set -e
name=$1; shift
root=$(cd "$(dirname "$0")/.." && pwd)
out=$root/paper_2412_02274_b200/_lib_v/$name
mkdir -p $out
cd $root/paper_2412_02274_b200/csrc
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC \
  -Xcompiler -ffp-contract=off -I ../../include -I . --expt-relaxed-constexpr -Xptxas -v "$@" \
  -c ${SRC:-skyline_grid.cu} -o $out/skyline_grid.cu.o 2> $out/ptxas.log
grep -A2 "k_grid_decide_tmaILi7" $out/ptxas.log | grep -E "registers|spill" | sed "s/^/[$name] /"
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libskygpu.so $out/skyline_grid.cu.o \
  $(ls $root/paper_2412_02274_b200/_lib/*.o | grep -v skyline_grid) -lcudart -ldl
