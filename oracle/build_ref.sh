#!/usr/bin/env bash
# Compile the UNMODIFIED reference library from its own sources where they lie
# (/root/reference/proj/src) into oracle/_ref/ — test/baseline infrastructure
# only (see oracle/README.md).  Nothing here copies reference sources; outputs
# go only to oracle/_ref/ (git-ignored, but it travels to the GPU box).
#
#   chk : the reference's default build (-O2 -g, contract checks ON, i.e. no
#         NDEBUG; proj/CMakeLists.txt:8-11) -> parity goldens
#   rel : Release-equivalent (-O3 -DNDEBUG) -> the CPU baseline timer
#
# Both with OpenMP (proj/src/CMakeLists.txt:12-14) and -ffp-contract=off
# (the reference is built without -march, so x86-64 never contracts; this
# keeps that true if CXXFLAGS ever gain -march).
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
REF="${REF_ROOT:-/root/reference/proj}"
OUT="$HERE/_ref"
JSON_INC="${JSON_INC:-/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann}"
if [ ! -d "$REF/src" ]; then
  echo "build_ref: reference sources not present at $REF (GPU box?) — skipping" >&2
  exit 0
fi
mkdir -p "$OUT/chk" "$OUT/rel"
SRCS="core oracle partition parallel gres datagen metrics harness"
CXX="${SKY_CXX:-/usr/bin/g++}"
COMMON="-std=c++20 -fPIC -fopenmp -ffp-contract=off -I$REF/include -I$JSON_INC -w"
build_variant() {
  local v="$1"; shift
  local flags="$*"
  local objs=()
  for s in $SRCS; do
    local o="$OUT/$v/$s.o"
    if [ ! -f "$o" ] || [ "$REF/src/$s.cpp" -nt "$o" ]; then
      $CXX $COMMON $flags -c "$REF/src/$s.cpp" -o "$o" &
    fi
    objs+=("$o")
  done
  wait
  rm -f "$OUT/libskypar_$v.a"
  ar rcs "$OUT/libskypar_$v.a" "${objs[@]}"
}
build_variant chk -O2 -g
build_variant rel -O3 -DNDEBUG
$CXX $COMMON -O2 -I"$REF/include" "$HERE/refdrive.cpp" "$OUT/libskypar_chk.a" -o "$OUT/refdrive_chk"
$CXX $COMMON -O3 -DNDEBUG -I"$REF/include" "$HERE/refdrive.cpp" "$OUT/libskypar_rel.a" -o "$OUT/refdrive"
echo "build_ref: ok -> $OUT"

# ---- drop-in link test: the reference's acceptance suite and library objects
# with parallel.o and gres.o REPLACED by the GPU adapter
ROOT="$(cd "$HERE/.." && pwd)"
LIBDIR="$ROOT/paper_2412_02274_b200/_lib"
if [ -f "$LIBDIR/libskygpu.so" ]; then
  for v in chk rel; do
    if [ "$v" = chk ]; then VF="-O2 -g"; else VF="-O3 -DNDEBUG"; fi
    $CXX $COMMON $VF -I"$ROOT/include" -c "$ROOT/paper_2412_02274_b200/adapter/skypar_gpu.cpp" \
        -o "$OUT/$v/skypar_gpu.o"
    rm -f "$OUT/libskypar_gpu_$v.a"
    ar rcs "$OUT/libskypar_gpu_$v.a" "$OUT/$v/core.o" "$OUT/$v/oracle.o" "$OUT/$v/partition.o" \
        "$OUT/$v/datagen.o" "$OUT/$v/metrics.o" "$OUT/$v/harness.o" "$OUT/$v/skypar_gpu.o"
  done
  RPATH="-Wl,-rpath,\$ORIGIN/../../paper_2412_02274_b200/_lib"
  $CXX $COMMON -O2 "$REF/tests/acceptance_main.cpp" "$OUT/libskypar_gpu_chk.a" -L"$LIBDIR" -lskygpu \
      $RPATH -o "$OUT/acceptance_gpu"
  $CXX $COMMON -O2 "$REF/tests/acceptance_main.cpp" "$OUT/libskypar_chk.a" -o "$OUT/acceptance_ref"
  $CXX $COMMON -O3 -DNDEBUG -I"$REF/include" "$HERE/refdrive.cpp" "$OUT/libskypar_gpu_rel.a" \
      -L"$LIBDIR" -lskygpu $RPATH -o "$OUT/refdrive_gpu"
  # the reference's own tools, UNMODIFIED (proj/tools/skypar_main.cpp and
  # bench_main.cpp), compiled against an original CLI11-subset header
  # (adapter/cli11_subset/CLI11.hpp; the real CLI11 is not vendored) — over
  # the GPU drop-in and over the CPU library, in the reference's default
  # (checked) build
  CLI_INC="-I$ROOT/paper_2412_02274_b200/adapter/cli11_subset"
  $CXX $COMMON -O2 -g $CLI_INC "$REF/tools/skypar_main.cpp" "$OUT/libskypar_gpu_chk.a" \
      -L"$LIBDIR" -lskygpu $RPATH -o "$OUT/skypar_gpu"
  $CXX $COMMON -O2 -g $CLI_INC "$REF/tools/skypar_main.cpp" "$OUT/libskypar_chk.a" -o "$OUT/skypar_ref"
  $CXX $COMMON -O2 -g $CLI_INC "$REF/tools/bench_main.cpp" "$OUT/libskypar_gpu_chk.a" \
      -L"$LIBDIR" -lskygpu $RPATH -o "$OUT/skypar_bench_gpu"
  $CXX $COMMON -O2 -g $CLI_INC "$REF/tools/bench_main.cpp" "$OUT/libskypar_chk.a" \
      -o "$OUT/skypar_bench_ref"
  # the CLI-determinism fixtures (acceptance criterion 9) travel with the
  # binaries; /root/reference does not exist on the GPU box
  mkdir -p "$OUT/fixtures"
  cp "$REF/data/fixtures/"*.csv "$OUT/fixtures/"
  echo "build_ref: drop-in binaries ok (acceptance_gpu, refdrive_gpu, skypar_gpu, skypar_ref)"
fi
