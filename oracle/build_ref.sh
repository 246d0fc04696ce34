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
