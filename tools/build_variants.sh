#!/bin/bash
# Build libpovar variants with extra -D flags into build_ab/libpovar_<name>.so.
# Usage: tools/build_variants.sh "name1:-DA=1 -DB=2" "name2:-DC=3" ...
set -e
cd "$(dirname "$0")/.."
mkdir -p build_ab build
[ -f build/pv_bal.o ] || make build/pv_bal.o
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC \
    -Xcompiler -O3 --expt-relaxed-constexpr $flags -shared -o build_ab/libpovar_$name.so \
    paper_2405_05079_b200/csrc/povar.cu build/pv_bal.o -lnccl -Xcompiler -pthread &
done
wait
ls -la build_ab
