#!/bin/bash
# Build libpgmres variants for tuning studies into paper_1906_04051_b200/_lib/var/<name>/libpgmres.so
# (in-tree .so files travel to the GPU box); run with tools/run_variants.sh.
#   tools/build_variants.sh name1 "-DFLAG=1 ..." name2 "-DFLAG=2" ...
set -e
cd "$(dirname "$0")/.."
mkdir -p paper_1906_04051_b200/_lib/var
while [ $# -gt 0 ]; do
  name=$1; flags=$2; shift 2
  mkdir -p paper_1906_04051_b200/_lib/var/$name
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -lineinfo \
    -Xcompiler -fPIC -shared $flags -o paper_1906_04051_b200/_lib/var/$name/libpgmres.so \
    paper_1906_04051_b200/csrc/pgmres.cu -ldl &
done
wait
