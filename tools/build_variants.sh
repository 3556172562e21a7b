#!/bin/bash
# Build libpgmres variants for tuning studies into tools/variants/<name>/libpgmres.so
set -e
cd "$(dirname "$0")/.."
rm -rf tools/variants
mkdir -p tools/variants
build() {
  name=$1; shift
  mkdir -p tools/variants/$name
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -lineinfo \
    -Xcompiler -fPIC -shared "$@" -o tools/variants/$name/libpgmres.so \
    paper_1906_04051_b200/csrc/pgmres.cu -ldl &
}
build m3 -DPGM_SPMV_MINB=3
build m4 -DPGM_SPMV_MINB=4
build m5 -DPGM_SPMV_MINB=5
build m4u8 -DPGM_SPMV_MINB=4 -DPGM_SPMV_UNROLL=8
wait
