#!/bin/bash
# Builds kernel-shape variants of the library into build/tune/ (tuning aid).
# usage: tools/tune_shapes.sh name:THREADS:ROWS_CONST:UNROLL:ROWS_VAR:TAB_BITS ...
set -e
cd "$(dirname "$0")/.."
CSRC=paper_2407_11349_b200/csrc
for spec in "$@"; do
  IFS=: read name th rows un mb tb <<< "$spec"
  nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -Xptxas -v \
    -DHK_THREADS=$th -DHK_ROWS_CONST=$rows -DHK_ROWS_VAR=$mb -DHK_UNROLL=$un -DHK_TAB_BITS=${tb:-8} \
    -shared $CSRC/hk_kernels.cu $CSRC/hk_capi.cu $CSRC/hk_host.cpp -o build/tune/lib_$name.so \
    2> build/tune/ptxas_$name.log &
done
wait
for spec in "$@"; do
  name=${spec%%:*}
  echo "$name: $(grep -A2 'pair_kernelILb0ELb1ELi0E' build/tune/ptxas_$name.log | grep -oE 'Used [0-9]+ registers|[0-9]+ bytes spill stores' | tr '\n' ' ')"
done
