#!/bin/bash
# Density-scaled trigger shape sweep (tuning aid): builds variants with
# HK_ROWS_VAR rows per thread and HK_MIN_BLOCKS_TRIG resident CTAs into
# build/tune/, then (on a GPU box, RUN=1) times the bench and county catalogs.
#   tools/tune_trig.sh name:ROWS_VAR:MIN_BLOCKS_TRIG ...
cd "$(dirname "$0")/.."
CSRC=paper_2407_11349_b200/csrc
mkdir -p build/tune
if [ "${RUN:-0}" != 1 ]; then
  for spec in "$@"; do
    IFS=: read name rv mb <<< "$spec"
    nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -Xptxas -v \
      -DHK_ROWS_VAR=$rv -DHK_MIN_BLOCKS_TRIG=$mb -shared $CSRC/hk_kernels.cu $CSRC/hk_capi.cu \
      $CSRC/hk_regions.cu $CSRC/hk_fgt.cu $CSRC/hk_cells.cu $CSRC/hk_host.cpp -o build/tune/lib_$name.so \
      2> build/tune/ptxas_$name.log &
  done
  wait
  for spec in "$@"; do
    name=${spec%%:*}
    echo "$name: $(grep -A2 'pair_kernelILb1ELb1ELi1ELb0ELi2E' build/tune/ptxas_$name.log | grep -oE 'Used [0-9]+ registers|[0-9]+ bytes spill stores' | tr '\n' ' ')"
  done
else
  for spec in "$@"; do
    name=${spec%%:*}
    for c in "" county; do
      echo "$name $c: $(HK_LIB=build/tune/lib_$name.so python tools/profile_pair.py 1000000 1 3 $c | grep -oE '\[.*\]')"
    done
  done
fi
