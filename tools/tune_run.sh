#!/bin/bash
# Times each build/tune/lib_*.so variant (tuning aid): N=1e5 LL+grad, both variants;
# with PARITY=1 also runs the GPU parity suite against each variant.
cd "$(dirname "$0")/.."
for lib in build/tune/lib_*.so; do
  name=$(basename $lib .so)
  for v in 0 1; do
    echo "$name v=$v $(HK_LIB=$lib python tools/profile_pair.py ${N:-100000} $v 3 | grep -oE 'pair_kernel/launch=[0-9.]+ ms pairs/s=[0-9.e+]+')"
  done
  if [ "${PARITY:-0}" = 1 ]; then
    echo "$name parity: $(HK_LIB=$lib python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -1)"
  fi
done
