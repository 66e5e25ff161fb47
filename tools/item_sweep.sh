#!/bin/bash
# Pair-kernel time vs the planner's work-item target (HK_ITEM_TARGET): the
# partial-sum buffer holds ceil(target / row blocks) slots per row.
cd "$(dirname "$0")/.."
for v in 0 1; do
  for tgt in ${TARGETS:-3552 7104 14208 31264}; do
    echo "target=$tgt $(HK_ITEM_TARGET=$tgt python tools/profile_pair.py ${N:-1000000} $v 4 | grep -oE 'variant=[0-9].*' | sed 's/ll=.*wall/wall/')"
  done
done
