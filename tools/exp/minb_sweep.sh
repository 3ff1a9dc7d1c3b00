#!/bin/bash
# k_cycle occupancy (min blocks per SM of __launch_bounds__) x tile size, rebuilt on the GPU box
VARS=${MINB_VARIANTS:-"4,2 3,2 3,4"}
for v in $VARS; do
  set -- ${v/,/ }
  DI_NVCC_DEFS="-DDI_ASYNC_MINB=$1 -DDI_CYC_ITEMS=$2" python tools/build.py --force > /dev/null 2>&1 || { echo build failed; exit 1; }
  grep -A2 "k_cycleILb0ELb0" paper_1204_6255_b200/ptxas.log | grep -o "[0-9]* bytes spill stores" | head -1
  for c in c4 c3 c2; do echo -n "minb $1 items $2 "; timeout 300 python tools/exp/async.py $c 2>&1 | head -1; done
done
python tools/build.py --force > /dev/null 2>&1
