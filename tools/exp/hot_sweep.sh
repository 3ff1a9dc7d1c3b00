#!/bin/bash
# replicated hot accumulators: number of hot ranks x copies, rebuilt on the GPU box
VARS=${HOT_VARIANTS:-"64,16 128,16 256,16 64,32 256,8"}
for v in $VARS; do
  set -- ${v/,/ }
  DI_NVCC_DEFS="-DDI_HOT_RANKS=$1 -DDI_HOT_COPIES=$2" python tools/build.py --force > /dev/null 2>&1 || { echo build failed; exit 1; }
  for c in c3 c2 c4; do echo -n "hot $1 copies $2 "; timeout 300 python tools/exp/async.py $c 2>&1 | head -1; done
done
python tools/build.py --force > /dev/null 2>&1
