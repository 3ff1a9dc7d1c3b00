# Warm tier: slots flushed ahead of their node's tile (DI_WARM_AHEAD = window in quarter grids of
# tiles; 0 = at the cycle's end only), C4 bench workload: bash tools/exp/warm_ahead_sweep.sh X1 X2 ...
mkdir -p gpurun_out
for x in "$@"; do
  echo "## DI_WARM_AHEAD=$x"
  DI_NVCC_DEFS="-DDI_WARM_AHEAD=$x" python tools/build.py --force > gpurun_out/wa_build.log 2>&1 || { echo build failed; continue; }
  python tools/exp/c4_ab.py warm=-1 warm=0
done
