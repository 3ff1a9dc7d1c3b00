# k_cycle long rows (lane-consecutive): column loads in flight per lane, software pipelining
mkdir -p gpurun_out
for defs in "-DDI_LL_BATCH=8" "-DDI_LL_PIPE=1" "-DDI_LL_BATCH=16" "-DDI_LL_BATCH=4 -DDI_LL_PIPE=1" "-DDI_LL_BATCH=16 -DDI_LL_PIPE=1"; do
  echo "## $defs"
  DI_NVCC_DEFS="$defs" python tools/build.py --force > gpurun_out/ll_build.log 2>&1 || { echo build failed; continue; }
  python tools/exp/c4_ab.py warm=-1
done
