# k_cycle: rows of DI_ASYNC_SMALL < links <= DI_ASYNC_MID go to 8-lane groups (int4 loads), longer
# ones to whole warps with lane-consecutive targets (option long_lanes): where should the split be?
mkdir -p gpurun_out
for defs in "-DDI_ASYNC_MID=256" "-DDI_ASYNC_MID=128" "-DDI_ASYNC_MID=64" "-DDI_ASYNC_MID=32"; do
  echo "## $defs"
  DI_NVCC_DEFS="$defs" python tools/build.py --force > gpurun_out/mid_build.log 2>&1 || { echo build failed; tail -5 gpurun_out/mid_build.log; continue; }
  python tools/exp/c4_ab.py warm=-1 warm=0
done
