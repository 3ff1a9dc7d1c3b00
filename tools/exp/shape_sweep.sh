mkdir -p gpurun_out
for defs in "-DDI_ASYNC_THREADS=512 -DDI_CYC_ITEMS=1 -DDI_ASYNC_MINB=2" "-DDI_ASYNC_THREADS=512 -DDI_CYC_ITEMS=2 -DDI_ASYNC_MINB=2" "-DDI_ASYNC_THREADS=1024 -DDI_CYC_ITEMS=1 -DDI_ASYNC_MINB=1" "-DDI_ASYNC_THREADS=256 -DDI_CYC_ITEMS=1 -DDI_ASYNC_MINB=4"; do
  echo "## $defs"
  DI_NVCC_DEFS="$defs" python tools/build.py --force > gpurun_out/shape_build.log 2>&1 || { echo build failed; tail -5 gpurun_out/shape_build.log; continue; }
  python tools/exp/c4_ab.py warm=0 warm=-1 warm=-1,warm_shift=8 warm=-1,warm_shift=6
done
