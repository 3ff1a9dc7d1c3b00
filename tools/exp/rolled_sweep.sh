# warm instantiation of k_cycle: push body rolled over the int4 group (code size) or unrolled
mkdir -p gpurun_out
for defs in "-DDI_WARM_ROLLED=1" "-DDI_WARM_ROLLED=0"; do
  echo "## $defs"
  DI_NVCC_DEFS="$defs" python tools/build.py --force > gpurun_out/rolled_build.log 2>&1 || { echo build failed; continue; }
  python tools/exp/c4_ab.py warm=-1
done
