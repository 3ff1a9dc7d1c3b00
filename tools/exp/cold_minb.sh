# C5 on one GPU: resident CTAs per SM of the COLD k_cycle (register cap 64 with spills, or 80)
mkdir -p gpurun_out
for m in 4 3; do
  echo "## DI_COLD_MINB=$m"
  DI_NVCC_DEFS="-DDI_COLD_MINB=$m" python tools/build.py --force > gpurun_out/cm_build.log 2>&1 || { echo build failed; continue; }
  python tools/exp/c5_gpu.py --solves 2 | tail -2
done
