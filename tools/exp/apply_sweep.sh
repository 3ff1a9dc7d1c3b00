# k_cold_apply: records in flight per thread (DI_APPLY_UNROLL) on C5, one GPU
mkdir -p gpurun_out
for u in 1 2 4 8; do
  echo "## DI_APPLY_UNROLL=$u"
  DI_NVCC_DEFS="-DDI_APPLY_UNROLL=$u" python tools/build.py --force > gpurun_out/apply_build.log 2>&1 || { echo build failed; continue; }
  python tools/exp/c5_gpu.py --solves 2
  python tools/exp/c5_gpu.py --solves 1 --profile | tail -2
done
