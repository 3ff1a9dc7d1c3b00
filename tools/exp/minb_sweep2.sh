# k_cycle resident CTAs per SM (DI_ASYNC_MINB: register cap 64 / 48 / 40), with the warm tier
mkdir -p gpurun_out
for m in 4 5 6; do
  echo "## DI_ASYNC_MINB=$m"
  DI_NVCC_DEFS="-DDI_ASYNC_MINB=$m" python tools/build.py --force > gpurun_out/minb_build.log 2>&1 || { echo build failed; continue; }
  python tools/exp/c4_ab.py warm=-1 warm=0
done
