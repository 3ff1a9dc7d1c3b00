# k_cycle select: a selected node's fluid taken with an atomic exchange (0) or as F_i -= f (1)
mkdir -p gpurun_out
for defs in "-DDI_TAKE_SUB=0" "-DDI_TAKE_SUB=1"; do
  echo "## $defs"
  DI_NVCC_DEFS="$defs" python tools/build.py --force > gpurun_out/take_build.log 2>&1 || { echo build failed; continue; }
  python tools/exp/c4_ab.py warm=-1 warm=0
  python tools/exp/c4_ab.py warm=-1 --config c3
done
DI_NVCC_DEFS="-DDI_TAKE_SUB=1" python tools/build.py --force > /dev/null 2>&1 && python -m pytest tests/test_gpu_solve.py -k "async_cycles or warm_tier or c4_full" -x -q 2>&1 | tail -2
