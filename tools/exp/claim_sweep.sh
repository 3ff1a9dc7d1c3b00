# k_cycle: the tile claim's atomic round trip hidden (claim one ahead) or not
mkdir -p gpurun_out
for defs in "-DDI_CLAIM_AHEAD=0" "-DDI_CLAIM_AHEAD=1"; do
  echo "## $defs"
  DI_NVCC_DEFS="$defs" python tools/build.py --force > gpurun_out/claim_build.log 2>&1 || { echo build failed; continue; }
  python tools/exp/c4_ab.py warm=-1
  python tools/exp/c4_ab.py warm=-1 --config c3
  python tools/exp/c4_ab.py warm=-1 --config c2
done
DI_NVCC_DEFS="-DDI_CLAIM_AHEAD=1" python tools/build.py --force > /dev/null 2>&1 && python tools/exp/c5_gpu.py --solves 2 | tail -1 && python -m pytest tests/test_gpu_solve.py tests/test_gpu_cold.py tests/test_gpu_dist.py -k "async or warm or cold or dist_parts or compact" -x -q 2>&1 | tail -2
