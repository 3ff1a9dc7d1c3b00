# Partitioned COLD cycle (k_cycle<DIST,COLD>) A/B of compile-time knobs on C5 over 8 emulated ranks
# (per-rank kernel times from the ncu launch list: the ranks' kernels serialise under ncu), and the
# single-GPU C5 solve with the same build:  bash tools/exp/dist_ab.sh "DEFS1" "DEFS2" ...
mkdir -p gpurun_out
i=0
for defs in "$@"; do
  i=$((i+1))
  echo "## [$i] defs: '$defs'"
  DI_NVCC_DEFS="$defs" python tools/build.py --force > gpurun_out/dab_build_$i.log 2>&1 || { echo build failed; continue; }
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_cycle|k_compact_remote|k_apply_inbox" \
      --csv --log-file gpurun_out/dab_$i.csv python tools/exp/c5_dist_proj.py 8 c5 > gpurun_out/dab_$i.log 2>&1
  grep "emulated ranks" gpurun_out/dab_$i.log
  python tools/exp/launch_avg.py gpurun_out/dab_$i.csv
  timeout 600 python tools/exp/c5_gpu.py --solves 2 2>&1 | grep -E "solve [01]"
done
