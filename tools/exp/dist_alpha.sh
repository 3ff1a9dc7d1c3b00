# Threshold scale alpha (F4, di_set_threshold_scale) on the partitioned COLD cycle: C5 on 8 emulated
# ranks, per-rank kernel totals from the ncu launch list (cycles x us per rank-cycle is what counts).
#   bash tools/exp/dist_alpha.sh 1 0.5 0.25 ...
mkdir -p gpurun_out
for al in "$@"; do
  echo "## alpha $al"
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_cycle|k_compact_remote|k_apply_inbox" \
      --csv --log-file gpurun_out/dal_$al.csv python tools/exp/c5_dist_proj.py 8 c5 --alpha $al > gpurun_out/dal_$al.log 2>&1
  grep "emulated ranks" gpurun_out/dal_$al.log
  python tools/exp/launch_avg.py gpurun_out/dal_$al.csv
done
