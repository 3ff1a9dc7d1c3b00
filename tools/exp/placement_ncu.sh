# L2 / DRAM counters of k_cycle<COLD> at C5 in the fast placement (library arrays lowest) and the slow
# one (17.3 GB of link tensors below them): bash tools/exp/placement_ncu.sh
mkdir -p gpurun_out
M=gpu__time_duration.sum,lts__t_tag_requests.max.pct_of_peak_sustained_elapsed,lts__t_tag_requests.avg.pct_of_peak_sustained_elapsed,lts__t_sector_hit_rate.pct,lts__throughput.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sectors_srcunit_tex_op_red.sum
for m in "" "--via-host"; do
  echo "## placement: ${m:-library arrays lowest}"
  timeout 600 ncu --metrics $M --clock-control none -k regex:"k_cycle|k_cold_apply" -s 12 -c 4 --csv \
      --log-file gpurun_out/place${m}.csv python tools/exp/c5_bench_diff5.py --host-loop $m > gpurun_out/place${m}.log 2>&1
  python - "gpurun_out/place${m}.csv" <<'PY'
import csv, sys
lines = open(sys.argv[1]).read().splitlines()
st = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
rows = list(csv.DictReader(lines[st:]))
ids = sorted({int(r["ID"]) for r in rows})
for i in ids:
    rr = [r for r in rows if int(r["ID"]) == i]
    name = rr[0]["Kernel Name"][:40]
    print(i, name, "; ".join("%s=%s %s" % (r["Metric Name"].replace(".pct_of_peak_sustained_elapsed", "%").replace("lts__t_", "").replace("gpu__", ""), r["Metric Value"], r["Metric Unit"]) for r in rr))
PY
done
