#!/bin/bash
# k_compact_remote tuning on the GPU box: rebuild with each (kCompPer, blocks/SM) and take the
# ncu launch list of one partitioned C4 solve on 2 emulated ranks
VARS=${COMP_VARIANTS:-"16,4 32,4 16,8 8,8 32,8"}
for v in $VARS; do
  v=${v/,/ }
  set -- $v
  DI_NVCC_DEFS="-DDI_COMP_PER=$1 -DDI_COMP_BPS=$2" python tools/build.py --force > /dev/null 2>&1 || { echo build failed; exit 1; }
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/comp_$1_$2.csv python tools/exp/dist_prof.py c4 2 > /dev/null 2>&1
  python - "$1" "$2" <<'PY'
import csv, sys
rows = list(csv.reader(open(f"gpurun_out/comp_{sys.argv[1]}_{sys.argv[2]}.csv")))
hdr = next(r for r in rows if "Kernel Name" in r); i = hdr.index("Kernel Name"); j = hdr.index("Metric Value")
t = [float(r[j].replace(",", "")) for r in rows[rows.index(hdr) + 1:] if len(r) == len(hdr) and "k_compact_remote" in r[i]]
print("per", sys.argv[1], "blocks/SM", sys.argv[2], "k_compact_remote avg us", round(sum(t) / len(t) / 1e3, 2), "n", len(t))
PY
done
python tools/build.py --force > /dev/null 2>&1
