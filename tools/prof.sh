#!/bin/bash
# usage (on the GPU box): bash tools/prof.sh TAG [config] [extra args for profile_solve.py]
# plain run -> launch list (gpu__time_duration) -> ncu --set full of k_select/k_push/k_pull
TAG=${1:-prof}; CFG=${2:-c4}; shift 2; EXTRA="$@"
mkdir -p gpurun_out
python tools/profile_solve.py --config $CFG --solves 2 $EXTRA > gpurun_out/${TAG}_plain.log 2>&1 || { echo "plain run failed"; tail gpurun_out/${TAG}_plain.log; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
    python tools/profile_solve.py --config $CFG --solves 2 $EXTRA > gpurun_out/${TAG}_ncu_l.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"${NCU_KERNELS:-k_select|k_push|k_pull|k_cycle}" -s ${NCU_SKIP:-60} -c ${NCU_COUNT:-9} \
    -o gpurun_out/${TAG} python tools/profile_solve.py --config $CFG --solves 1 $EXTRA > gpurun_out/${TAG}_ncu_f.log 2>&1
tail -2 gpurun_out/${TAG}_plain.log
