#!/bin/bash
# usage (on the GPU box): bash tools/round_profile.sh TAG
# GPU suite, bench + reference arm, the launch list of the bench command, ncu --set full of k_cycle
set -x
TAG=${1:-prof}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_gpu_tests.log 2>&1; tail -3 gpurun_out/${TAG}_gpu_tests.log
timeout 300 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; cat gpurun_out/${TAG}_bench.json
timeout 300 python bench.py --impl reference > gpurun_out/${TAG}_reference.json 2>/dev/null; cat gpurun_out/${TAG}_reference.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv -c 5000 --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/${TAG}_ncu_l.log 2>&1; echo ncu_l $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cycle -s 20 -c 3 -o gpurun_out/${TAG} python tools/profile_solve.py --config c4 --solves 1 --asynchronous > gpurun_out/${TAG}_ncu_f.log 2>&1; echo ncu_f $?
