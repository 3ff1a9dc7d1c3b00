#!/bin/bash
# Round evidence for the bench (on the GPU box; B200_PROFILING.md recipe):
#   bash tools/round_profile.sh TAG
# 1. the bench command itself without a profiler (must exit 0 first),
# 2. its ncu launch list (gpu__time_duration.sum, --clock-control none: cold and serialised, so
#    per-kernel SHARES of the step are what compares with the bench's own CUDA events),
# 3. one `ncu --set full` capture of k_cycle (C4, the bench's kernel) for roofline.traffic.
TAG=${1:-round}
mkdir -p gpurun_out
python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu --no-breadth > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err \
  || { echo "bench failed"; tail gpurun_out/${TAG}_bench.err; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu --no-breadth > gpurun_out/${TAG}_ncu_l.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_cycle" -s 20 -c 3 \
    -o gpurun_out/${TAG} python tools/profile_solve.py --config c4 --solves 1 --asynchronous > gpurun_out/${TAG}_ncu_f.log 2>&1
tail -c 400 gpurun_out/${TAG}_bench.json
