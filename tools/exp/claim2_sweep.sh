# k_cycle: next tile claimed by thread 0 before the end-of-tile barrier (double-buffered tile state)
mkdir -p gpurun_out
python tools/exp/c4_ab.py warm=-1
python tools/exp/c4_ab.py warm=-1 --config c3
python tools/exp/c4_ab.py warm=-1 --config c2
python tools/exp/c5_gpu.py --solves 2 | tail -1
python -m pytest tests/test_gpu_solve.py tests/test_gpu_cold.py tests/test_gpu_cycle_select.py tests/test_gpu_dist.py -x -q 2>&1 | tail -2
