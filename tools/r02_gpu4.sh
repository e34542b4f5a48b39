#!/bin/bash
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/r02_gpu_tests4.log 2>&1
tail -3 gpurun_out/r02_gpu_tests4.log
timeout 600 python tools/planner_bench.py --sizes 1000000 > gpurun_out/r02_planner4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_histogram_smem -c 1 -o gpurun_out/r02_k5b -f python tools/planner_bench.py --sizes 1000000 > gpurun_out/r02_k5b_ncu.log 2>&1
echo done
