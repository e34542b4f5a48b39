#!/bin/bash
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02_gpu_tests6.log 2>&1
tail -3 gpurun_out/r02_gpu_tests6.log
timeout 300 python tools/planner_bench.py --sizes 1000000 > gpurun_out/r02_planner6.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_histogram_smem -c 1 -o gpurun_out/r02_k5d -f python tools/planner_bench.py --sizes 1000000 > /dev/null 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench6_n1_s20.json 2> gpurun_out/r02_bench6_n1_s20.err
echo done
