#!/bin/bash
mkdir -p gpurun_out
for args in "4 0 2 direct" "4 0 2 two-level" "4 0 2 two-level rev" "4 1 2 two-level"; do
  echo "=== $args"; timeout 120 python tools/vr_debug.py $args 2>&1 | head -60
done > gpurun_out/r02_vr_debug3.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "aggregate or genetic or config2" > gpurun_out/r02_t3.log 2>&1
timeout 600 python tools/planner_bench.py --sizes 1000000 > gpurun_out/r02_planner.log 2>&1

timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_histogram -c 2 -o gpurun_out/r02_k5 -f python tools/planner_bench.py --sizes 1000000 > gpurun_out/r02_k5_ncu.log 2>&1
echo ncu done
