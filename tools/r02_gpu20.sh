#!/bin/bash
mkdir -p gpurun_out
C="python bench.py --steps 20 --warmup 3 --no-cpu --no-push"
$C > gpurun_out/r02_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches.csv $C > gpurun_out/r02_ncu_launches.log 2>&1
echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step_fused -s 10 -c 1 -o gpurun_out/r02_step_fused -f $C > gpurun_out/r02_ncu_full.log 2>&1
echo "full rc=$?"
