#!/bin/bash
mkdir -p gpurun_out
for v in default s16 b8 s16b8; do
  if [ $v != default ]; then export NEUROCOMM_B200_LIB=$PWD/paper_2205_07125_b200/libneurocomm_b200_$v.so; fi
  timeout 300 ncu --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__warps_active.avg.pct_of_peak_sustained_active -k regex:k_histogram_smem -c 1 python tools/planner_bench.py --sizes 1000000 2>&1 | grep -E "gpu__time_duration|dram__bytes_read|warps_active" | sed "s/^/$v /"
  unset NEUROCOMM_B200_LIB
done > gpurun_out/r02_k5_variants2.log
echo done
