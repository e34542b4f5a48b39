#!/bin/bash
mkdir -p gpurun_out
for v in default u8 t512 u8t512; do
  if [ $v != default ]; then export NEUROCOMM_B200_LIB=$PWD/paper_2205_07125_b200/libneurocomm_b200_$v.so; fi
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum -k regex:k_histogram_smem -c 3 python tools/planner_bench.py --sizes 1000000 2>&1 | grep -E "gpu__time_duration|dram__bytes_read" | tail -2 | sed "s/^/$v /"
  unset NEUROCOMM_B200_LIB
done > gpurun_out/r02_k5_variants.log
echo done
