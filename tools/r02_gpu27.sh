#!/bin/bash
# K5 uniform-weight path: parity, A/B of unroll / smem variants, ncu of the kernel
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "aggregate or genetic" > gpurun_out/r02_k5u_tests.log 2>&1
tail -2 gpurun_out/r02_k5u_tests.log
for l in paper_2205_07125_b200/libneurocomm_b200.so variants/k5u4.so variants/k5u8s32.so; do
  NEUROCOMM_B200_LIB=$l timeout 900 python tools/planner_bench.py --sizes 1000000 > gpurun_out/r02_k5u_$(basename $l .so).json 2>&1
  echo "$l: $(tail -1 gpurun_out/r02_k5u_$(basename $l .so).json)"
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_histogram_smem -c 2 -o gpurun_out/r02_k5u \
  python tools/planner_bench.py --sizes 1000000 --reps 1 > gpurun_out/r02_k5u_ncu.log 2>&1
echo "ncu rc=$?"
