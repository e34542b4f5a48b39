#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "auto_delivery or host_generator" > gpurun_out/r02_t7.log 2>&1
tail -1 gpurun_out/r02_t7.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step_fused -s 30 -c 1 -o gpurun_out/r02_cfg3_pull -f \
  python bench_configs.py --config 3 --engines fused --steps 10 --warmup 25 > gpurun_out/r02_cfg3_pull_ncu.log 2>&1
echo done
