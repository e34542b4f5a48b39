#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_configs_downscaled.py -q -p no:cacheprovider > gpurun_out/r02_t8.log 2>&1
tail -3 gpurun_out/r02_t8.log
for v in default pf0; do
  if [ $v = pf0 ]; then export NEUROCOMM_B200_LIB=$PWD/paper_2205_07125_b200/libneurocomm_b200_pf0.so; fi
  timeout 600 python bench_configs.py --config 3 --engines fused --steps 100 --warmup 10 --out gpurun_out/r02_pf_$v.jsonl > /dev/null 2>&1
  unset NEUROCOMM_B200_LIB
done
for v in default pf0; do python -c "
import json; d=json.loads(open('gpurun_out/r02_pf_$v.jsonl').readlines()[-1]); print('$v', d['steps_per_s'], d['kernel_ms'], d['clocks']['sm_mhz'])"; done
echo done
