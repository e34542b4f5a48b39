#!/bin/bash
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02_gpu_tests11.log 2>&1
tail -3 gpurun_out/r02_gpu_tests11.log
for w in 1 2 4; do
  timeout 900 python bench_configs.py --config 3 --engines persistent --push-windows $w --steps 500 --warmup 20 \
    --out gpurun_out/r02_win_cfg3_n1_w$w.jsonl > /dev/null 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/r02_win_cfg3_n1_w$w.jsonl').readlines()[-1]); print('w=$w', d['steps_per_s'], d['push_windows'], d['clocks']['sm_mhz'])"
done
echo done
