#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "config2 or push_only" > gpurun_out/r02_t2.log 2>&1
timeout 300 python tools/vr_debug.py 4 0 2 > gpurun_out/r02_vr_debug.log 2>&1
timeout 300 python tools/vr_debug.py 4 0 8 > gpurun_out/r02_vr_debug8.log 2>&1
timeout 900 python bench_configs.py --config 3 --out gpurun_out/r02_cfg3_n1.jsonl > gpurun_out/r02_cfg3_n1.log 2>&1
echo done
