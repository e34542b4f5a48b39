#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_virtual_ranks.py -q -p no:cacheprovider > gpurun_out/r02_t18.log 2>&1
tail -15 gpurun_out/r02_t18.log
