#!/bin/bash
mkdir -p gpurun_out
o=gpurun_out/r02_triple_ab.jsonl; : > $o
for rep in 1 2; do
  timeout 600 python tools/vr_kernel.py --worlds 8 --buffers 2 2>/dev/null | tee -a $o
  timeout 600 python tools/vr_kernel.py --worlds 8 --buffers 3 2>/dev/null | tee -a $o
done
timeout 600 python tools/vr_kernel.py --worlds 8 --tile-words 3936 --buffers 2 2>/dev/null | tee -a $o
timeout 600 python tools/vr_kernel.py --worlds 8 --tile-words 3936 --buffers 3 2>/dev/null | tee -a $o
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "tile or config2 or forced" > gpurun_out/r02_triple_tests.log 2>&1; tail -1 gpurun_out/r02_triple_tests.log
