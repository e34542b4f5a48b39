#!/bin/bash
mkdir -p gpurun_out
o=gpurun_out/r02_cta2_ab.jsonl; : > $o
run() { timeout 600 python tools/vr_kernel.py --steps 200 "$@" 2>&1 | grep '^{' | tee -a $o; }
for rep in 1 2; do
run --worlds 8 --tile-words 7840 --split 1
run --worlds 8 --tile-words 7840 --split 1 --cta-mult 2
run --worlds 8 --tile-words 7840 --split 0 --cta-mult 2
run --worlds 4 --tile-words 15648 --split 1
run --worlds 4 --tile-words 10432 --split 1 --cta-mult 2
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "tiled or config2" 2>&1 | tail -1
