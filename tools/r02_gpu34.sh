#!/bin/bash
# small-shard pull kernel A/B on one GPU via virtual ranks: tiles x block split at N = 8 and 4
mkdir -p gpurun_out
o=gpurun_out/r02_split_ab.jsonl; : > $o
run() { timeout 600 python tools/vr_kernel.py --steps 200 "$@" 2>>gpurun_out/r02_split_ab.err | tee -a $o; }
run --worlds 1,8
run --worlds 8 --split 2
run --worlds 8 --split 3
run --worlds 8 --tile-words 15648 --split 1
run --worlds 8 --tile-words 15648 --split 2
run --worlds 8 --tile-words 15648 --split 3
run --worlds 8 --tile-words 3936 --split 1
run --worlds 8 --tile-words 3936 --split 0
run --worlds 4
run --worlds 4 --split 2
run --worlds 4 --tile-words 7840 --split 1
run --worlds 4 --tile-words 7840 --split 0
