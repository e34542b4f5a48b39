#!/bin/bash
# small-shard tiling re-sweep after triple buffering + lean row sum (config 2 network, 4 and 8 virtual ranks)
mkdir -p gpurun_out
o=gpurun_out/r02_split_ab2.jsonl; : > $o
run() { timeout 600 python tools/vr_kernel.py --steps 200 "$@" 2>/dev/null | tee -a $o; }
run --worlds 8
run --worlds 8 --split 0
run --worlds 8 --split 2
run --worlds 8 --tile-words 5248 --split 1
run --worlds 8 --tile-words 5248 --split 0
run --worlds 8 --tile-words 3936 --split 0
run --worlds 8 --tile-words 15648 --split 1
run --worlds 4
run --worlds 4 --split 0
run --worlds 4 --tile-words 10432 --split 1
run --worlds 4 --tile-words 10432 --split 0
run --worlds 4 --tile-words 7840 --split 0
