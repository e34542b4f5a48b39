#!/bin/bash
# LIF ILP change: full GPU suite on 1 GPU, config 3 at N=1 (pull + persistent), config 2 bench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02_lif_gpu_tests.log 2>&1
tail -2 gpurun_out/r02_lif_gpu_tests.log
timeout 900 python bench_configs.py --config 3 --steps 1000 --out gpurun_out/r02_cfg3_n1_lif.jsonl > gpurun_out/r02_cfg3_n1_lif.log 2>&1; echo "cfg3 rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench_lif.json 2> gpurun_out/r02_bench_lif.err; echo "bench rc=$?"
