#!/bin/bash
mkdir -p gpurun_out
P="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 2"
timeout 1200 $P --master-port 29891 bench_configs.py --config 3 --steps 1000 --out gpurun_out/r02_cfg3_n2_long.jsonl > gpurun_out/r02_cfg3_n2_long.log 2>&1
echo "cfg3 rc=$?"
timeout 1200 $P --master-port 29892 bench_configs.py --config 5 --engines persistent --steps 1000 --out gpurun_out/r02_cfg5_n2_long.jsonl > gpurun_out/r02_cfg5_n2_long.log 2>&1
echo "cfg5 rc=$?"
timeout 900 python bench_configs.py --config 3 --steps 1000 --out gpurun_out/r02_cfg3_n1_long.jsonl > /dev/null 2>&1
echo "cfg3 n1 rc=$?"
