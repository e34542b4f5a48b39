#!/bin/bash
mkdir -p gpurun_out
P="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1800 $P --nproc-per-node 4 --master-port 29991 bench_configs.py --config 4 --engines persistent,fused --steps 500 --out gpurun_out/r11_cfg4_n4.jsonl > gpurun_out/r11_cfg4_n4.log 2>&1; echo "cfg4 rc=$?"
timeout 1500 $P --nproc-per-node 4 --master-port 29992 bench_configs.py --config 5 --steps 300 --out gpurun_out/r11_cfg5_n4.jsonl > gpurun_out/r11_cfg5_n4.log 2>&1; echo "cfg5 n4 rc=$?"
timeout 1200 $P --nproc-per-node 2 --master-port 29993 bench_configs.py --config 5 --engines persistent --steps 1000 --out gpurun_out/r11_cfg5_n2.jsonl > gpurun_out/r11_cfg5_n2.log 2>&1; echo "cfg5 n2 rc=$?"
