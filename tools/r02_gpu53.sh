#!/bin/bash
# cross-engine state agreement at real size: config 3 (N=1, 4), config 4 sweep (N=4), config 5 (N=4)
mkdir -p gpurun_out
P="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench_configs.py --config 3 --steps 1000 --out gpurun_out/r08_cfg3_n1.jsonl > gpurun_out/r08_cfg3_n1.log 2>&1; echo "cfg3 n1 rc=$?"; tail -1 gpurun_out/r08_cfg3_n1.jsonl | cut -c1-300
timeout 1200 $P --nproc-per-node 4 --master-port 29961 bench_configs.py --config 3 --steps 1000 --out gpurun_out/r08_cfg3_n4.jsonl > gpurun_out/r08_cfg3_n4.log 2>&1; echo "cfg3 n4 rc=$?"; tail -1 gpurun_out/r08_cfg3_n4.jsonl | cut -c1-300
timeout 1800 $P --nproc-per-node 4 --master-port 29962 bench_configs.py --config 4 --engines persistent,fused --steps 500 --out gpurun_out/r08_cfg4_n4.jsonl > gpurun_out/r08_cfg4_n4.log 2>&1; echo "cfg4 rc=$?"; grep cross_engine gpurun_out/r08_cfg4_n4.jsonl | cut -c1-400
timeout 1500 $P --nproc-per-node 4 --master-port 29963 bench_configs.py --config 5 --steps 300 --out gpurun_out/r08_cfg5_n4.jsonl > gpurun_out/r08_cfg5_n4.log 2>&1; echo "cfg5 n4 rc=$?"; grep cross_engine gpurun_out/r08_cfg5_n4.jsonl | cut -c1-400
