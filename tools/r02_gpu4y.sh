#!/bin/bash
# 4-GPU pass 2: config 3 on the reference partition, persistent-engine skew, fused-send A/B
mkdir -p gpurun_out
P="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for f in profiles/r02_k6_config3_greedy4.npz; do
  [ -f $f ] && timeout 1200 $P --nproc-per-node 4 --master-port 29821 bench_configs.py --config 3 \
     --partition greedy:$f --out gpurun_out/r02_cfg3_greedy_n4.jsonl > gpurun_out/r02_cfg3_greedy_n4.log 2>&1
done
echo "greedy rc=$?"
timeout 600 $P --nproc-per-node 4 --master-port 29822 tools/persist_skew.py --out gpurun_out/r02_persist_skew_n4.json > gpurun_out/r02_persist_skew_n4.log 2>&1
timeout 600 $P --nproc-per-node 2 --master-port 29823 tools/persist_skew.py --out gpurun_out/r02_persist_skew_n2.json > gpurun_out/r02_persist_skew_n2.log 2>&1
timeout 600 $P --nproc-per-node 4 --master-port 29824 tools/persist_skew.py --blocks-per-peer 8 --out gpurun_out/r02_persist_skew_n4_b8.json > /dev/null 2>&1
for fs in off on; do for n in 2 4; do
  timeout 600 $P --nproc-per-node $n --master-port 2983$n bench.py --gpus $n --steps 1000 --warmup 20 --no-push --no-cpu \
    --fused-send $fs > gpurun_out/r02_fs_${fs}_n$n.json 2>/dev/null
done; done
timeout 1200 $P --nproc-per-node 4 --master-port 29825 bench_configs.py --config 3 --steps 1000 --out gpurun_out/r02_cfg3_n4_long.jsonl > /dev/null 2>&1
echo done
