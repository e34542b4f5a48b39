#!/bin/bash
# 4-GPU final: config 3 on the reference partition (partition_greedy off the generator) vs blocks; bench N=2/4
mkdir -p gpurun_out
P="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1500 $P --nproc-per-node 4 --master-port 29881 bench_configs.py --config 3 --steps 1000 \
  --partition greedy:profiles/r02_k6_config3_greedy4.npz --out gpurun_out/r02_cfg3_greedy_n4.jsonl > gpurun_out/r02_cfg3_greedy_n4.log 2>&1
echo "cfg3 greedy rc=$?"
timeout 1500 $P --nproc-per-node 4 --master-port 29882 bench_configs.py --config 3 --steps 1000 \
  --out gpurun_out/r02_cfg3_blocks_n4.jsonl > gpurun_out/r02_cfg3_blocks_n4.log 2>&1
echo "cfg3 blocks rc=$?"
for n in 2 4; do
  timeout 900 $P --nproc-per-node $n --master-port 2989$n bench.py --gpus $n --steps 300 --warmup 20 \
    > gpurun_out/r02_final_bench_n$n.json 2> gpurun_out/r02_final_bench_n$n.err
  echo "bench n=$n rc=$?"
  timeout 600 $P --nproc-per-node $n --master-port 2990$n bench.py --gpus $n --impl reference --steps 20 --warmup 5 \
    > gpurun_out/r02_final_ref_n$n.json 2> gpurun_out/r02_final_ref_n$n.err
done
echo done
