#!/bin/bash
# 4-GPU re-measure after the LIF ILP change: multi-rank tests, configs 3 / 3-regional / 4 / 5,
# the reference partition of config 3, persistent-engine skew, config 2 N=2/4
mkdir -p gpurun_out
P="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_multirank.py -q -p no:cacheprovider > gpurun_out/r03_multirank.log 2>&1
tail -1 gpurun_out/r03_multirank.log
timeout 1200 $P --nproc-per-node 2 --master-port 29901 bench_configs.py --config 3 --steps 1000 --out gpurun_out/r03_cfg3_n2_long.jsonl > gpurun_out/r03_cfg3_n2_long.log 2>&1; echo "cfg3 n2 rc=$?"
timeout 1200 $P --nproc-per-node 4 --master-port 29902 bench_configs.py --config 3 --steps 1000 --out gpurun_out/r03_cfg3_n4_long.jsonl > gpurun_out/r03_cfg3_n4_long.log 2>&1; echo "cfg3 n4 rc=$?"
timeout 1200 $P --nproc-per-node 4 --master-port 29903 bench_configs.py --config 3 --steps 1000 --engines persistent \
  --partition greedy:profiles/r02_k6_config3_greedy4.npz --out gpurun_out/r03_cfg3_greedy_n4.jsonl > gpurun_out/r03_cfg3_greedy_n4.log 2>&1; echo "cfg3 greedy rc=$?"
timeout 1200 $P --nproc-per-node 4 --master-port 29904 bench_configs.py --config 3 --communities 8 --steps 1000 --engines persistent --out gpurun_out/r03_cfg3r_n4.jsonl > gpurun_out/r03_cfg3r_n4.log 2>&1; echo "cfg3r n4 rc=$?"
timeout 1200 $P --nproc-per-node 2 --master-port 29905 bench_configs.py --config 3 --communities 8 --steps 1000 --engines persistent --out gpurun_out/r03_cfg3r_n2.jsonl > gpurun_out/r03_cfg3r_n2.log 2>&1; echo "cfg3r n2 rc=$?"
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench_configs.py --config 3 --communities 8 --steps 1000 --engines persistent --out gpurun_out/r03_cfg3r_n1.jsonl > gpurun_out/r03_cfg3r_n1.log 2>&1; echo "cfg3r n1 rc=$?"
timeout 1800 $P --nproc-per-node 4 --master-port 29906 bench_configs.py --config 4 --engines persistent,fused --steps 500 \
  --out gpurun_out/r03_cfg4_n4.jsonl > gpurun_out/r03_cfg4_n4.log 2>&1; echo "cfg4 rc=$?"
timeout 1200 $P --nproc-per-node 2 --master-port 29907 bench_configs.py --config 5 --engines persistent --steps 1000 --out gpurun_out/r03_cfg5_n2_long.jsonl > gpurun_out/r03_cfg5_n2_long.log 2>&1; echo "cfg5 n2 rc=$?"
timeout 1500 $P --nproc-per-node 4 --master-port 29908 bench_configs.py --config 5 --steps 300 --out gpurun_out/r03_cfg5_n4.jsonl > gpurun_out/r03_cfg5_n4.log 2>&1; echo "cfg5 n4 rc=$?"
for n in 2 4; do
  timeout 900 $P --nproc-per-node $n --master-port 2991$n tools/persist_skew.py --out gpurun_out/r03_persist_skew_n$n.json > gpurun_out/r03_persist_skew_n$n.log 2>&1; echo "skew n=$n rc=$?"
  timeout 900 $P --nproc-per-node $n --master-port 2992$n bench.py --gpus $n --steps 300 --warmup 20 > gpurun_out/r03_bench_n$n.json 2> gpurun_out/r03_bench_n$n.err; echo "bench n=$n rc=$?"
done
echo done
