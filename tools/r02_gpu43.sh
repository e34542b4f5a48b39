#!/bin/bash
# 4-GPU re-measure after the push-phase prefetch: tests, configs 3 / 3-regional / 4 / 5, skew, config 2 N=2/4
mkdir -p gpurun_out
P="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1200 $P --nproc-per-node 2 --master-port 29950 bench_configs.py --config 5 --engines persistent --steps 1000 --out gpurun_out/r06_cfg5_n2_long.jsonl > gpurun_out/r06_cfg5_n2_long.log 2>&1; echo "cfg5 n2 rc=$?"
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r06_gpu_tests_4gpu.log 2>&1
tail -1 gpurun_out/r06_gpu_tests_4gpu.log
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench_configs.py --config 3 --steps 1000 --out gpurun_out/r06_cfg3_n1_long.jsonl > gpurun_out/r06_cfg3_n1_long.log 2>&1; echo "cfg3 n1 rc=$?"
timeout 1200 $P --nproc-per-node 2 --master-port 29951 bench_configs.py --config 3 --steps 1000 --out gpurun_out/r06_cfg3_n2_long.jsonl > gpurun_out/r06_cfg3_n2_long.log 2>&1; echo "cfg3 n2 rc=$?"
timeout 1200 $P --nproc-per-node 4 --master-port 29952 bench_configs.py --config 3 --steps 1000 --out gpurun_out/r06_cfg3_n4_long.jsonl > gpurun_out/r06_cfg3_n4_long.log 2>&1; echo "cfg3 n4 rc=$?"
timeout 1200 $P --nproc-per-node 4 --master-port 29953 bench_configs.py --config 3 --steps 1000 --engines persistent \
  --partition greedy:profiles/r02_k6_config3_greedy4.npz --out gpurun_out/r06_cfg3_greedy_n4.jsonl > gpurun_out/r06_cfg3_greedy_n4.log 2>&1; echo "cfg3 greedy rc=$?"
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench_configs.py --config 3 --communities 8 --steps 1000 --engines persistent --out gpurun_out/r06_cfg3r_n1.jsonl > gpurun_out/r06_cfg3r_n1.log 2>&1; echo "cfg3r n1 rc=$?"
timeout 1200 $P --nproc-per-node 2 --master-port 29954 bench_configs.py --config 3 --communities 8 --steps 1000 --engines persistent --out gpurun_out/r06_cfg3r_n2.jsonl > gpurun_out/r06_cfg3r_n2.log 2>&1; echo "cfg3r n2 rc=$?"
timeout 1200 $P --nproc-per-node 4 --master-port 29955 bench_configs.py --config 3 --communities 8 --steps 1000 --engines persistent --out gpurun_out/r06_cfg3r_n4.jsonl > gpurun_out/r06_cfg3r_n4.log 2>&1; echo "cfg3r n4 rc=$?"
timeout 1200 $P --nproc-per-node 4 --master-port 29956 bench_configs.py --config 3 --communities 8 --steps 1000 --engines persistent \
  --partition greedy:profiles/r02_k6_config3r_greedy4.npz --out gpurun_out/r06_cfg3r_greedy_n4.jsonl > gpurun_out/r06_cfg3r_greedy_n4.log 2>&1; echo "cfg3r greedy rc=$?"
timeout 1800 $P --nproc-per-node 4 --master-port 29957 bench_configs.py --config 4 --engines persistent,fused --steps 500 \
  --out gpurun_out/r06_cfg4_n4.jsonl > gpurun_out/r06_cfg4_n4.log 2>&1; echo "cfg4 rc=$?"
timeout 1500 $P --nproc-per-node 4 --master-port 29958 bench_configs.py --config 5 --steps 300 --out gpurun_out/r06_cfg5_n4.jsonl > gpurun_out/r06_cfg5_n4.log 2>&1; echo "cfg5 n4 rc=$?"
for n in 2 4; do
  timeout 900 $P --nproc-per-node $n --master-port 2996$n tools/persist_skew.py --out gpurun_out/r06_persist_skew_n$n.json > gpurun_out/r06_persist_skew_n$n.log 2>&1; echo "skew n=$n rc=$?"
  timeout 900 $P --nproc-per-node $n --master-port 2997$n bench.py --gpus $n --steps 300 --warmup 20 > gpurun_out/r06_bench_n$n.json 2> gpurun_out/r06_bench_n$n.err; echo "bench n=$n rc=$?"
done
echo done
