#!/bin/bash
# 4-GPU pass on the final code: GPU tests (incl. multi-rank), config 2 strong scaling N=2/4,
# config 3 regional (C = 8, 90 % intra) at N = 1 / 2 / 4
mkdir -p gpurun_out
P="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02_final4_gpu_tests.log 2>&1
tail -2 gpurun_out/r02_final4_gpu_tests.log
for n in 2 4; do
  timeout 900 $P --nproc-per-node $n --master-port 2961$n bench.py --gpus $n --steps 300 --warmup 20 \
    > gpurun_out/r02_final_bench_n$n.json 2> gpurun_out/r02_final_bench_n$n.err
  echo "bench n=$n rc=$? $(tail -c 300 gpurun_out/r02_final_bench_n$n.json)"
done
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench_configs.py --config 3 --communities 8 --steps 300 \
  --out gpurun_out/r02_cfg3r_n1.jsonl > gpurun_out/r02_cfg3r_n1.log 2>&1; echo "cfg3r n1 rc=$?"
for n in 2 4; do
  timeout 900 $P --nproc-per-node $n --master-port 2962$n bench_configs.py --config 3 --communities 8 --steps 300 \
    --out gpurun_out/r02_cfg3r_n$n.jsonl > gpurun_out/r02_cfg3r_n$n.log 2>&1
  echo "cfg3r n=$n rc=$?"
done
echo done
