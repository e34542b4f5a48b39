#!/bin/bash
mkdir -p gpurun_out
P="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for n in 2 4; do
  timeout 900 $P --nproc-per-node $n --master-port 2996$n bench.py --gpus $n --steps 300 --warmup 20 > gpurun_out/r14_bench_n$n.json 2> gpurun_out/r14_bench_n$n.err; echo "bench n=$n rc=$?"
  timeout 900 $P --nproc-per-node $n --master-port 2997$n bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/r14_bench_n${n}_s20.json 2> gpurun_out/r14_bench_n${n}_s20.err; echo "bench s20 n=$n rc=$?"
done
timeout 900 $P --nproc-per-node 4 --master-port 29981 tools/cfg1_bench.py --steps 2000 > gpurun_out/r14_cfg1_4gpu.jsonl 2> gpurun_out/r14_cfg1.err; echo "cfg1 rc=$?"
timeout 1200 $P --nproc-per-node 4 --master-port 29982 bench_configs.py --config 3 --steps 1000 --out gpurun_out/r14_cfg3_n4.jsonl > gpurun_out/r14_cfg3_n4.log 2>&1; echo "cfg3 n4 rc=$?"
timeout 1200 $P --nproc-per-node 2 --master-port 29983 bench_configs.py --config 3 --steps 1000 --out gpurun_out/r14_cfg3_n2.jsonl > gpurun_out/r14_cfg3_n2.log 2>&1; echo "cfg3 n2 rc=$?"
