#!/bin/bash
# Per-GPU loads of configs 3 and 5 on 4 GPUs (weak: 1.25 M and 6.25 M neurons per GPU)
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29601 \
  bench.py --gpus 4 --scaling weak --neurons 1250000 --steps 300 --warmup 10 > gpurun_out/cfg3_like.json 2> gpurun_out/cfg3_like.err; echo "cfg3 rc=$?"
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29602 \
  bench.py --gpus 4 --scaling weak --neurons 6250000 --communities 64 --steps 200 --warmup 5 > gpurun_out/cfg5_like.json 2> gpurun_out/cfg5_like.err; echo "cfg5 rc=$?"
