#!/bin/bash
# driver-like scaling series on one 4-GPU box: bench.py at N = 1, 2, 4 back to back (20 and 300 steps)
mkdir -p gpurun_out
o=gpurun_out/r02_scale_series.jsonl; : > $o
P="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for steps in 20 300; do
  CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --steps $steps --warmup 5 --no-cpu --no-e2e-api 2>/dev/null | tail -1 >> $o
  for n in 2 4; do
    timeout 900 $P --nproc-per-node $n --master-port 2985$n bench.py --gpus $n --steps $steps --warmup 5 2>/dev/null | tail -1 >> $o
  done
done
python -c "
import json
for l in open('$o'):
    d=json.loads(l); print(d['n_gpus'], d['steps'], d['value'], d['roofline']['frac'], (d.get('exchange_us') or {}).get('p50'), d['clocks']['sm_mhz'])
"
