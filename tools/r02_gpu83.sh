#!/bin/bash
mkdir -p gpurun_out
P="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "graph or config2 or simulate" 2>&1 | tail -1
for rep in 1 2 3; do
  for n in 4 2; do
    timeout 900 $P --nproc-per-node $n --master-port 2995$n bench.py --gpus $n --steps 20 --warmup 5 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); x=d['exchange_us']; print($n, d['value'], x['p50'], x['p99'], d['e2e']['value'])"
  done
done
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e-api 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(1, d['value'], d['e2e']['value'])"
