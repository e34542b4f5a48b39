#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_multirank.py -x -q 2>&1 | tail -2
for r in 1 2; do
  for n in 2 4; do
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port 2963$n bench.py --gpus $n --steps 1000 --warmup 20 --no-push --no-cpu 2>/dev/null | tail -n 1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
x=d['exchange_us']
print('acq_rel N=$n value', d['value'], 'ms', d['ms_per_step'], 'kernel_ms', d['roofline']['kernel_ms'], 'xchg p50', x['p50'], 'incl_skew', x['p50_incl_skew'], 'e2e', d['e2e']['value'])"
  done
done
