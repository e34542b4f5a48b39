#!/bin/bash
# GPU parity suite, then A/B of the fused P2P send (--fused-send off sends from the exchange kernel)
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for r in 1 2; do
for fs in off on; do
  for n in 2 4; do
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port 2962$n bench.py --gpus $n --steps 1000 --warmup 20 --no-push --no-cpu --fused-send $fs 2>/dev/null | tail -n 1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
x=d['exchange_us']
print('fused_send=$fs N=$n value', d['value'], 'ms', d['ms_per_step'], 'kernel_ms', d['roofline']['kernel_ms'], 'xchg p50', x['p50'], 'transfer_only', x['p50_transfer_only'], 'e2e', d['e2e']['value'])"
  done
done; done
