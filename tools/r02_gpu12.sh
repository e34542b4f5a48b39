#!/bin/bash
mkdir -p gpurun_out
P="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 2"
for w in 1 2 4; do
  timeout 900 $P --master-port 2984$w bench_configs.py --config 5 --engines persistent --push-windows $w --steps 300 \
    --warmup 20 --out gpurun_out/r02_win_cfg5_n2_w$w.jsonl > gpurun_out/r02_win_cfg5_n2_w$w.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/r02_win_cfg5_n2_w$w.jsonl').readlines()[-1]); x=d['exchange_us']; print('w=$w', d['steps_per_s'], d['push_windows'], x['p50'], x['p99'], d['memory_per_gpu'], d['clocks']['sm_mhz'])"
done
echo done
