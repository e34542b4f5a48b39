#!/bin/bash
# 4-GPU pass 3: config 4 with the reference's analytic model + calibration, config 5 at 4 GPUs with push windows 1/2
mkdir -p gpurun_out
P="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 4"
timeout 1500 $P --master-port 29851 bench_configs.py --config 4 --engines persistent,fused --steps 500 \
  --out gpurun_out/r02_cfg4_n4_model.jsonl > gpurun_out/r02_cfg4_n4_model.log 2>&1
echo "cfg4 rc=$?"
for w in 1 2; do
  timeout 900 $P --master-port 2986$w bench_configs.py --config 5 --engines persistent --push-windows $w --steps 300 \
    --out gpurun_out/r02_win_cfg5_n4_w$w.jsonl > /dev/null 2>&1
  echo "cfg5 w=$w rc=$?"
done
echo done
