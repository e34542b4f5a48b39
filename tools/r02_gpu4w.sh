#!/bin/bash
# 4-GPU: multi-rank parity after the pipelined relay; config 4 sweep (two-level latency)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multirank.py -q -p no:cacheprovider > gpurun_out/r02_multirank2.log 2>&1
tail -2 gpurun_out/r02_multirank2.log
P="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 4"
timeout 1500 $P --master-port 29871 bench_configs.py --config 4 --engines persistent,fused --steps 500 \
  --out gpurun_out/r02_cfg4_n4_pipelined.jsonl > gpurun_out/r02_cfg4_n4_pipelined.log 2>&1
echo "cfg4 rc=$?"
timeout 600 $P --master-port 29872 tools/cfg1_bench.py > gpurun_out/r02_cfg1_4gpu.jsonl 2> gpurun_out/r02_cfg1_4gpu.err
echo "cfg1 rc=$?"
echo done
