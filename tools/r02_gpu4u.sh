#!/bin/bash
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02_gpu_tests_4gpu.log 2>&1
tail -3 gpurun_out/r02_gpu_tests_4gpu.log
python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 --master-port=29531 tests/workers/dist_parity.py > gpurun_out/r02_dist_parity_4.log 2>&1
python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 --master-port=29532 tests/workers/dist_aggregate.py > gpurun_out/r02_dist_aggregate_4.log 2>&1
grep -E "ranks\]" gpurun_out/r02_dist_parity_4.log gpurun_out/r02_dist_aggregate_4.log | tail -30
