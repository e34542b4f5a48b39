#!/bin/bash
# GPU parity suite, then the scaling series, then the 8-GPU-like per-GPU load on 4 GPUs
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
bash tools/scaling_series.sh
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29571 \
  bench.py --gpus 4 --neurons 500000 --no-cpu > gpurun_out/like8.json 2> gpurun_out/like8.err; echo "like8 rc=$?"
