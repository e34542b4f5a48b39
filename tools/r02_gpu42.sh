#!/bin/bash
mkdir -p gpurun_out
P="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "persistent or windowed or binned or push" > gpurun_out/r05_tests.log 2>&1; tail -1 gpurun_out/r05_tests.log
CUDA_VISIBLE_DEVICES=0 timeout 600 python tools/persistent_phases.py 10000000 2>&1 | tail -3
CUDA_VISIBLE_DEVICES=0 timeout 600 python tools/persistent_phases.py 1000000 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_multirank.py -q -p no:cacheprovider -x > gpurun_out/r05_multirank.log 2>&1; tail -1 gpurun_out/r05_multirank.log
for n in 4 2; do
timeout 1200 $P --nproc-per-node $n --master-port 2994$n bench_configs.py --config 3 --steps 1000 --engines persistent --out gpurun_out/r05_cfg3_n$n.jsonl > gpurun_out/r05_cfg3_n$n.log 2>&1; echo "cfg3 n$n rc=$?"
python -c "
import json
d=json.loads(open('gpurun_out/r05_cfg3_n$n.jsonl').readlines()[-1]); x=d['exchange_us']; print($n, d['steps_per_s'], x['p50'], x['p99'], d['clocks']['sm_mhz'])"
done
