#!/bin/bash
# spike-list push in the persistent engine: parity tests (1 GPU + 4 GPU multirank) and config 3 at N = 1/2/4
mkdir -p gpurun_out
P="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/r04_gpu_tests.log 2>&1
tail -2 gpurun_out/r04_gpu_tests.log
CUDA_VISIBLE_DEVICES=0 timeout 600 python tools/persistent_phases.py 10000000 2>&1 | tail -2; CUDA_VISIBLE_DEVICES=0 timeout 600 python tools/persistent_phases.py 1000000 2>&1 | tail -2
timeout 1200 $P --nproc-per-node 4 --master-port 29931 bench_configs.py --config 3 --steps 1000 --engines persistent --out gpurun_out/r04_cfg3_n4.jsonl > gpurun_out/r04_cfg3_n4.log 2>&1; echo "cfg3 n4 rc=$?"
timeout 1200 $P --nproc-per-node 2 --master-port 29932 bench_configs.py --config 3 --steps 1000 --engines persistent --out gpurun_out/r04_cfg3_n2.jsonl > gpurun_out/r04_cfg3_n2.log 2>&1; echo "cfg3 n2 rc=$?"
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench_configs.py --config 3 --steps 1000 --engines persistent --out gpurun_out/r04_cfg3_n1.jsonl > gpurun_out/r04_cfg3_n1.log 2>&1; echo "cfg3 n1 rc=$?"
python - <<'PY'
import json
for n in (1, 2, 4):
    try:
        for l in open(f'gpurun_out/r04_cfg3_n{n}.jsonl'):
            d = json.loads(l); x = d.get('exchange_us') or {}
            print(n, d['engine'], d['steps_per_s'], x.get('p50'), x.get('p99'), d['clocks']['sm_mhz'])
    except Exception as e:
        print(n, 'error', e)
PY
