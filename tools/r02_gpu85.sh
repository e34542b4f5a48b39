#!/bin/bash
mkdir -p gpurun_out
P="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r15_gpu_tests_4gpu.log 2>&1; tail -1 gpurun_out/r15_gpu_tests_4gpu.log
timeout 1200 $P --nproc-per-node 4 --master-port 29986 bench_configs.py --config 3 --steps 1000 --out gpurun_out/r15_cfg3_n4.jsonl > gpurun_out/r15_cfg3_n4.log 2>&1; echo "cfg3 n4 rc=$?"
timeout 1200 $P --nproc-per-node 2 --master-port 29987 bench_configs.py --config 3 --steps 1000 --out gpurun_out/r15_cfg3_n2.jsonl > gpurun_out/r15_cfg3_n2.log 2>&1; echo "cfg3 n2 rc=$?"
for n in 2 4; do
  timeout 900 $P --nproc-per-node $n --master-port 2998$n bench.py --gpus $n --steps 300 --warmup 20 > gpurun_out/r15_bench_n$n.json 2> gpurun_out/r15_bench_n$n.err; echo "bench n=$n rc=$?"
done
python - <<'PY'
import json
for f in ['r15_cfg3_n2','r15_cfg3_n4']:
    for l in open(f'gpurun_out/{f}.jsonl'):
        d=json.loads(l)
        if 'engine' not in d: print(f, 'agree', d.get('cross_engine_state_agreement')); continue
        x=d['exchange_us'] or {}
        print(f, d['engine'], d['steps_per_s'], x.get('p50'), x.get('p99'), x.get('p50_transfer_only'))
for n in (2, 4):
    d=json.loads(open(f'gpurun_out/r15_bench_n{n}.json').read().strip().splitlines()[-1]); x=d['exchange_us']
    print('bench', n, d['value'], d['roofline']['frac'], x['p50'], x['p99'], x['p50_transfer_only'], d['e2e']['value'], d['event_driven']['value'])
PY
