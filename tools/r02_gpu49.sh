#!/bin/bash
# final 4-GPU pass: every GPU test, config 2 N=2/4 bench, config 3 persistent N=4 (1000 steps)
mkdir -p gpurun_out
P="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r07_gpu_tests_4gpu.log 2>&1
tail -1 gpurun_out/r07_gpu_tests_4gpu.log
for n in 2 4; do
  timeout 900 $P --nproc-per-node $n --master-port 2998$n bench.py --gpus $n --steps 300 --warmup 20 > gpurun_out/r07_bench_n$n.json 2> gpurun_out/r07_bench_n$n.err; echo "bench n=$n rc=$?"
  python -c "
import json
d=json.loads(open('gpurun_out/r07_bench_n$n.json').read().strip().splitlines()[-1]); x=d['exchange_us']
print($n, d['value'], d['roofline']['frac'], x['p50'], x['p99'], d['e2e']['value'], d['event_driven']['value'])"
done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
