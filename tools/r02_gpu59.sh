#!/bin/bash
# final 4-GPU pass on the final kernel
mkdir -p gpurun_out
P="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r09_gpu_tests_4gpu.log 2>&1
tail -1 gpurun_out/r09_gpu_tests_4gpu.log
for n in 2 4; do
  timeout 900 $P --nproc-per-node $n --master-port 2999$n bench.py --gpus $n --steps 300 --warmup 20 > gpurun_out/r09_bench_n$n.json 2> gpurun_out/r09_bench_n$n.err; echo "bench n=$n rc=$?"
  python -c "
import json
d=json.loads(open('gpurun_out/r09_bench_n$n.json').read().strip().splitlines()[-1]); x=d['exchange_us']
print($n, d['value'], d['roofline']['frac'], d['roofline']['kernel_ms'], x['p50'], x['p99'], x['p50_transfer_only'], d['e2e']['value'], d['event_driven']['value'])"
done
timeout 1200 $P --nproc-per-node 4 --master-port 29971 bench_configs.py --config 3 --steps 1000 --out gpurun_out/r09_cfg3_n4.jsonl > gpurun_out/r09_cfg3_n4.log 2>&1; echo "cfg3 n4 rc=$?"
timeout 1200 $P --nproc-per-node 2 --master-port 29972 bench_configs.py --config 3 --steps 1000 --out gpurun_out/r09_cfg3_n2.jsonl > gpurun_out/r09_cfg3_n2.log 2>&1; echo "cfg3 n2 rc=$?"
