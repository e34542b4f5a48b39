#!/bin/bash
# persistent engine: own-spike push overlapped with the exchange -- parity + A/B at config 3 N=2/4
mkdir -p gpurun_out
P="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "multirank or persistent or windowed or push" > gpurun_out/r12_tests.log 2>&1; tail -1 gpurun_out/r12_tests.log
o=gpurun_out/r12_overlap_ab.txt; : > $o
for rep in 1 2; do
for l in default variants/noov; do
  if [ $l = default ]; then E=""; else E="NEUROCOMM_B200_LIB=$l/libneurocomm_b200.so"; fi
  for n in 4 2; do
    env $E timeout 900 $P --nproc-per-node $n --master-port 2990$n bench_configs.py --config 3 --engines persistent,fused --steps 1000 --out gpurun_out/r12_$n.jsonl > /dev/null 2>&1
    python -c "
import json
for l in open('gpurun_out/r12_$n.jsonl'):
    d=json.loads(l)
    if 'engine' in d and d['engine']=='persistent': x=d['exchange_us']; print('$l', $n, d['steps_per_s'], x['p50'], x['p99'])
    if 'cross_engine_state_agreement' in d: print('$l', $n, 'agree', d['cross_engine_state_agreement'])
" | tee -a $o
    rm -f gpurun_out/r12_$n.jsonl
  done
done
done
