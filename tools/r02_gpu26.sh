#!/bin/bash
# A/B: inhibitory ids grouped after the excitatory ones (default) vs degree order only; pull kernel
mkdir -p gpurun_out
for r in 1 2; do
for v in "" "--no-ei-group"; do
  for n in 1000000 10000000; do
    timeout 900 python bench_configs.py --config 3 --neurons $n --engines fused --steps 300 --warmup 20 $v \
      --out gpurun_out/r02_eigroup_ab.jsonl > /dev/null 2>&1
  done
done; done
python -c "
import json
for l in open('gpurun_out/r02_eigroup_ab.jsonl'):
    d=json.loads(l); print(d['neurons'], 'ei_group', d['ei_group'], d['steps_per_s'], d['kernel_ms'], d['pull_layout_bytes_per_synapse'], d['bitmap_tiles'], d['clocks']['sm_mhz'])"
