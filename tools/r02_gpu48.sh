#!/bin/bash
# L2 evict-first synapse stream A/B: config 3 pull (global partials) and config 2 pull
mkdir -p gpurun_out
o=gpurun_out/r02_evict_ab.log; : > $o
for l in default variants/ef default variants/ef; do
  if [ $l = default ]; then E=""; else E="NEUROCOMM_B200_LIB=$l/libneurocomm_b200.so"; fi
  r=$(env $E timeout 900 python bench_configs.py --config 3 --engines fused --steps 200 --out /dev/stdout 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg3', d['steps_per_s'], d['kernel_ms'], d['clocks']['sm_mhz'])")
  echo "$l $r" | tee -a $o
  r=$(env $E timeout 900 python bench.py --steps 200 --warmup 5 --no-cpu --no-push --no-e2e-api 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg2', d['value'], d['roofline']['kernel_ms'], d['roofline']['frac'], d['clocks']['sm_mhz'])")
  echo "$l $r" | tee -a $o
done
