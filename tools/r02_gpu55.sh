#!/bin/bash
# lean row-sum A/B: per-rank kernel at 1/4/8 virtual ranks, config-2 bench kernel, config-3 pull, ncu instruction count
mkdir -p gpurun_out
o=gpurun_out/r02_fma_ab.jsonl; : > $o
for rep in 1 2; do
  for l in default variants/fma; do
    if [ $l = default ]; then E=""; else E="NEUROCOMM_B200_LIB=$l/libneurocomm_b200.so"; fi
    env $E timeout 900 python tools/vr_kernel.py --worlds 1,4,8 --steps 200 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); d['lib']='$l'; print(json.dumps(d))" | tee -a $o
    env $E timeout 900 python bench.py --steps 300 --warmup 5 --no-cpu --no-push --no-e2e-api 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(json.dumps({'lib':'$l','bench':d['value'],'kernel_ms':d['roofline']['kernel_ms'],'frac':d['roofline']['frac'],'mhz':d['clocks']['sm_mhz']}))" | tee -a $o
  done
done
for l in default variants/fma; do
  if [ $l = default ]; then E=""; else E="NEUROCOMM_B200_LIB=$l/libneurocomm_b200.so"; fi
  env $E timeout 600 ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_step_fused -s 10 -c 1 --csv \
    python bench.py --steps 20 --warmup 3 --no-cpu --no-push --no-e2e-api 2>/dev/null | grep -E "inst_executed|duration|alu" | sed "s#^#$l #" | tee -a gpurun_out/r02_fma_ncu.txt
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "tiled or config2 or fused or two_level or matches or persistent" > gpurun_out/r02_fma_tests.log 2>&1; tail -1 gpurun_out/r02_fma_tests.log
for l in default variants/fma; do
  if [ $l = default ]; then E=""; else E="NEUROCOMM_B200_LIB=$l/libneurocomm_b200.so"; fi
  env $E timeout 900 python bench_configs.py --config 3 --engines fused --steps 300 --out /dev/stdout 2>/dev/null | grep '"engine"' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$l cfg3', d['steps_per_s'], d['kernel_ms'], d['clocks']['sm_mhz'])" | tee -a gpurun_out/r02_fma_ab.jsonl.txt
done
