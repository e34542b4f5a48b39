#!/bin/bash
mkdir -p gpurun_out
o=gpurun_out/r02_unroll_ab.jsonl; : > $o
for rep in 1 2; do
  for l in default variants/u6 variants/u10 variants/u12; do
    if [ $l = default ]; then E=""; else E="NEUROCOMM_B200_LIB=$l/libneurocomm_b200.so"; fi
    env $E timeout 900 python tools/vr_kernel.py --worlds 1,4,8 --steps 200 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); d['lib']='$l'; print(json.dumps(d))" | tee -a $o
  done
done
