#!/bin/bash
# A/B the kernel variants in variants/*.so on one bench command: tools/ab_libs.sh "<bench args>" lib1 lib2 ...
args="$1"; shift
for l in "$@"; do
  NEUROCOMM_B200_LIB=$l python bench.py $args 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$l', d['config'].get('neurons'), 'value', d['value'], 'kernel_ms', d['roofline']['kernel_ms'], 'frac', d['roofline']['frac'])"
done
