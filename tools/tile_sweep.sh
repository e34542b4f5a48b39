#!/bin/bash
# Pull-kernel roofline fraction vs bitmap tile size: tools/tile_sweep.sh N "tw1 tw2 ..." [extra bench args]
n=$1; shift; tws=$1; shift
for tw in $tws; do
  python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29512 \
    bench.py --gpus $n --steps 100 --warmup 5 --no-push --tile-words $tw "$@" 2>/dev/null | tail -n 1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('N=$n tw=$tw tiles', d['config']['bitmap_tiles'], 'value', d['value'], 'kernel_ms', d['roofline']['kernel_ms'], 'frac', d['roofline']['frac'])"
done
