#!/bin/bash
# Strong-scaling pull kernel vs forced bitmap tile count: tools/strong_tiles.sh N "tw1 tw2 ..."
n=$1; tws=$2
for tw in $tws; do
  extra=""; [ "$tw" != "auto" ] && extra="--tile-words $tw"
  python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29541 \
    bench.py --gpus $n --steps 1000 --warmup 20 --no-push --no-cpu $extra 2>/dev/null | tail -n 1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('N=$n tw=$tw tiles', d['config']['bitmap_tiles'], 'value', d['value'], 'kernel_ms', d['roofline']['kernel_ms'], 'frac', d['roofline']['frac'], 'e2e', d['e2e']['value'])"
done
