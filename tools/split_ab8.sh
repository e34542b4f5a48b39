# N=8-like per-GPU load (125k rows x 1k synapses) on 4 GPUs: 500k-neuron network, forced tile counts
for s in 0 1 2; do
for tw in 7840 3936 1984; do
  NC_BLOCK_SPLIT=$s python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29561 \
    bench.py --gpus 4 --neurons 500000 --steps 1000 --warmup 20 --no-push --no-cpu --tile-words $tw 2>/dev/null | tail -n 1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('split=$s tw=$tw tiles', d['config']['bitmap_tiles'], 'value', d['value'], 'kernel_ms', d['roofline']['kernel_ms'], 'frac', d['roofline']['frac'], 'ms', d['ms_per_step'])"
done; done
