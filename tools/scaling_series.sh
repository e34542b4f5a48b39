#!/bin/bash
# The driver's series: bench.py at N = 1, 2, 4 (default flags) + the reference arm at N=1.
# Output: gpurun_out/series_n{N}.json, gpurun_out/series_ref_n1.json
python bench.py > gpurun_out/series_n1.json 2> gpurun_out/series_n1.err; echo "n=1 rc=$?"
for n in 2 4; do
  python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2955$n \
    bench.py --gpus $n > gpurun_out/series_n$n.json 2> gpurun_out/series_n$n.err; echo "n=$n rc=$?"
done
python bench.py --impl reference > gpurun_out/series_ref_n1.json 2> gpurun_out/series_ref_n1.err; echo "ref rc=$?"
