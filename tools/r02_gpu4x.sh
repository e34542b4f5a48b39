#!/bin/bash
# 4-GPU pass: multi-rank parity, driver-style bench at N=2/4, configs 3/4/5 at real size
mkdir -p gpurun_out
nvidia-smi topo -m > gpurun_out/r02_topo.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "aggregate or genetic" > gpurun_out/r02_k5_tests.log 2>&1
tail -1 gpurun_out/r02_k5_tests.log
timeout 300 python tools/planner_bench.py --sizes 1000000 > gpurun_out/r02_planner5.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_histogram_smem -c 1 -o gpurun_out/r02_k5c -f python tools/planner_bench.py --sizes 1000000 > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_multirank.py -q -p no:cacheprovider > gpurun_out/r02_multirank.log 2>&1
tail -2 gpurun_out/r02_multirank.log
for n in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2970$n \
    bench.py --gpus $n --steps 300 --warmup 20 > gpurun_out/r02_bench_n$n.json 2> gpurun_out/r02_bench_n$n.err
done
run() { # n config extra...
  local n=$1; shift; local c=$1; shift
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29811 \
    bench_configs.py --config $c --out gpurun_out/r02_cfg${c}_n$n.jsonl "$@" > gpurun_out/r02_cfg${c}_n$n.log 2>&1
  echo "cfg$c n=$n rc=$?"
}
run 2 3
run 4 3
run 4 4
run 4 5
run 2 5 --engines persistent
echo done
