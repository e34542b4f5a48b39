#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "aggregate or genetic" > gpurun_out/r02_k5b_tests.log 2>&1; tail -1 gpurun_out/r02_k5b_tests.log
timeout 600 python tools/k5_kernel_ab.py 2>&1 | tail -1
timeout 600 python tools/planner_bench.py --sizes 1000000 > gpurun_out/r02_planner_1e6b.json 2>&1; tail -1 gpurun_out/r02_planner_1e6b.json
timeout 600 python -c "
import time, torch, sys
sys.path.insert(0, '.')
from paper_2205_07125_b200 import sim as S, traffic as T, PartitionMap
import numpy as np
spec = S.GeneratorSpec.random(10_000_000, 1000.0, seed=1)
pm = PartitionMap(4, np.repeat(np.arange(4), 2_500_000))
T.aggregate_generated(spec, pm); torch.cuda.synchronize()
t = time.time(); gt = T.aggregate_generated(spec, pm); torch.cuda.synchronize(); print('aggregate_generated config 3', round(time.time() - t, 4), 's')
"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_histogram_smem -c 1 -o gpurun_out/r02_k5e python tools/k5_kernel_ab.py > gpurun_out/r02_k5e_ncu.log 2>&1; echo "ncu rc=$?"
