#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs_downscaled.py -q -p no:cacheprovider -k "generated or generator or config2 or config3 or config5 or aggregate or push" > gpurun_out/r02_t19.log 2>&1
tail -15 gpurun_out/r02_t19.log
python - <<'PY' > gpurun_out/r02_aggregate_generated.log 2>&1
import sys, time; sys.path.insert(0, '.')
import numpy as np, torch
import paper_2205_07125_b200 as nc
from paper_2205_07125_b200 import sim as S
for n, c, deg, gpus in [(10_000_000, 1, 1000.0, 4), (50_000_000, 64, 1000.0, 4)]:
    if c == 1:
        spec = S.GeneratorSpec.random(n, deg, seed=1)
    else:
        size = n / c
        spec = S.GeneratorSpec(n, c, 0.9 * deg / (size - 1), 0.1 * deg / (n - size), seed=1)
    lay = S.ShardLayout.blocks(n, gpus)
    pm = nc.PartitionMap(gpus, lay.owner.astype(np.int64))
    nc.traffic.aggregate_generated(S.GeneratorSpec.random(1000, 10.0), nc.PartitionMap(gpus, np.arange(1000) % gpus))
    torch.cuda.synchronize(); t = time.time()
    gt = nc.traffic.aggregate_generated(spec, pm)
    torch.cuda.synchronize(); dt = time.time() - t
    print({"neurons": n, "communities": c, "gpus": gpus, "seconds": round(dt, 2), "pg_sum": float(gt.pg.sum()),
           "diag_frac": float(np.trace(gt.pg) / gt.pg.sum())}, flush=True)
PY
cat gpurun_out/r02_aggregate_generated.log
