#!/bin/bash
# final-code ncu captures: config-2 pull kernel (bench default network) and config-3 pull kernel (20 tiles)
mkdir -p gpurun_out
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu --no-push --no-e2e-api > gpurun_out/r02_final_plain.json 2>&1; echo "plain rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step_fused -s 10 -c 1 -o gpurun_out/r02_final_step_fused \
  python bench.py --steps 20 --warmup 3 --no-cpu --no-push --no-e2e-api > gpurun_out/r02_final_step_fused_ncu.log 2>&1; echo "ncu cfg2 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_final_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-push --no-e2e-api > gpurun_out/r02_final_launches.log 2>&1; echo "launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_step_fused -s 30 -c 1 -o gpurun_out/r02_final_cfg3_pull \
  python bench_configs.py --config 3 --engines fused --steps 40 --warmup 5 > gpurun_out/r02_final_cfg3_pull_ncu.log 2>&1; echo "ncu cfg3 rc=$?"
