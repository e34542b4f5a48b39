#!/bin/bash
# final pass after the lean row sum: 1-GPU driver-equivalent + ncu capture of the config-2 kernel
bash tools/r02_final1.sh
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step_fused -s 10 -c 1 -o gpurun_out/r02_final2_step_fused \
  python bench.py --steps 20 --warmup 3 --no-cpu --no-push --no-e2e-api > gpurun_out/r02_final2_step_fused_ncu.log 2>&1; echo "ncu rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_final2_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-push --no-e2e-api > gpurun_out/r02_final2_launches.log 2>&1; echo "launches rc=$?"
