#!/bin/bash
# K5 uniform wrapper (device narrowing) + upload pipeline + device raster: tests and timings
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "aggregate or genetic or upload_edges or device_edge or simulate or config2" > gpurun_out/r02_gpu29_tests.log 2>&1
tail -2 gpurun_out/r02_gpu29_tests.log
timeout 600 python tools/k5_wrapper_profile.py > gpurun_out/r02_k5_wrapper2.log 2>&1; head -c 600 gpurun_out/r02_k5_wrapper2.log; echo
timeout 600 python tools/planner_bench.py --sizes 1000000 > gpurun_out/r02_planner_1e6.json 2>&1; tail -1 gpurun_out/r02_planner_1e6.json
timeout 600 python tools/e2e_api_breakdown.py > gpurun_out/r02_e2e_api_breakdown2.json 2> gpurun_out/r02_e2e_api_breakdown2.err; cat gpurun_out/r02_e2e_api_breakdown2.json
