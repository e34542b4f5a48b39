#!/bin/bash
# driver-equivalent pass on one GPU: build check, GPU tests, smoke, bench (driver flags and default), reference arm
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02_final_gpu_tests.log 2>&1
tail -3 gpurun_out/r02_final_gpu_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_final_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_final_bench_s20.json 2> gpurun_out/r02_final_bench_s20.err; echo "bench rc=$?"
timeout 900 python bench.py > gpurun_out/r02_final_bench.json 2> gpurun_out/r02_final_bench.err; echo "bench default rc=$?"
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02_final_ref.json 2> gpurun_out/r02_final_ref.err; echo "ref rc=$?"
echo done
