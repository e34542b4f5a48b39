#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_virtual_ranks.py tests/test_gpu_parity.py -q -p no:cacheprovider -k "virtual or two_level or config1 or persistent" > gpurun_out/r02_t16.log 2>&1
tail -3 gpurun_out/r02_t16.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
echo done
