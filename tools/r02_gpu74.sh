#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "upload_edges or device_edge or simulate or config2" 2>&1 | tail -1
timeout 600 python tools/e2e_api_breakdown.py > gpurun_out/r02_e2e_api_breakdown4.json 2> gpurun_out/r02_e2e_api_breakdown4.err; cat gpurun_out/r02_e2e_api_breakdown4.json
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu --no-push 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('e2e_api', d['e2e_api'])"
