#!/bin/bash
timeout 600 python tools/lif_time.py 2>&1 | tail -1
timeout 600 python tools/persistent_phases.py 10000000 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "push or persistent or binned or windowed" 2>&1 | tail -1
