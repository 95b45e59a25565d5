#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_ppo.py -q -x -k "wgrad" 2>&1 | tail -n 2
timeout 600 python tools/wgrad_probe.py 2>&1 | tail -n 4
echo partials:; SG_WGRAD_PARTIALS=1 timeout 600 python tools/wgrad_probe.py 2>&1 | tail -n 4 | head -n 3
