#!/bin/bash
O=gpurun_out/r3w; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_ppo.py -q -x -k "wgrad" > $O/pytest_wgrad.log 2>&1; echo wgrad pytest rc=$?
tail -n 2 $O/pytest_wgrad.log
timeout 600 python tools/wgrad_probe.py 2>&1 | tail -n 4
