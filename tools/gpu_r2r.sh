#!/bin/bash
# Noise-ahead rollout: parity, policy/ppo bench lines, policy prologue probe.
O=gpurun_out/r2r; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_policy.py tests/test_gpu_ppo.py -q -x > $O/pytest.log 2>&1; echo pytest rc=$?
tail -n 3 $O/pytest.log
timeout 600 python3 bench.py --config policy --steps 640 > $O/bench_policy.log 2>&1; echo policy rc=$?
tail -n 1 $O/bench_policy.log | cut -c1-700
timeout 900 python3 bench.py --config ppo --no-cpu-baseline > $O/bench_ppo.log 2>&1; echo ppo rc=$?
tail -n 1 $O/bench_ppo.log | cut -c1-900
SG_LIB_PATH=abtest/pprobe.so timeout 300 python tools/policy_probe.py 2>&1 | grep pprobe | tail -n 8
timeout 300 python tools/policy_probe.py 2>&1 | tail -n 5
