#!/bin/bash
# First round-2 GPU pass: tests, the driver's headline command (gated and the
# round-1 ungated protocol), the default bench, the random-init-policy line,
# and the K=20 / K=250 ncu captures.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
timeout 300 python3 bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_k20.log 2>&1; echo k20 rc=$?
timeout 300 python3 bench.py --gpus 1 --steps 20 --warmup 5 --no-gate --no-cpu-baseline > gpurun_out/bench_k20_nogate.log 2>&1
timeout 600 python3 bench.py --no-cpu-baseline > gpurun_out/bench_default.log 2>&1; echo default rc=$?
timeout 600 python3 bench.py --config policy --steps 640 > gpurun_out/bench_policy.log 2>&1; echo policy rc=$?
bash tools/profile_r2.sh psm gpurun_out/prof_r2
tail -n 2 gpurun_out/*.log | cut -c1-3000
