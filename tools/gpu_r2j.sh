#!/bin/bash
# Round-2 re-entry check: GPU tests, smoke, the driver's headline bench, and the
# K=20 / K=250 ncu captures of the headline kernel (profiles/r2).
O=gpurun_out/r2j; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo pytest rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo smoke rc=$?
timeout 600 python3 bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench_k20.log 2>&1; echo bench rc=$?
timeout 600 python3 bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $O/bench_ref.log 2>&1; echo ref rc=$?
timeout 1200 bash tools/profile_r2.sh psm $O/prof > $O/prof.log 2>&1; echo prof rc=$?
tail -5 $O/pytest_gpu.log; tail -2 $O/smoke.log; tail -1 $O/bench_k20.log | cut -c1-3000; tail -1 $O/bench_ref.log | cut -c1-600
