#!/bin/bash
# Re-entry check on one B200 after the container rebuild: GPU tests, smoke, driver command, reference arm.
O=gpurun_out/r6a; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo pytest rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$?
timeout 600 python3 bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench_driver.log 2>&1; echo driver rc=$?
timeout 600 python3 bench.py > $O/bench_psm_default.log 2>&1; echo psm rc=$?
tail -n 3 $O/pytest_gpu.log; tail -n 1 $O/smoke.log
for f in $O/bench_*.log; do echo "$f: $(tail -n 1 $f | cut -c1-300)"; done
