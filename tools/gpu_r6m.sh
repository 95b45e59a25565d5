#!/bin/bash
# Final tree check on one B200: GPU tests, smoke, driver command, reference arm, PPO line.
O=gpurun_out/r6m; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo pytest rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$?
timeout 600 python3 bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench_driver.log 2>&1; echo driver rc=$?
timeout 600 python3 bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $O/bench_ref.log 2>&1; echo ref rc=$?
timeout 900 python3 bench.py --config ppo > $O/bench_ppo.log 2>&1; echo ppo rc=$?
tail -n 3 $O/pytest_gpu.log; tail -n 1 $O/smoke.log
for f in $O/bench_*.log; do echo "$f: $(tail -n 1 $f | cut -c1-220)"; done
