#!/bin/bash
O=gpurun_out/r3c; mkdir -p $O
timeout 600 ncu --clock-control none --metrics gpu__time_duration.sum --csv --log-file $O/launches_policy.csv \
  python3 bench.py --config policy --steps 64 --warmup 3 --runs 1 --no-cpu-baseline --e2e-steps 0 > $O/policy.log 2>&1; echo rc=$?
