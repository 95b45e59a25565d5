#!/bin/bash
O=gpurun_out/r3s; mkdir -p $O
timeout 900 ncu --clock-control none --metrics gpu__time_duration.sum --csv --log-file $O/launches_ppo.csv \
  python3 bench.py --config ppo --steps 32 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo rc=$?
