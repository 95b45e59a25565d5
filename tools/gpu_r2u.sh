#!/bin/bash
O=gpurun_out/r2u; mkdir -p $O
./tools/launch_probe | tee $O/launch_probe.txt
timeout 900 ncu --clock-control none --metrics gpu__time_duration.sum --csv --log-file $O/launches_ppo.csv \
  python3 bench.py --config ppo --steps 32 --warmup 3 --no-cpu-baseline > $O/ppo.log 2>&1; echo ncu rc=$?
ls -la $O
