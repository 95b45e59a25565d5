#!/bin/bash
O=gpurun_out/r2y; mkdir -p $O
timeout 600 ncu --clock-control none --set full --import-source on -k regex:policy_train_fwd_kernel -s 20 -c 1 -o $O/train_fwd \
  python3 bench.py --config ppo --steps 32 --warmup 2 --no-cpu-baseline > /dev/null 2>&1
ncu -i $O/train_fwd.ncu-rep --page details --csv > $O/train_fwd_details.csv 2>/dev/null
grep -E '"Duration"|Issue Slots Busy|Achieved Occupancy|DRAM Throughput"|Memory Throughput' $O/train_fwd_details.csv | cut -c110-230
timeout 600 ncu --clock-control none --metrics gpu__time_duration.sum --csv --log-file $O/launches_ppo.csv \
  python3 bench.py --config ppo --steps 32 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo rc=$?
