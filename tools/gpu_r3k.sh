#!/bin/bash
O=gpurun_out/r3k; mkdir -p $O
timeout 600 ncu --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file $O/launches.csv \
  python3 bench.py --config ppo --steps 32 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo rc=$?
timeout 600 ncu --clock-control none --set full --import-source on -k regex:policy_dgrad_elu_kernel -s 6 -c 3 -o $O/dgrad \
  python3 bench.py --config ppo --steps 32 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo rc=$?
