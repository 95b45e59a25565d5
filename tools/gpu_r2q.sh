#!/bin/bash
O=gpurun_out/r2q; mkdir -p $O
./tools/launch_probe | tee $O/launch_probe.txt
SG_LIB_PATH=abtest/tprobe.so timeout 300 python3 bench.py --steps 20 --fuse 20 --warmup 5 --no-cpu-baseline --e2e-steps 0 2>&1 | grep tprobe | tail -n 6 | tee $O/tprobe.txt
timeout 300 python3 bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 0 > $O/k20.log 2>&1; tail -n 1 $O/k20.log | cut -c1-300
