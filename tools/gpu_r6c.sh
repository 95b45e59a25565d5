#!/bin/bash
# Launch-path probe + in-kernel globaltimer phases of the PSM K=20 launch.
O=gpurun_out/r6c; mkdir -p $O
./tools/launch_probe2 | tee $O/launch_probe2.txt
SG_LIB_PATH=abtest/tprobe.so timeout 300 python3 bench.py --config psm --steps 20 --fuse 20 --warmup 5 --no-cpu-baseline --e2e-steps 5 > $O/tprobe20.log 2>&1
grep tprobe $O/tprobe20.log | tail -8
SG_LIB_PATH=abtest/tprobe.so timeout 300 python3 bench.py --config psm --steps 80 --fuse 80 --warmup 5 --no-cpu-baseline --e2e-steps 5 > $O/tprobe80.log 2>&1
grep tprobe $O/tprobe80.log | tail -4
