#!/bin/bash
# Launch timeline of the fused step (globaltimer probe) at K = 1, 20, 250, cold (L2 flushed) and warm.
O=gpurun_out/r2f; mkdir -p $O
for K in 1 20 250; do for F in "" "--no-flush"; do
  echo "== K=$K $F"
  SG_LIB_PATH=abtest/tprobe.so timeout 300 python3 bench.py --steps $K --fuse $K --warmup 5 --runs 5 --e2e-steps 0 --no-cpu-baseline $F 2>&1 | grep -E "tprobe K=$K" | tail -3
  timeout 300 python3 bench.py --steps $K --fuse $K --warmup 5 --runs 5 --e2e-steps 0 --no-cpu-baseline $F 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('event-timed', d['roofline']['avg_launch_us'], 'us', d['runs']['ms_per_run'])"
done; done > $O/timeline.txt 2>&1
cat $O/timeline.txt
