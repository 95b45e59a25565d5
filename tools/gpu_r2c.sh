#!/bin/bash
# Phase probe of the two-warp team kernel + saturating-dynamics variant A/B.
O=gpurun_out/r2c; mkdir -p $O
SG_LIB_PATH=abtest/probe.so timeout 300 python3 bench.py --steps 250 --fuse 250 --warmup 1 --runs 1 --e2e-steps 0 --no-cpu-baseline > $O/probe.log 2>&1
SG_LIB_PATH=abtest/sat.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q > $O/pytest_sat.log 2>&1; echo sat pytest rc=$?
for rep in 1 2; do for lib in paper_2310_04676_b200/lib/libsg_env.so abtest/sat.so; do for cfg in psm ecm star; do
  for K in 20 250; do
    ST=$K; [ $K = 250 ] && ST=20000
    SG_LIB_PATH=$lib timeout 300 python3 bench.py --config $cfg --steps $ST --fuse $K --warmup 5 --no-cpu-baseline --e2e-steps 0 2>&1 | tail -1 | \
      python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg K=$K', '$lib', round(d['value']/1e9, 3), 'G', round(d['roofline']['avg_launch_us'],2), 'us')"
  done; done; done; done > $O/ab.txt 2>&1
cat $O/ab.txt; grep "probe cta" $O/probe.log | tail -12; tail -3 $O/pytest_sat.log
