#!/bin/bash
# Policy forward v2 (TMEM-resident activations, actor / critic pipelines): parity, bench, ncu.
O=gpurun_out/r2l; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_policy.py tests/test_gpu_ppo.py -q -x > $O/pytest_policy.log 2>&1; echo pytest rc=$?
tail -15 $O/pytest_policy.log
timeout 600 python3 bench.py --config policy --steps 640 --no-cpu-baseline > $O/bench_policy.log 2>&1; echo policy rc=$?
timeout 600 ncu --clock-control none --set full --import-source on -k regex:policy_fwd_kernel -s 40 -c 1 -o $O/policy_fwd \
  python3 bench.py --config policy --steps 64 --warmup 3 --runs 1 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
ncu -i $O/policy_fwd.ncu-rep --page details --csv > $O/policy_fwd_details.csv 2>/dev/null
ncu -i $O/policy_fwd.ncu-rep --page raw --csv > $O/policy_fwd_raw.csv 2>/dev/null
tail -1 $O/bench_policy.log | cut -c1-1800
