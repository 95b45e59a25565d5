#!/bin/bash
# ncu --set full of the policy forward / act kernel inside the random-init-policy rollout (one launch),
# plus the PPO config line with its CPU baseline and e2e.
O=gpurun_out/r6i; mkdir -p $O
timeout 900 python3 bench.py --config ppo > $O/bench_ppo.log 2>&1; echo ppo rc=$?; tail -n 1 $O/bench_ppo.log | cut -c1-400
timeout 900 ncu --set full --clock-control none --import-source on -k regex:policy_fwd_kernel -s 40 -c 1 \
  -o $O/policy_fwd python3 bench.py --config policy --steps 64 --runs 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/ncu_policy.log 2>&1; echo ncu rc=$?
tail -3 $O/ncu_policy.log
ncu -i $O/policy_fwd.ncu-rep --page details --csv > $O/policy_fwd_details.csv 2>&1
ncu -i $O/policy_fwd.ncu-rep --page raw --csv > $O/policy_fwd_raw.csv 2>&1
ls -la $O
