#!/bin/bash
O=gpurun_out/r2i; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo pytest rc=$?
timeout 600 python3 bench.py --config policy --steps 640 > $O/bench_policy.log 2>&1; echo policy rc=$?
timeout 900 python3 bench.py --config ppo --no-cpu-baseline > $O/bench_ppo.log 2>&1; echo ppo rc=$?
timeout 600 ncu --clock-control none --metrics gpu__time_duration.sum --csv --log-file $O/launches_policy.csv \
  python3 bench.py --config policy --steps 64 --warmup 3 --runs 1 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
timeout 600 ncu --clock-control none --set full --import-source on -k regex:policy_fwd_kernel -s 40 -c 1 -o $O/policy_fwd \
  python3 bench.py --config policy --steps 64 --warmup 3 --runs 1 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
tail -15 $O/pytest_gpu.log; tail -1 $O/bench_policy.log | cut -c1-1500; tail -1 $O/bench_ppo.log | cut -c1-1200
