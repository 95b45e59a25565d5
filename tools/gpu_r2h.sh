#!/bin/bash
O=gpurun_out/r2h; mkdir -p $O
./build/launch_probe > $O/launch_probe.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "k20 or control or star_path_following_shards" > $O/pytest.log 2>&1; echo pytest rc=$?
timeout 600 ncu --clock-control none --metrics gpu__time_duration.sum --csv --log-file $O/launches_policy.csv \
  python3 bench.py --config policy --steps 64 --warmup 3 --runs 1 --no-cpu-baseline --e2e-steps 0 > $O/policy.log 2>&1
cat $O/launch_probe.txt; tail -3 $O/pytest.log
