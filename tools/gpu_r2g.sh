#!/bin/bash
# Host-step (e2e) A/B: completion-flag polling x residency floor (waves).
O=gpurun_out/r2g; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cpp.py -q -x -k "host or cpp" > $O/pytest_host.log 2>&1; echo host tests rc=$?
for rep in 1 2; do for poll in 0 1; do for floor in 0 60000 100000 160000; do
  SG_HOST_POLL=$poll SG_HOST_SMEM_FLOOR=$floor timeout 300 python3 bench.py --steps 300 --e2e-steps 600 --runs 1 --no-cpu-baseline 2>&1 | tail -1 | \
    python3 -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('poll=$poll floor=$floor', round(e['value']/1e6,1), 'M env-steps/s', round(16384/e['value']*1e6,2), 'us/step', 'bursts', e['reset_burst_steps'])"
done; done; done > $O/ab.txt 2>&1
cat $O/ab.txt; tail -3 $O/pytest_host.log
