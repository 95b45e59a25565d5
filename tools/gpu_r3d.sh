#!/bin/bash
O=gpurun_out/r3d; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_ppo.py tests/test_gpu_policy.py -q -x > $O/pytest.log 2>&1; echo pytest rc=$?
tail -n 3 $O/pytest.log
for rep in 1 2; do
timeout 600 python3 bench.py --config policy --steps 640 --no-cpu-baseline --e2e-steps 0 > $O/policy_$rep.log 2>&1
python3 -c "
import json; l=json.loads(open('$O/policy_$rep.log').read().strip().splitlines()[-1])
print('policy', round(l['value']/1e6,1), 'M/s  fwd us', round(l['roofline']['avg_launch_us'],2))" 2>&1 | tail -n 1
done
timeout 900 python3 bench.py --config ppo --no-cpu-baseline > $O/ppo.log 2>&1
python3 -c "
import json; l=json.loads(open('$O/ppo.log').read().strip().splitlines()[-1]); c=l['config']
print('ppo', round(l['value']/1e6,2), 'M/s rollout', round(c['rollout_ms_per_iter'],3), 'update', round(c['update_ms_per_iter'],3))" 2>&1 | tail -n 1
