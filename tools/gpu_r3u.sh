#!/bin/bash
O=gpurun_out/r3u; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_ppo.py -q -x -k "wgrad" > $O/pytest_wgrad.log 2>&1; echo wgrad pytest rc=$?
tail -n 25 $O/pytest_wgrad.log | grep -E 'passed|failed|Error|assert' | head -8
timeout 900 python -m pytest tests/test_gpu_ppo.py tests/test_gpu_policy.py -q -x > $O/pytest.log 2>&1; echo pytest rc=$?
tail -n 2 $O/pytest.log
for rep in 1 2; do for D in 0 1; do
SG_NO_WGRAD=$D timeout 900 python3 bench.py --config ppo --no-cpu-baseline > $O/ppo_${D}_$rep.log 2>&1
python3 -c "
import json; l=json.loads(open('$O/ppo_${D}_$rep.log').read().strip().splitlines()[-1]); c=l['config']
print('no_wgrad=$D', round(l['value']/1e6,2), 'M/s update', round(c['update_ms_per_iter'],3))" 2>&1 | tail -n 1
done; done
