#!/bin/bash
# the last two layers' backward as one launch: parity + A/B
O=gpurun_out/r5d; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_policy.py -q -x -k "dgrad or layer_backward or tail" > $O/pytest.log 2>&1; echo pytest rc=$?; tail -n 12 $O/pytest.log
timeout 600 python -m pytest tests/test_gpu_ppo.py tests/test_gpu_policy.py -q -x > $O/pytest_ppo.log 2>&1; echo pytest ppo rc=$?; tail -n 4 $O/pytest_ppo.log
for rep in 1 2; do for D in 0 1; do
if [ $D = 1 ]; then export SG_NO_FUSE_TAIL=1; else unset SG_NO_FUSE_TAIL; fi
timeout 900 python3 bench.py --config ppo --no-cpu-baseline > $O/ppo_${D}_$rep.log 2>&1
python3 -c "
import json; l=json.loads(open('$O/ppo_${D}_$rep.log').read().strip().splitlines()[-1]); c=l['config']
print('no_fuse_tail=$D', round(l['value']/1e6,2), 'M/s update', round(c['update_ms_per_iter'],3))" 2>&1 | tail -n 1
done; done
