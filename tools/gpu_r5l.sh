#!/bin/bash
# next update's permutations drawn on a side stream (A/B: SG_NO_PERM_PREFETCH=1)
O=gpurun_out/r5l; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_ppo.py -q -x > $O/pytest_ppo.log 2>&1; echo pytest ppo rc=$?; tail -n 2 $O/pytest_ppo.log
for rep in 1 2; do for D in 0 1; do
if [ $D = 1 ]; then export SG_NO_PERM_PREFETCH=1; else unset SG_NO_PERM_PREFETCH; fi
timeout 900 python3 bench.py --config ppo --no-cpu-baseline > $O/ppo_${D}_$rep.log 2>&1
python3 -c "
import json; l=json.loads(open('$O/ppo_${D}_$rep.log').read().strip().splitlines()[-1]); c=l['config']
print('no_prefetch=$D', round(l['value']/1e6,2), 'M/s update', round(c['update_ms_per_iter'],3), 'rollout', round(c['rollout_ms_per_iter'],3))" 2>&1 | tail -n 1
done; done
