#!/bin/bash
# programmatic dependent launch of the policy act after the env step (A/B: SG_NO_PDL=1)
O=gpurun_out/r5o; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_policy.py tests/test_gpu_ppo.py -q -x > $O/pytest.log 2>&1; echo pytest rc=$?; tail -n 3 $O/pytest.log
for rep in 1 2; do for D in 0 1; do
if [ $D = 1 ]; then export SG_NO_PDL=1; else unset SG_NO_PDL; fi
timeout 900 python3 bench.py --config policy --no-cpu-baseline > $O/pol_${D}_$rep.log 2>&1
python3 -c "
import json; l=json.loads(open('$O/pol_${D}_$rep.log').read().strip().splitlines()[-1])
print('no_pdl=$D policy', round(l['value']/1e6,1), 'M/s', 'e2e', l.get('e2e',{}).get('value'))" 2>&1 | tail -n 1
timeout 900 python3 bench.py --config ppo --no-cpu-baseline > $O/ppo_${D}_$rep.log 2>&1
python3 -c "
import json; l=json.loads(open('$O/ppo_${D}_$rep.log').read().strip().splitlines()[-1]); c=l['config']
print('no_pdl=$D ppo', round(l['value']/1e6,2), 'M/s update', round(c['update_ms_per_iter'],3), 'rollout', round(c['rollout_ms_per_iter'],3))" 2>&1 | tail -n 1
done; done
