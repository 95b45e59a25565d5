#!/bin/bash
# Rollout env steps launched behind the policy act (PDL) vs plain launches: parity + A/B of the policy / ppo lines.
O=gpurun_out/r6h; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_ppo.py -q -x > $O/pytest_ppo.log 2>&1; echo pytest rc=$?; tail -2 $O/pytest_ppo.log
for rep in 1; do for v in 0 1; do
  SG_NO_ENV_PDL=$v timeout 600 python3 bench.py --config policy --no-cpu-baseline --e2e-steps 0 > $O/policy_$v.log 2>&1
  python3 -c "import json; l=json.loads(open('$O/policy_$v.log').read().strip().splitlines()[-1]); print('policy no_env_pdl=$v', round(l['value']/1e6,1), 'M')"
done; done
for v in 0 1; do
  SG_NO_ENV_PDL=$v timeout 900 python3 bench.py --config ppo --no-cpu-baseline > $O/ppo_$v.log 2>&1
  python3 -c "import json; l=json.loads(open('$O/ppo_$v.log').read().strip().splitlines()[-1]); print('ppo no_env_pdl=$v', round(l['value']/1e6,2), 'M', 'rollout_ms', round(l['config']['rollout_ms_per_iter'],3), 'e2e', round(l['e2e']['value']/1e6,2))"
done
