#!/bin/bash
# Fused dgrad + ELU' backward: parity and PPO A/B (SG_NO_FUSED_BWD=1).
O=gpurun_out/r3j; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_policy.py tests/test_gpu_ppo.py -q -x > $O/pytest.log 2>&1; echo pytest rc=$?
tail -n 15 $O/pytest.log | grep -v '^$' | tail -n 8
for rep in 1 2; do for D in 0 1; do
SG_NO_FUSED_BWD=$D timeout 900 python3 bench.py --config ppo --no-cpu-baseline > $O/bench_ppo_${D}_$rep.log 2>&1
python3 -c "
import json; l=json.loads(open('$O/bench_ppo_${D}_$rep.log').read().strip().splitlines()[-1]); c=l['config']
print('no_fused_bwd=$D', round(l['value']/1e6,2), 'M/s rollout', round(c['rollout_ms_per_iter'],3), 'update', round(c['update_ms_per_iter'],3))" 2>&1 | tail -n 1
done; done
