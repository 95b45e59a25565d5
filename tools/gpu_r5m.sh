#!/bin/bash
# gather folded into the training forward and the loss: parity + A/B (SG_NO_GATHER_FUSE=1)
O=gpurun_out/r5m; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_policy.py tests/test_gpu_ppo.py -q -x > $O/pytest.log 2>&1; echo pytest rc=$?; tail -n 4 $O/pytest.log
for rep in 1 2; do for D in 0 1; do
if [ $D = 1 ]; then export SG_NO_GATHER_FUSE=1; else unset SG_NO_GATHER_FUSE; fi
timeout 900 python3 bench.py --config ppo --no-cpu-baseline > $O/ppo_${D}_$rep.log 2>&1
python3 -c "
import json; l=json.loads(open('$O/ppo_${D}_$rep.log').read().strip().splitlines()[-1]); c=l['config']
print('no_gather_fuse=$D', round(l['value']/1e6,2), 'M/s update', round(c['update_ms_per_iter'],3), 'rollout', round(c['rollout_ms_per_iter'],3))" 2>&1 | tail -n 1
done; done
unset SG_NO_GATHER_FUSE
timeout 300 python3 tools/prof_ppo.py bf16 2>&1 | grep -E 'policy_|gather|loss|Self CUDA time'
