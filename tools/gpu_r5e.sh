#!/bin/bash
# backward kernels with vectorised column sums: parity + PPO bench + probe
O=gpurun_out/r5e; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_policy.py -q -x -k "dgrad or layer_backward or tail" > $O/pytest.log 2>&1; echo pytest rc=$?; tail -n 12 $O/pytest.log
timeout 600 python -m pytest tests/test_gpu_ppo.py tests/test_gpu_policy.py -q -x > $O/pytest_ppo.log 2>&1; echo pytest ppo rc=$?; tail -n 4 $O/pytest_ppo.log
timeout 300 python3 tools/dgrad_probe.py 2>&1 | tail -n 4
for rep in 1 2; do
timeout 900 python3 bench.py --config ppo --no-cpu-baseline > $O/ppo_$rep.log 2>&1
python3 -c "
import json; l=json.loads(open('$O/ppo_$rep.log').read().strip().splitlines()[-1]); c=l['config']
print('ppo', round(l['value']/1e6,2), 'M/s update', round(c['update_ms_per_iter'],3))" 2>&1 | tail -n 1
done
timeout 300 python3 tools/prof_ppo.py bf16 2>&1 | grep -E 'policy_|gather|Radix|loss|elu_bwd|adam|Self CUDA time'
