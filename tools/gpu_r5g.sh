#!/bin/bash
# vectorised unpadded gather: parity + PPO bench
O=gpurun_out/r5g; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_ppo.py -q -x > $O/pytest.log 2>&1; echo pytest rc=$?; tail -n 2 $O/pytest.log
for rep in 1 2; do
timeout 900 python3 bench.py --config ppo --no-cpu-baseline > $O/ppo_$rep.log 2>&1
python3 -c "
import json; l=json.loads(open('$O/ppo_$rep.log').read().strip().splitlines()[-1]); c=l['config']
print('ppo', round(l['value']/1e6,2), 'M/s update', round(c['update_ms_per_iter'],3))" 2>&1 | tail -n 1
done
timeout 300 python3 tools/prof_ppo.py bf16 2>&1 | grep -E 'policy_|gather|Radix|loss|adam|Self CUDA time'
