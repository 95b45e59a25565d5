#!/bin/bash
# pipelined backward head (layer 1 + dW_0) vs the one-tile kernel (SG_BWD_HEAD_ONETILE=1)
O=gpurun_out/r5k; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_policy.py -q -x -k "layer_backward or tail" > $O/pytest.log 2>&1; echo pytest rc=$?; tail -n 3 $O/pytest.log
timeout 600 python -m pytest tests/test_gpu_ppo.py -q -x > $O/pytest_ppo.log 2>&1; echo pytest ppo rc=$?; tail -n 2 $O/pytest_ppo.log
for rep in 1 2; do for D in 0 1; do
if [ $D = 1 ]; then export SG_BWD_HEAD_ONETILE=1; else unset SG_BWD_HEAD_ONETILE; fi
timeout 900 python3 bench.py --config ppo --no-cpu-baseline > $O/ppo_${D}_$rep.log 2>&1
python3 -c "
import json; l=json.loads(open('$O/ppo_${D}_$rep.log').read().strip().splitlines()[-1]); c=l['config']
print('onetile=$D', round(l['value']/1e6,2), 'M/s update', round(c['update_ms_per_iter'],3))" 2>&1 | tail -n 1
done; done
unset SG_BWD_HEAD_ONETILE
timeout 300 python3 tools/prof_ppo.py bf16 2>&1 | grep -E 'bwd_|dgrad'
