#!/bin/bash
# training forward: 32-byte activation stores vs 16-byte (SG_STORE_V4 variant)
O=gpurun_out/r5f; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_policy.py -q -x -k "train_forward" > $O/pytest.log 2>&1; echo pytest rc=$?; tail -n 2 $O/pytest.log
for rep in 1 2; do for V in main v4; do
if [ $V = v4 ]; then export SG_LIB_PATH=$PWD/abtest/v4.so; else unset SG_LIB_PATH; fi
timeout 900 python3 bench.py --config ppo --no-cpu-baseline > $O/ppo_${V}_$rep.log 2>&1
python3 -c "
import json; l=json.loads(open('$O/ppo_${V}_$rep.log').read().strip().splitlines()[-1]); c=l['config']
print('$V', round(l['value']/1e6,2), 'M/s update', round(c['update_ms_per_iter'],3))" 2>&1 | tail -n 1
done; done
unset SG_LIB_PATH
timeout 300 python3 tools/prof_ppo.py bf16 2>&1 | grep -E 'train_fwd'
