#!/bin/bash
O=gpurun_out/r2z; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_policy.py -q -x -k "train or fused" > $O/pytest.log 2>&1; echo pytest rc=$?
tail -n 2 $O/pytest.log
for rep in 1 2; do for L in paper_2310_04676_b200/lib/libsg_env.so abtest/trainstag.so; do
t=$(basename $L .so)
SG_LIB_PATH=$L timeout 900 python3 bench.py --config ppo --no-cpu-baseline > $O/bench_ppo_${t}_$rep.log 2>&1
python3 -c "
import json; l=json.loads(open('$O/bench_ppo_${t}_$rep.log').read().strip().splitlines()[-1]); c=l['config']
print('$t', round(l['value']/1e6,2), 'M/s rollout', round(c['rollout_ms_per_iter'],3), 'update', round(c['update_ms_per_iter'],3))" 2>&1 | tail -n 1
done; done
