#!/bin/bash
O=gpurun_out/r2v; mkdir -p $O
for rep in 1 2; do for D in 0 1; do
SG_NO_DIRECT_GRAD=$D timeout 900 python3 bench.py --config ppo --no-cpu-baseline > $O/bench_ppo_${D}_$rep.log 2>&1
python3 -c "
import json; l=json.loads(open('$O/bench_ppo_${D}_$rep.log').read().strip().splitlines()[-1]); c=l['config']
print('no_direct=$D', round(l['value']/1e6,2), 'M/s rollout', round(c['rollout_ms_per_iter'],3), 'update', round(c['update_ms_per_iter'],3))"
done; done
