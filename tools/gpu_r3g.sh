#!/bin/bash
O=gpurun_out/r3g; mkdir -p $O
for S in 640 3200 6400 32000; do
timeout 900 python3 bench.py --config policy --steps $S --no-cpu-baseline --e2e-steps 0 > $O/policy_$S.log 2>&1
python3 -c "
import json; l=json.loads(open('$O/policy_$S.log').read().strip().splitlines()[-1]); r=l['runs']
print('steps $S', round(l['value']/1e6,1), 'M/s', 'gate', r['gate_held'], 'std', round(r['value_std']/1e6,1))" 2>&1 | tail -n 1
done
