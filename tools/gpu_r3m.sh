#!/bin/bash
# Host step with copy-engine observation chunks (SG_HOST_CE_CHUNKS) vs zero-copy rows.
O=gpurun_out/r3m; mkdir -p $O
SG_HOST_CE_CHUNKS=4 timeout 900 python -m pytest tests -m gpu -q -x -k "host or cpp" > $O/pytest.log 2>&1; echo pytest rc=$?
tail -n 3 $O/pytest.log
for rep in 1 2; do for C in 0 2 4 8 16; do
SG_HOST_CE_CHUNKS=$C timeout 300 python3 bench.py --steps 2000 --warmup 5 --no-cpu-baseline > $O/e2e_${C}_$rep.log 2>&1
python3 -c "
import json; l=json.loads(open('$O/e2e_${C}_$rep.log').read().strip().splitlines()[-1]); e=l['e2e']
print('ce chunks $C', round(e['value']/1e6,1), 'M env-steps/s e2e', round(1e6*16384/e['value'],1), 'us/step')" 2>&1 | tail -n 1
done; done
