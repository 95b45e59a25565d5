#!/bin/bash
# Host step rolling PCIe read window: parity with the window on, e2e A/B over window sizes.
O=gpurun_out/r3a; mkdir -p $O
SG_HOST_READ_WINDOW=128 timeout 900 python -m pytest tests -m gpu -q -x -k "host or cpp" > $O/pytest.log 2>&1; echo pytest rc=$?
tail -n 2 $O/pytest.log
for rep in 1 2; do for W in 0 64 128 256 384; do
SG_HOST_READ_WINDOW=$W timeout 300 python3 bench.py --steps 2000 --warmup 5 --no-cpu-baseline > $O/e2e_${W}_$rep.log 2>&1
python3 -c "
import json; l=json.loads(open('$O/e2e_${W}_$rep.log').read().strip().splitlines()[-1]); e=l['e2e']
print('window $W', round(e['value']/1e6,1), 'M env-steps/s e2e', round(1e6*16384/e['value'],1), 'us/step')" 2>&1 | tail -n 1
done; done
