#!/bin/bash
# A/B: TMA-epilogue fused data gradient (SG_FUSED_BWD=1) vs library GEMM + ELU pass
O=gpurun_out/r5a; mkdir -p $O
timeout 300 python3 tools/dgrad_probe.py 2>&1 | tail -n 4
timeout 600 python -m pytest tests/test_gpu_policy.py -q -x -k "dgrad" > $O/pytest.log 2>&1; echo pytest rc=$?; tail -n 3 $O/pytest.log
timeout 600 python -m pytest tests/test_gpu_ppo.py -q -x > $O/pytest_ppo.log 2>&1; echo pytest ppo rc=$?; tail -n 2 $O/pytest_ppo.log
for rep in 1 2; do for D in 0 1; do
if [ $D = 1 ]; then export SG_FUSED_BWD=1; else unset SG_FUSED_BWD; fi
timeout 900 python3 bench.py --config ppo --no-cpu-baseline > $O/ppo_${D}_$rep.log 2>&1
python3 -c "
import json; l=json.loads(open('$O/ppo_${D}_$rep.log').read().strip().splitlines()[-1]); c=l['config']
print('fused_bwd=$D', round(l['value']/1e6,2), 'M/s update', round(c['update_ms_per_iter'],3))" 2>&1 | tail -n 1
done; done
unset SG_FUSED_BWD
timeout 300 python3 tools/dgrad_probe.py 2>&1 | tail -n 4
