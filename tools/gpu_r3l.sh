#!/bin/bash
O=gpurun_out/r3l; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_policy.py -q -x -k "dgrad or fused" > $O/pytest.log 2>&1; echo pytest rc=$?
tail -n 2 $O/pytest.log
for rep in 1 2; do for V in def nob dg3; do
  case $V in def) L=paper_2310_04676_b200/lib/libsg_env.so; D=0;; nob) L=paper_2310_04676_b200/lib/libsg_env.so; D=1;; dg3) L=abtest/dgrad3.so; D=0;; esac
  SG_LIB_PATH=$L SG_NO_FUSED_BWD=$D timeout 900 python3 bench.py --config ppo --no-cpu-baseline > $O/ppo_${V}_$rep.log 2>&1
  python3 -c "
import json; l=json.loads(open('$O/ppo_${V}_$rep.log').read().strip().splitlines()[-1]); c=l['config']
print('$V', round(l['value']/1e6,2), 'M/s update', round(c['update_ms_per_iter'],3))" 2>&1 | tail -n 1
done; done
