#!/bin/bash
# ELU exp2 split between MUFU and an FMA-pipe polynomial: every 4th pair (default), 3rd, 8th, none.
O=gpurun_out/r3i; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_policy.py tests/test_gpu_ppo.py -q -x > $O/pytest.log 2>&1; echo pytest rc=$?
tail -n 2 $O/pytest.log
for rep in 1 2; do for L in paper_2310_04676_b200/lib/libsg_env.so abtest/poly0.so abtest/poly3.so abtest/poly8.so; do
  t=$(basename $L .so)
  echo "$t $(SG_LIB_PATH=$L timeout 300 python tools/policy_probe.py 2>&1 | grep -E 'cuda graph' | tr '\n' ' ')"
done; done
for L in paper_2310_04676_b200/lib/libsg_env.so abtest/poly0.so; do
  t=$(basename $L .so)
  SG_LIB_PATH=$L timeout 600 python3 bench.py --config policy --no-cpu-baseline --e2e-steps 0 > $O/policy_$t.log 2>&1
  python3 -c "
import json; l=json.loads(open('$O/policy_$t.log').read().strip().splitlines()[-1])
print('$t policy', round(l['value']/1e6,1), 'M/s  fwd us', round(l['roofline']['avg_launch_us'],2))" 2>&1 | tail -n 1
done
