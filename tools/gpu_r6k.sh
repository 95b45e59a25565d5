#!/bin/bash
# A/B: exp(log-std) of the sampled actions computed with the draws (during layer 2) instead of in the act tail.
O=gpurun_out/r6k; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_ppo.py tests/test_gpu_policy.py -q -x > $O/pytest.log 2>&1; echo pytest rc=$?; tail -2 $O/pytest.log
for rep in 1 2; do for lib in abtest/old.so abtest/new.so; do
  SG_LIB_PATH=$lib timeout 600 python3 bench.py --config policy --no-cpu-baseline --e2e-steps 0 > $O/p.log 2>&1
  python3 -c "import json; l=json.loads(open('$O/p.log').read().strip().splitlines()[-1]); print('$lib', round(l['value']/1e6,1), 'M', 'fwd_us', round(l['roofline']['avg_launch_us'],2))"
done; done
