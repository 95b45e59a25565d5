#!/bin/bash
# Policy forward: sampling behind layer 2; trunk stagger A/B; phase probes.
O=gpurun_out/r2m; mkdir -p $O
DEF=paper_2310_04676_b200/lib/libsg_env.so
timeout 600 python -m pytest tests/test_gpu_policy.py tests/test_gpu_ppo.py -q -x > $O/pytest_policy.log 2>&1; echo pytest rc=$?
SG_LIB_PATH=abtest/pstagger.so timeout 600 python -m pytest tests/test_gpu_policy.py tests/test_gpu_ppo.py -q -x > $O/pytest_stagger.log 2>&1; echo pytest stagger rc=$?
for rep in 1 2; do for L in $DEF abtest/pstagger.so; do
  t=$(basename $L .so)
  SG_LIB_PATH=$L timeout 300 python3 bench.py --config policy --steps 640 --no-cpu-baseline --e2e-steps 0 > $O/policy_${t}_$rep.log 2>&1
  python3 -c "
import json; l=json.loads(open('$O/policy_${t}_$rep.log').read().strip().splitlines()[-1])
print('$t', round(l['value']/1e6,1), 'M/s  fwd us', round(l['roofline']['avg_launch_us'],2))" 2>&1 | tail -1
done; done
for L in pprobe pprobe_stagger; do
  SG_LIB_PATH=abtest/$L.so timeout 300 python3 bench.py --config policy --steps 64 --runs 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>&1 | grep pprobe | tail -8 > $O/$L.txt
  echo $L; cat $O/$L.txt
done
tail -2 $O/pytest_*.log
