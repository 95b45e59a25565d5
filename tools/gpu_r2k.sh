#!/bin/bash
# A/B: sub-partition role spread (SG_ROLE_SPREAD) vs default; policy / ppo lines.
O=gpurun_out/r2k; mkdir -p $O
DEF=paper_2310_04676_b200/lib/libsg_env.so
ab() {  # lib cfg steps fuse tag
  SG_LIB_PATH=$1 timeout 300 python3 bench.py --config $2 --steps $3 --fuse $4 --warmup 5 --no-cpu-baseline --e2e-steps 0 > $O/$5.log 2>&1
  python3 -c "
import json; l=json.loads(open('$O/$5.log').read().strip().splitlines()[-1]); r=l['runs']
print('$5', round(l['value']/1e9,3), 'G  us/launch', round(l['roofline']['avg_launch_us'],2), 'std', round(r['value_std']/1e9,3))" 2>&1 | tail -1
}
for rep in 1 2; do
  for L in $DEF abtest/spread.so; do
    t=$(basename $L .so)
    ab $L psm 20 20 psm_k20_${t}_$rep
    ab $L psm 2500 250 psm_k250_${t}_$rep
    ab $L ecm 2500 250 ecm_k250_${t}_$rep
    ab $L star 3000 250 star_k250_${t}_$rep
  done
done
SG_LIB_PATH=abtest/spread.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x > $O/pytest_spread.log 2>&1; echo spread pytest rc=$?
timeout 600 python3 bench.py --config policy --steps 640 > $O/bench_policy.log 2>&1; echo policy rc=$?
timeout 900 python3 bench.py --config ppo --no-cpu-baseline > $O/bench_ppo.log 2>&1; echo ppo rc=$?
tail -3 $O/pytest_spread.log; tail -1 $O/bench_policy.log | cut -c1-2500; echo; tail -1 $O/bench_ppo.log | cut -c1-1500
