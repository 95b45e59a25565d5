#!/bin/bash
# Producer-stored observation rows (default) vs scorer-stored (SG_SCORER_ROWS): parity + A/B.
O=gpurun_out/r2p; mkdir -p $O
DEF=paper_2310_04676_b200/lib/libsg_env.so
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -n 3 $O/pytest_gpu.log
ab() {  # lib cfg steps fuse tag
  SG_LIB_PATH=$1 timeout 300 python3 bench.py --config $2 --steps $3 --fuse $4 --warmup 5 --no-cpu-baseline --e2e-steps 0 > $O/$5.log 2>&1
  python3 -c "
import json; l=json.loads(open('$O/$5.log').read().strip().splitlines()[-1]); r=l['runs']
print('$5', round(l['value']/1e9,3), 'G  us/launch', round(l['roofline']['avg_launch_us'],2), 'std', round(r['value_std']/1e9,3))" 2>&1 | tail -n 1
}
for rep in 1 2; do
  for L in $DEF abtest/scorerrows.so; do
    t=$(basename $L .so)
    ab $L psm 20 20 psm_k20_${t}_$rep
    ab $L psm 2500 250 psm_k250_${t}_$rep
    ab $L ecm 2500 250 ecm_k250_${t}_$rep
    ab $L star 3000 250 star_k250_${t}_$rep
  done
done
