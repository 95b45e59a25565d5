#!/bin/bash
# Packed layout with full 32-env teams (SG_PACKED32) vs legacy vs packed quads.
O=gpurun_out/r3h; mkdir -p $O
SG_LIB_PATH=abtest/packed32.so SG_TEAM_LAYOUT=packed timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > $O/pytest.log 2>&1; echo pytest rc=$?
tail -n 2 $O/pytest.log
DEF=paper_2310_04676_b200/lib/libsg_env.so
ab() {  # lib layout cfg steps fuse tag
  SG_LIB_PATH=$1 SG_TEAM_LAYOUT=$2 timeout 300 python3 bench.py --config $3 --steps $4 --fuse $5 --warmup 5 --no-cpu-baseline --e2e-steps 0 > $O/$6.log 2>&1
  python3 -c "
import json; l=json.loads(open('$O/$6.log').read().strip().splitlines()[-1])
print('$6', round(l['value']/1e9,3), 'G  us/launch', round(l['roofline']['avg_launch_us'],2))" 2>&1 | tail -n 1
}
for rep in 1 2; do
  ab $DEF legacy psm 20 20 k20_legacy_$rep
  ab abtest/packed32.so packed psm 20 20 k20_packed32_$rep
  ab $DEF packed psm 20 20 k20_packedq_$rep
  ab $DEF legacy psm 2500 250 k250_legacy_$rep
  ab abtest/packed32.so packed psm 2500 250 k250_packed32_$rep
  ab $DEF legacy star 2500 250 star_legacy_$rep
  ab abtest/packed32.so packed star 2500 250 star_packed32_$rep
done
