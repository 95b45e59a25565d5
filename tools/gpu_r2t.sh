#!/bin/bash
# Record kernel: unrolled walker; 4 blocks/SM (spills) vs unconstrained (3 blocks/SM).
O=gpurun_out/r2t; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x -k "star or path or record or fullsize or shard" > $O/pytest.log 2>&1; echo pytest rc=$?
tail -n 2 $O/pytest.log
for rep in 1 2; do for L in paper_2310_04676_b200/lib/libsg_env.so abtest/recminb1.so abtest/recquad.so; do
  t=$(basename $L .so)
  SG_LIB_PATH=$L timeout 300 python3 bench.py --config star --steps 3000 --fuse 250 --warmup 5 --no-cpu-baseline --e2e-steps 0 > $O/star_${t}_$rep.log 2>&1
  python3 -c "
import json; l=json.loads(open('$O/star_${t}_$rep.log').read().strip().splitlines()[-1])
print('$t', round(l['value']/1e9,3), 'G  us/launch', round(l['roofline']['avg_launch_us'],2))" 2>&1 | tail -n 1
done; done
timeout 600 ncu --clock-control none --set full --import-source on -k regex:path_record_kernel -s 2 -c 1 -o $O/path_record \
  python3 bench.py --config star --steps 500 --fuse 250 --warmup 5 --runs 1 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
ncu -i $O/path_record.ncu-rep --page details --csv 2>/dev/null | grep -E '"Duration"|Issue Slots Busy' | cut -c100-220
