#!/bin/bash
O=gpurun_out/r3q; mkdir -p $O
for probe in sanitize_r2 sanitize_probe; do
  timeout 1200 compute-sanitizer --tool synccheck --error-exitcode 3 python tools/$probe.py > $O/sync_$probe.log 2>&1; echo synccheck $probe rc=$?
  grep -E 'ERROR SUMMARY' $O/sync_$probe.log | head -2; grep ' at ' $O/sync_$probe.log | sort | uniq -c | head -3
done
for rep in 1 2; do for L in paper_2310_04676_b200/lib/libsg_env.so abtest/redbar.so; do t=$(basename $L .so)
  SG_LIB_PATH=$L timeout 300 python3 bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 0 > $O/k20_${t}_$rep.log 2>&1
  SG_LIB_PATH=$L timeout 300 python3 bench.py --steps 2500 --warmup 5 --no-cpu-baseline --e2e-steps 0 > $O/k250_${t}_$rep.log 2>&1
  SG_LIB_PATH=$L timeout 300 python3 bench.py --config ecm --steps 2500 --warmup 5 --no-cpu-baseline --e2e-steps 0 > $O/ecm_${t}_$rep.log 2>&1
  SG_LIB_PATH=$L timeout 300 python3 bench.py --config star --steps 2500 --warmup 5 --no-cpu-baseline --e2e-steps 0 > $O/star_${t}_$rep.log 2>&1
  for f in k20 k250 ecm star; do python3 -c "
import json; l=json.loads(open('$O/${f}_${t}_$rep.log').read().strip().splitlines()[-1])
print('$f $t', round(l['value']/1e9,3), 'G us/launch', round(l['roofline']['avg_launch_us'],2))"; done
done; done
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo pytest rc=$?; tail -n 2 $O/pytest.log
