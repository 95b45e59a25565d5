#!/bin/bash
O=gpurun_out/r3o; mkdir -p $O
for tool in synccheck racecheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 3 python tools/sanitize_r2.py > $O/$tool.log 2>&1; echo $tool rc=$?
  grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $O/$tool.log | head -3
done
timeout 1200 compute-sanitizer --tool synccheck --error-exitcode 3 python tools/sanitize_probe.py > $O/synccheck_r1probe.log 2>&1; echo synccheck r1 probe rc=$?
grep -E 'ERROR SUMMARY' $O/synccheck_r1probe.log | head -3; grep 'at ' $O/synccheck_r1probe.log | sort | uniq -c | head -5
for rep in 1 2; do
  timeout 300 python3 bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 0 > $O/k20_$rep.log 2>&1
  timeout 300 python3 bench.py --steps 2500 --warmup 5 --no-cpu-baseline --e2e-steps 0 > $O/k250_$rep.log 2>&1
  timeout 300 python3 bench.py --config star --steps 2500 --warmup 5 --no-cpu-baseline --e2e-steps 0 > $O/star_$rep.log 2>&1
  for f in k20 k250 star; do python3 -c "
import json; l=json.loads(open('$O/${f}_$rep.log').read().strip().splitlines()[-1])
print('$f', round(l['value']/1e9,3), 'G us/launch', round(l['roofline']['avg_launch_us'],2))"; done
done
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo pytest rc=$?; tail -n 2 $O/pytest.log
