#!/bin/bash
# Packed team layout: parity under both layouts, A/B throughput, one ncu capture.
mkdir -p gpurun_out/r2b
O=gpurun_out/r2b
SG_TEAM_LAYOUT=packed timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_packed.log 2>&1; echo packed pytest rc=$?
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_auto.log 2>&1; echo auto pytest rc=$?
for L in legacy packed; do
  for cfg in psm star; do
    SG_TEAM_LAYOUT=$L timeout 300 python3 bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 0 > $O/k20_${cfg}_$L.log 2>&1
    SG_TEAM_LAYOUT=$L timeout 300 python3 bench.py --config $cfg --steps 20000 --no-cpu-baseline --e2e-steps 0 > $O/k250_${cfg}_$L.log 2>&1
  done
done
timeout 300 python3 bench.py --gpus 1 --steps 20 --warmup 5 > $O/driver_cmd.log 2>&1
timeout 600 ncu --clock-control none --set full --import-source on -k regex:env_step_kernel -s 6 -c 1 -o $O/env_step_psm_packed_k250 \
    python3 bench.py --steps 250 --fuse 250 --warmup 5 --runs 1 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
ncu -i $O/env_step_psm_packed_k250.ncu-rep --page raw --csv > $O/env_step_psm_packed_k250_raw.csv 2>/dev/null
ncu -i $O/env_step_psm_packed_k250.ncu-rep --page details --csv > $O/env_step_psm_packed_k250_details.csv 2>/dev/null
rm -f $O/*.ncu-rep
for f in $O/k*.log $O/driver_cmd.log; do echo "$f $(python3 -c "
import json,sys
l=json.loads(open('$f').read().strip().splitlines()[-1]); r=l['roofline']
print(round(l['value']/1e9,2),'G', 'ms/step', l['ms_per_step'], 'avg_launch_us', round(r['avg_launch_us'],2), 'frac', round(r['frac'],3), 'runs', l['runs'].get('ms_per_run'), l['runs'].get('attempts'))
" 2>&1 | tail -1)"; done
tail -n 3 $O/pytest_*.log
