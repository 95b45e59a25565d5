#!/bin/bash
# A/B timing of two builds of libsg_env.so on the same box: tools/ab.sh a.so b.so [G...]
A=$1; B=$2; shift 2
for g in ${@:-2}; do for lib in $A $B $A $B; do
  SG_LIB_PATH=$lib SG_TEAM_WARPS=$g timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', 'G=$g', round(d['value']/1e9, 3))"
done; done
