#!/bin/bash
# A/B timing of builds of libsg_env.so on the same box:
#   tools/ab.sh "a.so b.so" "psm ecm star" "2 4"
LIBS=${1:?libs}; CFGS=${2:-psm}; GS=${3:-2}
for cfg in $CFGS; do for g in $GS; do for rep in 1 2; do for lib in $LIBS; do
  SG_LIB_PATH=$lib SG_TEAM_WARPS=$g timeout 300 python bench.py --config $cfg --e2e-steps 0 --no-cpu-baseline 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', '$lib', 'G=$g', round(d['value']/1e9, 3))"
done; done; done; done
