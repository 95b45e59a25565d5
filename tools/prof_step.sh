#!/bin/bash
# ncu --set full capture of one fused env_step launch (PSM, 16,384 envs) + exports
# usage (under gpurun): bash tools/prof_step.sh OUT_DIR [config] [G]
OUT=${1:-gpurun_out/prof}; CFG=${2:-psm}; G=${3:-2}; mkdir -p $OUT
SG_TEAM_WARPS=$G timeout 300 ncu --set full --clock-control none --import-source on -k regex:env_step_kernel -s 4 -c 1 \
  -o $OUT/env_step_$CFG python bench.py --config $CFG --steps 2000 --fuse 250 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
ncu -i $OUT/env_step_$CFG.ncu-rep --page source --print-source cuda,sass --csv > $OUT/env_step_${CFG}_src.csv 2>/dev/null
ncu -i $OUT/env_step_$CFG.ncu-rep --page source --print-source sass --csv > $OUT/env_step_${CFG}_sass.csv 2>/dev/null
ncu -i $OUT/env_step_$CFG.ncu-rep --page raw --csv > $OUT/env_step_${CFG}_raw.csv 2>/dev/null
ncu -i $OUT/env_step_$CFG.ncu-rep --page details --csv > $OUT/env_step_${CFG}_details.csv 2>/dev/null
