#!/bin/bash
# mt_step_kernel source-level ncu capture (per-line instruction / stall counts)
OUT=${1:-gpurun_out/prof_multi_src}; mkdir -p $OUT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mt_step_kernel -s 4 -c 1 \
  -o $OUT/mt_step python bench.py --config multitool --steps 1000 --fuse 250 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
ncu -i $OUT/mt_step.ncu-rep --page source --print-source cuda,sass --csv > $OUT/mt_step_src.csv 2>/dev/null
ncu -i $OUT/mt_step.ncu-rep --page raw --csv > $OUT/mt_step_raw.csv 2>/dev/null
rm -f $OUT/mt_step.ncu-rep
