#!/bin/bash
# ImageMatching (PSM, 16,384 envs): ncu --set full of one fused im_step_kernel launch.
OUT=${1:-gpurun_out/prof_image}; mkdir -p $OUT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:im_step_kernel -s 4 -c 1 \
  -o $OUT/im_step python bench.py --config image --steps 500 --fuse 250 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
ncu -i $OUT/im_step.ncu-rep --page details --csv > $OUT/im_step_details.csv 2>/dev/null
ncu -i $OUT/im_step.ncu-rep --page raw --csv > $OUT/im_step_raw.csv 2>/dev/null
ncu -i $OUT/im_step.ncu-rep --page source --print-source cuda,sass --csv > $OUT/im_step_src.csv 2>/dev/null
ls -la $OUT
