#!/bin/bash
# MultiToolReaching (trimanual, 16,384 envs): bench line + ncu --set full of one
# fused mt_step_kernel launch + launch list. Run under gpurun (one GPU).
OUT=${1:-gpurun_out/prof_multi}; mkdir -p $OUT
timeout 600 python bench.py --config multitool --cpu-budget 10 > $OUT/bench_multitool.log 2>&1
timeout 600 ncu --clock-control none --metrics gpu__time_duration.sum --csv --log-file $OUT/launches_multitool.csv \
  python bench.py --config multitool --steps 2000 --fuse 250 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mt_step_kernel -s 4 -c 1 \
  -o $OUT/mt_step python bench.py --config multitool --steps 2000 --fuse 250 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
ncu -i $OUT/mt_step.ncu-rep --page details --csv > $OUT/mt_step_details.csv 2>/dev/null
ncu -i $OUT/mt_step.ncu-rep --page raw --csv > $OUT/mt_step_raw.csv 2>/dev/null
ncu -i $OUT/mt_step.ncu-rep --page source --print-source sass --csv > $OUT/mt_step_sass.csv 2>/dev/null
rm -f $OUT/mt_step.ncu-rep.bak
ls -la $OUT; tail -c 1500 $OUT/bench_multitool.log
