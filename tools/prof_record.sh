#!/bin/bash
# STAR path following: ncu --set full of one path_record_kernel launch (16,384 envs).
OUT=${1:-gpurun_out/prof_record}; mkdir -p $OUT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:path_record_kernel -s 2 -c 1 \
  -o $OUT/path_record python bench.py --config star --steps 1000 --fuse 250 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
ncu -i $OUT/path_record.ncu-rep --page details --csv > $OUT/path_record_details.csv 2>/dev/null
ncu -i $OUT/path_record.ncu-rep --page raw --csv > $OUT/path_record_raw.csv 2>/dev/null
ncu -i $OUT/path_record.ncu-rep --page source --print-source cuda,sass --csv > $OUT/path_record_src.csv 2>/dev/null
ls -la $OUT
