OUT=gpurun_out/prof_b; mkdir -p $OUT
for G in 2 3; do
SG_TEAM_WARPS=$G timeout 300 ncu --set full --clock-control none --import-source on -k regex:env_step_kernel -s 4 -c 1 \
  -o $OUT/env_step_g$G python bench.py --steps 2000 --fuse 250 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
ncu -i $OUT/env_step_g$G.ncu-rep --page source --print-source sass --csv > $OUT/env_step_g${G}_sass.csv 2>/dev/null
ncu -i $OUT/env_step_g$G.ncu-rep --page raw --csv > $OUT/env_step_g${G}_raw.csv 2>/dev/null
done
ls -la $OUT
