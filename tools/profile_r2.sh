#!/bin/bash
# Round-2 profiling of the DRIVER's headline command (run under gpurun on ONE GPU):
#   python3 bench.py --gpus 1 --steps 20 --warmup 5
# 1. ncu launch list of that exact command (cold-cache, serialised per-launch times)
# 2. one `ncu --set full` capture of the first TIMED env_step launch of it
#    (K = 20 fused steps: launches 1-5 are the warm-up single steps, 6 the untimed
#    K = 20 launch, 7 the first timed one)
# 3. the same capture at K = 250 (the default bench's fused launch)
# Then tools/traffic_r2.py writes profiles/r2/traffic_<config>_k<K>.json (DRAM +
# L2 bytes per launch, issue-slot use) that bench.py attaches to its roofline.
# Usage: tools/profile_r2.sh [config] [outdir]
CFG=${1:-psm}
OUT=${2:-gpurun_out/prof_r2}
mkdir -p $OUT
NCU="ncu --clock-control none"
timeout 600 $NCU --metrics gpu__time_duration.sum --csv --log-file $OUT/launches_${CFG}_k20.csv \
  python3 bench.py --config $CFG --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > $OUT/launches_${CFG}_k20.log 2>&1
for K in 20 250; do
  STEPS=$K
  timeout 600 $NCU --set full --import-source on -k regex:env_step_kernel -s 6 -c 1 -o $OUT/env_step_${CFG}_k$K \
    python3 bench.py --config $CFG --steps $STEPS --fuse $K --warmup 5 --runs 1 --e2e-steps 0 --no-cpu-baseline \
    > $OUT/env_step_${CFG}_k$K.log 2>&1
  if [ -f $OUT/env_step_${CFG}_k$K.ncu-rep ]; then
    ncu -i $OUT/env_step_${CFG}_k$K.ncu-rep --page details --csv > $OUT/env_step_${CFG}_k${K}_details.csv 2>/dev/null
    ncu -i $OUT/env_step_${CFG}_k$K.ncu-rep --page raw --csv > $OUT/env_step_${CFG}_k${K}_raw.csv 2>/dev/null
  fi
done
ls -la $OUT
