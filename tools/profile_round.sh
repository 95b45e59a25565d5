#!/bin/bash
# Profiling pass for profiles/ (run under gpurun on ONE GPU; never a multi-rank command).
#   1. ncu launch list (gpu__time_duration per launch) of a short headline bench run
#   2. one `ncu --set full` capture of the dominant kernel (env_step_kernel, fused bench variant)
#   3. one `ncu --set full` capture of the tcgen05 policy forward kernel
# Outputs land in gpurun_out/ (scratch); summaries are copied into profiles/ by hand.
set -x
OUT=${1:-gpurun_out}
mkdir -p $OUT
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  python bench.py --steps 2000 --fuse 250 --e2e-steps 0 --no-cpu-baseline > $OUT/launches_bench.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:env_step_kernel -s 4 -c 1 \
  -o $OUT/env_step python bench.py --steps 2000 --fuse 250 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:policy_fwd_kernel -s 3 -c 1 \
  -o $OUT/policy_fwd python -c "
import torch, sys; sys.path.insert(0, '.')
from paper_2310_04676_b200 import sg
env = sg.VecTaskEnv(robots=('psm',), n_envs=16384); obs = env.reset()
pol = sg.Policy(27, 7); pol.load_params(torch.from_numpy(pol.init_params(0)).cuda())
for _ in range(6): pol.forward(obs)
torch.cuda.synchronize()" > /dev/null 2>&1
for f in env_step policy_fwd; do
  ncu -i $OUT/$f.ncu-rep --page details --csv > $OUT/${f}_details.csv 2>/dev/null
  ncu -i $OUT/$f.ncu-rep --page raw --csv > $OUT/${f}_raw.csv 2>/dev/null
done
ls -la $OUT
