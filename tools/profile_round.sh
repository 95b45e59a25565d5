#!/bin/bash
# Profiling pass for profiles/ (run under gpurun on ONE GPU; never a multi-rank command).
#   1. ncu launch list (gpu__time_duration per launch, cold-cache serialised) of a
#      short headline bench run (PSM reach, 16,384 envs, fused 250-step launches)
#   2. one `ncu --set full` capture of the dominant kernel (fused env_step) per
#      BASELINE config (PSM, ECM, STAR)
#   3. one `ncu --set full` capture of the tcgen05 policy forward kernel
#   4. launch list of two PPO iterations (config 5)
# Outputs land in $OUT (scratch, gpurun_out/); tools/summarize_profiles.py turns
# them into the committed profiles/<round>/ summaries.
OUT=${1:-gpurun_out/prof_round}
mkdir -p $OUT
NCU="ncu --clock-control none"
timeout 600 $NCU --metrics gpu__time_duration.sum --csv --log-file $OUT/launches_psm.csv \
  python bench.py --steps 2000 --fuse 250 --e2e-steps 0 --no-cpu-baseline > $OUT/launches_psm.log 2>&1
for cfg in psm ecm star; do
  timeout 600 $NCU --set full --import-source on -k regex:env_step_kernel -s 4 -c 1 -o $OUT/env_step_$cfg \
    python bench.py --config $cfg --steps 2000 --fuse 250 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
done
timeout 600 $NCU --set full --import-source on -k regex:policy_fwd_kernel -s 3 -c 1 -o $OUT/policy_fwd python -c "
import torch, sys; sys.path.insert(0, '.')
from paper_2310_04676_b200 import sg
env = sg.VecTaskEnv(robots=('psm',), n_envs=16384); obs = env.reset()
pol = sg.Policy(27, 7); pol.load_params(torch.from_numpy(pol.init_params(0)).cuda())
for _ in range(6): pol.forward(obs)
torch.cuda.synchronize()" > /dev/null 2>&1
# the section-8f task kernels: multi-tool team kernel, ImageMatching renderer,
# and the PathFollowing reset-record kernel (STAR)
timeout 600 $NCU --set full --import-source on -k regex:mt_step_kernel -s 4 -c 1 -o $OUT/mt_step_multitool \
  python bench.py --config multitool --steps 2000 --fuse 250 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
timeout 600 $NCU --set full --import-source on -k regex:im_step_kernel -s 4 -c 1 -o $OUT/im_step_image \
  python bench.py --config image --steps 500 --fuse 250 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
timeout 600 $NCU --set full --import-source on -k regex:path_record_kernel -s 2 -c 1 -o $OUT/path_record_star \
  python bench.py --config star --steps 1000 --fuse 250 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
timeout 900 $NCU --metrics gpu__time_duration.sum --csv --log-file $OUT/launches_ppo.csv \
  python bench.py --config ppo --steps 64 --warmup 3 --no-cpu-baseline > $OUT/launches_ppo.log 2>&1
for f in env_step_psm env_step_ecm env_step_star policy_fwd mt_step_multitool im_step_image path_record_star; do
  [ -f $OUT/$f.ncu-rep ] || continue
  ncu -i $OUT/$f.ncu-rep --page details --csv > $OUT/${f}_details.csv 2>/dev/null
  ncu -i $OUT/$f.ncu-rep --page raw --csv > $OUT/${f}_raw.csv 2>/dev/null
  # SASS page only for the headline kernel (the pages are ~7 MB each and
  # gpurun copies back at most 64 MiB)
  [ $f = env_step_psm ] && ncu -i $OUT/$f.ncu-rep --page source --print-source sass --csv > $OUT/${f}_sass.csv 2>/dev/null
done
rm -f $OUT/*.ncu-rep
ls -la $OUT
