#!/bin/bash
# A/B: constant-cache warm-up of the parameter block (SG_PARAM_WARM) vs default, PSM 16K K=20 and K=250.
O=gpurun_out/r6e; mkdir -p $O
for rep in 1 2 3; do for lib in paper_2310_04676_b200/lib/libsg_env.so abtest/warm.so; do
  for K in 20 250; do
    SG_LIB_PATH=$lib timeout 300 python3 bench.py --config psm --steps $K --fuse $K --warmup 5 --no-cpu-baseline --e2e-steps 0 > $O/ab.log 2>&1
    python3 -c "import json,sys; l=json.loads(open('$O/ab.log').read().strip().splitlines()[-1]); print('$lib K=$K', round(l['roofline']['avg_launch_us'],2))"
  done
done; done
