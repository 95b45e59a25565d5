#!/bin/bash
# A/B: scorer DoF count (SG_SCORER_DOFS=1 / 3 vs the default 2) for PSM 16K at K=20 and K=250.
O=gpurun_out/r6l; mkdir -p $O
for rep in 1 2; do for lib in paper_2310_04676_b200/lib/libsg_env.so abtest/sd1.so abtest/sd3.so; do
  for K in 20 250; do
    SG_LIB_PATH=$lib timeout 300 python3 bench.py --config psm --steps $K --fuse $K --warmup 5 --no-cpu-baseline --e2e-steps 0 > $O/ab.log 2>&1
    python3 -c "import json; l=json.loads(open('$O/ab.log').read().strip().splitlines()[-1]); print('$lib K=$K', round(l['roofline']['avg_launch_us'],2))" 2>&1 | tail -1
  done
done; done
