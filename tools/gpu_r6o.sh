#!/bin/bash
# A/B: observation rows stored by every team warp after a second barrier B'(k) (SG_SPLIT_ROWS) vs the scorer alone.
O=gpurun_out/r6o; mkdir -p $O
SG_LIB_PATH=abtest/split.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x > $O/pytest_split.log 2>&1; echo pytest rc=$?; tail -2 $O/pytest_split.log
for rep in 1 2; do for lib in paper_2310_04676_b200/lib/libsg_env.so abtest/split.so; do
  for K in 20 250; do
    SG_LIB_PATH=$lib timeout 300 python3 bench.py --config psm --steps $K --fuse $K --warmup 5 --no-cpu-baseline --e2e-steps 0 > $O/ab.log 2>&1
    python3 -c "import json; l=json.loads(open('$O/ab.log').read().strip().splitlines()[-1]); print('$lib psm K=$K', round(l['roofline']['avg_launch_us'],2))" 2>&1 | tail -1
  done
done; done
for lib in paper_2310_04676_b200/lib/libsg_env.so abtest/split.so; do for c in ecm star; do
  SG_LIB_PATH=$lib timeout 300 python3 bench.py --config $c --no-cpu-baseline --e2e-steps 0 > $O/ab.log 2>&1
  python3 -c "import json; l=json.loads(open('$O/ab.log').read().strip().splitlines()[-1]); print('$lib $c', round(l['value']/1e9,2), 'G')" 2>&1 | tail -1
done; done
