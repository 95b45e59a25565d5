#!/bin/bash
# Team-warp count x scorer DoF count sweep (abtest/z.so: scorer owns no DoF).
O=gpurun_out/r2d; mkdir -p $O
SG_LIB_PATH=abtest/z.so SG_TEAM_WARPS=3 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q > $O/pytest_z3.log 2>&1; echo z3 pytest rc=$?
for rep in 1 2; do for cfg in psm ecm star; do for K in 20 250; do
  for v in "paper_2310_04676_b200/lib/libsg_env.so 2" "abtest/z.so 2" "abtest/z.so 3" "abtest/z.so 4" "abtest/g3s1.so 3" "paper_2310_04676_b200/lib/libsg_env.so 3"; do
    set -- $v
    ST=$K; [ $K = 250 ] && ST=20000
    SG_LIB_PATH=$1 SG_TEAM_WARPS=$2 timeout 300 python3 bench.py --config $cfg --steps $ST --fuse $K --warmup 5 --runs 3 --no-cpu-baseline --e2e-steps 0 2>&1 | tail -1 | \
      python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg K=$K', '$1 G=$2', round(d['value']/1e9, 3), 'G', round(d['roofline']['avg_launch_us'],2), 'us')"
  done; done; done; done > $O/ab.txt 2>&1
cat $O/ab.txt; tail -3 $O/pytest_z3.log
