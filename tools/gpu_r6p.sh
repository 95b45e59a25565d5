#!/bin/bash
# A/B: path_record_kernel blocks per SM (SG_REC_MINB 3 / 4 default / 5), STAR path following 16K.
O=gpurun_out/r6p; mkdir -p $O
for rep in 1 2; do for lib in paper_2310_04676_b200/lib/libsg_env.so abtest/rec3.so abtest/rec5.so; do
  SG_LIB_PATH=$lib timeout 300 python3 bench.py --config star --no-cpu-baseline --e2e-steps 0 > $O/ab.log 2>&1
  python3 -c "import json; l=json.loads(open('$O/ab.log').read().strip().splitlines()[-1]); print('$lib star', round(l['value']/1e9,3), 'G')" 2>&1 | tail -1
done; done
