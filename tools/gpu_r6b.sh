#!/bin/bash
# Fixed cost of a fused PSM 16K launch: per-launch time vs K (1..80), L2 flushed and not.
O=gpurun_out/r6b; mkdir -p $O
for K in 1 2 5 10 20 40 80; do
  for F in "" "--no-flush"; do
    timeout 300 python3 bench.py --config psm --steps $K --fuse $K --warmup 5 --no-cpu-baseline --e2e-steps 5 $F > $O/k${K}${F}.log 2>&1
    python3 - "$O/k${K}${F}.log" "$K" "$F" <<'PY'
import json,sys
l=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("K=%s %s launch_us=%.2f per_step_us=%.3f" % (sys.argv[2], sys.argv[3] or "flush", l["roofline"]["avg_launch_us"], l["roofline"]["avg_launch_us"]/int(sys.argv[2])))
PY
  done
done
./tools/launch_probe 2>&1 | tail -4 || true
