set -x
# Round-end check on one B200: GPU tests, smoke, every bench config (headline
# PSM line with the CPU baseline, the reference arm, then configs 3-5 and the
# section-8f tasks).
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 600 python bench.py > gpurun_out/bench_psm.log 2>&1; echo bench rc=$?
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo ref rc=$?
for c in ecm star ppo multitool image; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1
done
tail -n 3 gpurun_out/*.log
