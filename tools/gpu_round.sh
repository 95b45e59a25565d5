set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 600 python bench.py > gpurun_out/bench_psm.log 2>&1; echo bench rc=$?
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo ref rc=$?
timeout 600 python bench.py --config ecm --no-cpu-baseline > gpurun_out/bench_ecm.log 2>&1
timeout 600 python bench.py --config star --no-cpu-baseline > gpurun_out/bench_star.log 2>&1
timeout 900 python bench.py --config ppo --no-cpu-baseline > gpurun_out/bench_ppo.log 2>&1
tail -n 3 gpurun_out/*.log
