#!/bin/bash
# Round-2 closing check on one B200: GPU tests, smoke, driver command (plain and under torchrun),
# reference arm, every config, and the ncu launch list of the driver command.
O=gpurun_out/r6f; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo pytest rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$?
timeout 600 python3 bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench_driver.log 2>&1; echo driver rc=$?
timeout 600 python3 -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench_torchrun.log 2>&1; echo torchrun rc=$?
timeout 600 python3 bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $O/bench_ref.log 2>&1; echo ref rc=$?
timeout 600 python3 bench.py > $O/bench_psm_default.log 2>&1; echo psm rc=$?
for c in ecm star policy ppo multitool image; do
  timeout 900 python3 bench.py --config $c > $O/bench_$c.log 2>&1; echo $c rc=$?
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_driver.csv python3 bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > $O/ncu_driver.log 2>&1; echo ncu rc=$?
tail -n 3 $O/pytest_gpu.log; tail -n 1 $O/smoke.log
for f in $O/bench_*.log; do echo "$f: $(tail -n 1 $f | cut -c1-200)"; done
