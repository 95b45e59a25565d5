#!/bin/bash
# ncu captures of the PPO update's tensor-core kernels + a launch list of one PPO iteration
O=gpurun_out/r5n; mkdir -p $O
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"policy_bwd_(head|tail)|policy_train_fwd" -c 3 -o $O/ppo_kernels python3 tools/head_probe.py > $O/ncu.log 2>&1; echo ncu rc=$?; tail -n 2 $O/ncu.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches_ppo.csv python3 tools/prof_ppo.py bf16 > $O/ncu2.log 2>&1; echo ncu2 rc=$?
