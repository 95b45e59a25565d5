#!/bin/bash
O=gpurun_out/r5p; mkdir -p $O
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"policy_train_fwd" -c 1 -o $O/train_fwd python3 tools/head_probe.py > $O/ncu.log 2>&1; echo ncu rc=$?; tail -n 2 $O/ncu.log
