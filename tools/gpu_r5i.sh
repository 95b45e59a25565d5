#!/bin/bash
O=gpurun_out/r5i; mkdir -p $O
python3 tools/head_probe.py
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"policy_bwd_(head|tail)" -c 2 -o $O/bwd python3 tools/head_probe.py > $O/ncu.log 2>&1; echo ncu rc=$?; tail -n 3 $O/ncu.log
