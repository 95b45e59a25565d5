#!/bin/bash
O=gpurun_out/r2o; mkdir -p $O
for L in paper_2310_04676_b200/lib/libsg_env.so abtest/pnostag.so; do echo $L; SG_LIB_PATH=$L timeout 300 python tools/policy_probe.py 2>&1 | tail -n 6; done
SG_LIB_PATH=abtest/pprobe.so timeout 300 python tools/policy_probe.py 2>&1 | grep pprobe | tail -n 4
