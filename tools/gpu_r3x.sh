#!/bin/bash
O=gpurun_out/r3x; mkdir -p $O
timeout 600 ncu --clock-control none --set full --import-source on -k regex:wgrad -c 4 -o $O/wgrad python tools/wgrad_probe.py > /dev/null 2>&1; echo rc=$?
ncu -i $O/wgrad.ncu-rep --page details --csv 2>/dev/null | grep -E '"Duration"|Issue Slots Busy|Achieved Occupancy|"Memory Throughput"|Registers Per' | cut -c1-60,100-220
