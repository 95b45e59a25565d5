#!/bin/bash
O=gpurun_out/r3n; mkdir -p $O
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 3 python tools/sanitize_r2.py > $O/$tool.log 2>&1; echo $tool rc=$?
  grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|ok$' $O/$tool.log | head -5
done
