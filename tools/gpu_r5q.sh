#!/bin/bash
O=gpurun_out/r5q; mkdir -p $O
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 900 $CS --tool memcheck python3 tools/sanitize_r5.py > $O/memcheck.log 2>&1; echo memcheck rc=$?; tail -n 2 $O/memcheck.log
timeout 900 $CS --tool racecheck python3 tools/sanitize_r5.py > $O/racecheck.log 2>&1; echo racecheck rc=$?; tail -n 2 $O/racecheck.log
timeout 900 $CS --tool synccheck python3 tools/sanitize_r5.py > $O/synccheck.log 2>&1; echo synccheck rc=$?; tail -n 2 $O/synccheck.log
SG_BWD_HEAD_ONETILE=1 timeout 900 $CS --tool racecheck python3 tools/sanitize_r5.py > $O/racecheck_onetile.log 2>&1; echo racecheck1 rc=$?; tail -n 2 $O/racecheck_onetile.log
