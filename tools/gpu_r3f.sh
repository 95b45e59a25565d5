#!/bin/bash
timeout 300 python tools/rollout_host_probe.py 2>&1 | tail -n 4
