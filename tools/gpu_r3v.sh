#!/bin/bash
timeout 600 python tools/wgrad_probe.py 2>&1 | tail -n 4
