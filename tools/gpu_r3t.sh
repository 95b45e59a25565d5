#!/bin/bash
timeout 600 python tools/gw_probe2.py 2>&1 | tail -n 8
