#!/bin/bash
timeout 600 python tools/ppo_adds_probe.py 2>&1 | tail -60
