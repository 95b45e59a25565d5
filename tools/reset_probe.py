"""Fused-step cost with and without reset bursts (episode_len 300 vs never):
isolates the reset_row share of a bench launch.  python tools/reset_probe.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_04676_b200 import sg  # noqa: E402


def rate(robot, task, n, sigma, ep_len, fuse=250, launches=8):
    env = sg.VecTaskEnv(robots=(robot,), n_envs=n, seed=0, task=task, goal_sigma=sigma, episode_len=ep_len)
    env.reset()
    env.bench_begin(0)
    for _ in range(3):
        env.bench_step(fuse)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(launches):
        env.bench_step(fuse)
    e1.record()
    torch.cuda.synchronize()
    return n * fuse * launches / (e0.elapsed_time(e1) * 1e-3) / 1e9


for robot, task, n, sigma in (("psm", "target_reaching", 16384, 0.05), ("ecm", "target_reaching", 65536, 0.05),
                              ("star", "path_following", 16384, 0.15), ("star", "target_reaching", 16384, 0.15)):
    print(robot, task, "resets every 300:", round(rate(robot, task, n, sigma, 300), 3),
          "never:", round(rate(robot, task, n, sigma, 1 << 30), 3), "G env-steps/s")
