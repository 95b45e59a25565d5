"""Small runs of every kernel family for compute-sanitizer (memcheck / racecheck)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_04676_b200 import sg  # noqa: E402

for kw in (dict(robots=("psm",), task="target_reaching"), dict(robots=("star",), task="path_following", goal_sigma=0.15),
           dict(robots=("psm", "psm", "ecm"), task="multi_tool_reaching"), dict(robots=("psm",), task="image_matching")):
    env = sg.VecTaskEnv(n_envs=70, seed=1, episode_len=5, **kw)
    env.reset()
    env.bench_begin(1)
    env.bench_step(1)
    env.bench_step(7)
    a = torch.from_numpy(np.random.default_rng(0).uniform(-1.2, 1.2, (70, env.action_dim)).astype(np.float32)).cuda()
    for _ in range(6):
        env.step(a)
    env.step_host(a.cpu().numpy())
    env.synchronize()
    print(kw["task"], "ok")
