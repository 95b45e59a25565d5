"""Small PPO iteration (policy forward, sampling, GAE, update kernels) for compute-sanitizer."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_04676_b200 import sg, ppo  # noqa: E402

env = sg.VecTaskEnv(robots=("psm",), n_envs=256, seed=0)
pol = sg.Policy(env.obs_dim, env.action_dim)
tr = ppo.Trainer(env, pol, ppo.TrainConfig(seed=0, n_steps=32, cuda_graph=False))
print(tr.iterate()["iteration"], "ok")
