"""Rollout timing with and without the CUDA-graph path (config 5 sizes)."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_04676_b200 import sg, ppo  # noqa: E402
for graph in (False, True):
    env = sg.VecTaskEnv(robots=("psm",), n_envs=16384, seed=0)
    pol = sg.Policy(env.obs_dim, env.action_dim)
    tr = ppo.Trainer(env, pol, ppo.TrainConfig(seed=0, cuda_graph=graph))
    tr.iterate(); tr.iterate()
    torch.cuda.synchronize()
    for rep in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); tr.rollout(); e1.record(); torch.cuda.synchronize()
        print("graph" if graph else "eager", rep, round(e0.elapsed_time(e1), 3), "ms")
    if graph:
        from torch.profiler import profile, ProfilerActivity
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            tr.rollout(); torch.cuda.synchronize()
        print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=12, max_name_column_width=70))
