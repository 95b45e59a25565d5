import sys, torch, time
sys.path.insert(0, '.')
from paper_2310_04676_b200 import sg, ppo
env = sg.VecTaskEnv(robots=("psm",), n_envs=16384, seed=0)
pol = sg.Policy(env.obs_dim, env.action_dim)
tr = ppo.Trainer(env, pol, ppo.TrainConfig(seed=0, update_precision=sys.argv[1], cuda_graph=False))
tr.iterate(); torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    tr.rollout(); tr.gae(); tr.update(); torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25, max_name_column_width=60))
t0=time.time(); tr.update(); torch.cuda.synchronize(); print("update wall", time.time()-t0)
