"""Host cost of one trainer rollout call (CUDA-graph replay) vs its GPU time
(A/B probe, not a product path)."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2310_04676_b200 import ppo, sg  # noqa: E402

env = sg.VecTaskEnv(robots=("psm",), n_envs=16384, seed=0)
tr = ppo.Trainer(env, sg.Policy(env.obs_dim, env.action_dim), ppo.TrainConfig(seed=0))
for _ in range(3):
    tr.rollout()
torch.cuda.synchronize()
for n in (10, 100):
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        tr.rollout()
    t1 = time.perf_counter()
    e1.record()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{n} rollouts: host enqueue {1e6 * (t1 - t0) / n:.1f} us/rollout, wall {1e6 * (t2 - t0) / n:.1f}, "
          f"GPU {1e3 * e0.elapsed_time(e1) / n:.1f} us/rollout")
g = tr.rollout_graph
t0 = time.perf_counter()
for _ in range(100):
    g.replay()
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"bare graph.replay host {1e6 * (t1 - t0) / 100:.1f} us")
