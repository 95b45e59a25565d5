"""Which ops launch the elementwise adds inside one eager PPO update (A/B
probe, not a product path): counts of aten::add* / mul* per update with the
Python call sites."""
import collections
import sys

import torch

sys.path.insert(0, ".")
from paper_2310_04676_b200 import ppo, sg  # noqa: E402

env = sg.VecTaskEnv(robots=("psm",), n_envs=16384, seed=0)
pol = sg.Policy(env.obs_dim, env.action_dim)
tr = ppo.Trainer(env, pol, ppo.TrainConfig(seed=0, update_precision="bf16", cuda_graph=False))
tr.iterate()
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CPU], with_stack=True) as prof:
    tr.update()
    torch.cuda.synchronize()
cnt = collections.Counter()
for e in prof.events():
    if e.name.startswith("aten::add") or e.name.startswith("aten::mul") or e.name.startswith("aten::copy_"):
        stack = [s for s in (e.stack or []) if "paper_2310" in s or "torch/autograd" in s]
        cnt[(e.name, stack[0] if stack else "?")] += 1
for (name, where), c in cnt.most_common(20):
    print(f"{c:6d}  {name:20s} {where}")
print(prof.key_averages().table(sort_by="count", row_limit=25, max_name_column_width=50))
