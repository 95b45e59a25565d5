"""Small runs of the round-2 kernels for compute-sanitizer (memcheck / racecheck):
the TMEM-resident policy forward (forward, fused act, act + folded bootstrap,
noise + act_noise), the persistent training forward, the fused dgrad + ELU',
the warp-specialised path record kernel, and the host step's read window."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_04676_b200 import ppo, sg  # noqa: E402

n = 300  # 3 tiles, the last ragged
pol = sg.Policy(27, 7)
pol.load_params(torch.from_numpy(pol.init_params(1)).cuda())
obs = torch.randn(n, 27, device="cuda")
pol.forward(obs)
pol.act(obs, seed=2, draw_pos=17)
sz, lp = pol.noise(n, seed=2, draw_pos=17)
pol.act_noise(obs, sz)
# act + folded bootstrap (some rows timed out)
L = sg.lib()
acts, logp, val, boot = (torch.empty(n, 7, device="cuda"), torch.empty(n, device="cuda"),
                         torch.empty(n, device="cuda"), torch.empty(n, device="cuda"))
tout = (torch.arange(n, device="cuda") % 5 == 0).to(torch.uint8)
term = torch.zeros(n, dtype=torch.uint8, device="cuda")
ls = torch.full((7,), -1.0, device="cuda")
pos = torch.zeros(1, dtype=torch.int64, device="cuda")
s0, inc = sg.make_stream(0, sg.TRAIN_STREAM)
st = torch.cuda.current_stream().cuda_stream
sg._pcheck(L.sg_policy_act_bootstrap(pol._h, obs.data_ptr(), n, 27, ls.data_ptr(), s0, inc, pos.data_ptr(), 0,
                                     acts.data_ptr(), logp.data_ptr(), None, val.data_ptr(), obs.data_ptr(), 27,
                                     tout.data_ptr(), term.data_ptr(), boot.data_ptr(), st))
# training forward + fused backward on a padded layout
layout, ls_pad, total, _ = ppo.padded_layout(27, 7)
flat = torch.randn(total, device="cuda") * 0.1
tp = sg.Policy(27, 7)
tp.set_param_layout(layout, [32, 256, 128, 64])
tp.load_params(flat)
x = torch.zeros(n, 32, dtype=torch.bfloat16, device="cuda")
x[:, :27] = torch.randn(n, 27, device="cuda").to(torch.bfloat16)
h1, h2, h3, out = (torch.empty(2, n, w, dtype=torch.bfloat16, device="cuda") for w in (256, 128, 64, 8))
tp.train_forward(x, h1, h2, h3, out)
imgs = sg.WtImages(layout, 0)
imgs.pack(flat)
g = torch.randn(n, 8, device="cuda").to(torch.bfloat16)
for l, h in ((3, h3[0]), (2, h2[0]), (1, h1[0])):
    g = sg.dgrad_elu(g, imgs.image(0, l), h.shape[1], h)
torch.cuda.synchronize()
print("policy kernels ok")
# STAR path following: fused launches (record kernel), host steps (read window)
env = sg.VecTaskEnv(robots=("star",), n_envs=200, seed=1, episode_len=5, task="path_following", goal_sigma=0.15)
env.reset()
env.bench_begin(1)
env.bench_step(7)
env.bench_step(7)
a = np.random.default_rng(0).uniform(-1, 1, (200, env.action_dim)).astype(np.float32)
for _ in range(3):
    env.step_host(a)
env.synchronize()
print("env kernels ok")
