"""Small runs of the PPO backward kernels for compute-sanitizer (memcheck /
racecheck / synccheck): sg_policy_layer_backward (64 / 128 / 256 wide, with
and without the first layer's weight gradient -- the pipelined head kernel and
the one-tile kernel), sg_policy_backward_tail, sg_policy_wgrad, on ragged row
counts (several tiles per CTA on a small grid is not reachable: the grid is
min(tiles, SMs), so a few hundred rows give one tile per CTA, and 40,000 rows
give two-plus tiles per CTA)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_04676_b200 import ppo, sg  # noqa: E402

layout, _, total, _ = ppo.padded_layout(27, 7)
flat = torch.randn(total, device="cuda") * 0.1
imgs = sg.WtImages(layout, 0)
imgs.pack(flat)
z = lambda *s: torch.zeros(*s, device="cuda")  # noqa: E731
bf = lambda *s: torch.randn(*s, device="cuda").to(torch.bfloat16)  # noqa: E731
for m in (300, 40000):
    for n_in, k, l in ((256, 128, 1), (128, 64, 2), (64, 8, 3)):
        sg.layer_backward(bf(m, k), imgs.image(0, l), n_in, bf(m, n_in), z(n_in), z(k, n_in))
    sg.layer_backward(bf(m, 128), imgs.image(0, 1), 256, bf(m, 256), z(256), z(128, 256), x0=bf(m, 32),
                      wgrad0=z(256, 32))
    sg.backward_tail(bf(m, 8), imgs.image(0, 3), imgs.image(0, 2), bf(m, 64), bf(m, 128), z(8), z(8, 64), z(64),
                     z(64, 128), z(128))
    part = torch.empty(148 * 128 * 256, device="cuda")
    for o, i in ((256, 32), (128, 256), (64, 128), (8, 64)):
        sg.wgrad(bf(m, o), bf(m, i), part, z(o, i))
torch.cuda.synchronize()
print("sanitize_r5 done")
