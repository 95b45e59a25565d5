"""Backward head / tail kernels at the minibatch size (ncu target, A/B only)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2310_04676_b200 import sg, ppo  # noqa: E402

m = 131072
layout, _, total, _ = ppo.padded_layout(27, 7)
flat = torch.randn(total, device="cuda") * 0.1
imgs = sg.WtImages(layout, 0)
imgs.pack(flat)
dy = torch.randn(m, 128, device="cuda").to(torch.bfloat16)
h = torch.randn(m, 256, device="cuda").to(torch.bfloat16)
x0 = torch.randn(m, 32, device="cuda").to(torch.bfloat16)
cs, wg, wg0 = torch.zeros(256, device="cuda"), torch.zeros(128, 256, device="cuda"), torch.zeros(256, 32, device="cuda")
dy3 = torch.randn(m, 8, device="cuda").to(torch.bfloat16)
h3, h2 = torch.randn(m, 64, device="cuda").to(torch.bfloat16), torch.randn(m, 128, device="cuda").to(torch.bfloat16)
z = lambda *s: torch.zeros(*s, device="cuda")  # noqa: E731
for _ in range(3):
    sg.layer_backward(dy, imgs.image(0, 1), 256, h, cs, wg, x0=x0, wgrad0=wg0)
    sg.backward_tail(dy3, imgs.image(0, 3), imgs.image(0, 2), h3, h2, z(8), z(8, 64), z(64), z(64, 128), z(128))
# the training forward on the same minibatch size (bf16 obs rows, padded layout)
O, A = 27, 7
tp = sg.Policy(O, A)
tp.set_param_layout(layout, [32, 256, 128, 64])
tp.load_params(flat)
obs = torch.randn(m, 32, device="cuda").to(torch.bfloat16)
acts = [torch.empty(2, m, w, device="cuda", dtype=torch.bfloat16) for w in (256, 128, 64, 8)]
for _ in range(2):
    tp.train_forward(obs, *acts)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    sg.layer_backward(dy, imgs.image(0, 1), 256, h, cs, wg, x0=x0, wgrad0=wg0)
e1.record()
torch.cuda.synchronize()
print(f"head {e0.elapsed_time(e1) * 1e3 / 20:.1f} us")
