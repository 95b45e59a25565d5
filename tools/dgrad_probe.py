"""Timing of the backward through one hidden layer (A/B probe): the TMA-epilogue
fused kernel (sg_policy_dgrad_elu_colsum, dZ + next db), the per-row fused
kernel (sg_policy_dgrad_elu) + a colsum pass, and the library GEMM + the
train.cu ELU'/colsum pass (the default path)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2310_04676_b200 import sg, ppo  # noqa: E402

m = 131072
def t(fn, reps=50):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps
layout, _, total, _ = ppo.padded_layout(27, 7)
flat = torch.randn(total, device="cuda") * 0.1
imgs = sg.WtImages(layout, 0)
imgs.pack(flat)
for n_in, k, l in [(256, 128, 1), (128, 64, 2), (64, 8, 3)]:
    (w0, o, i), _ = layout[l]
    Wm = flat[w0: w0 + o * i].view(o, i).to(torch.bfloat16)
    dy = torch.randn(m, k, device="cuda").to(torch.bfloat16)
    h = torch.randn(m, n_in, device="cuda").to(torch.bfloat16)
    cs = torch.zeros(n_in, device="cuda")
    a = t(lambda: sg.layer_backward(dy, imgs.image(0, l), n_in, h, cs))
    wg = torch.zeros(k, n_in, device="cuda")
    a2 = t(lambda: sg.layer_backward(dy, imgs.image(0, l), n_in, h, cs, wg))
    b = t(lambda: sg.elu_backward_colsum(None, sg.dgrad_elu(dy, imgs.image(0, l), n_in, h), cs, out=False))
    c = t(lambda: sg.elu_backward_colsum(h, dy @ Wm, cs))
    mb = m * (k + 2 * n_in) * 2 / 1e6
    print(f"(n_in {n_in}, k {k}) tma {a:.1f} us  +wgrad {a2:.1f} us  per-row {b:.1f} us  library {c:.1f} us"
          f"  ({mb:.0f} MB: {mb / a:.2f} TB/s)")
