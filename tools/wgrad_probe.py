"""Timing of sg_policy_wgrad vs torch.mm for the four layer shapes (A/B probe)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2310_04676_b200 import sg  # noqa: E402

m = 131072
partial = torch.empty(148 * 128 * 256, device="cuda")
def t(fn, reps=50):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps
for o, i in [(256, 32), (128, 256), (64, 128), (8, 64)]:
    dy = torch.randn(m, o, device="cuda").to(torch.bfloat16)
    x = torch.randn(m, i, device="cuda").to(torch.bfloat16)
    out = torch.empty(o, i, device="cuda")
    a = t(lambda: sg.wgrad(dy, x, partial, out))
    b = t(lambda: torch.mm(dy.t(), x, out_dtype=torch.float32, out=out))
    mb = m * (o + i) * 2 / 1e6
    print(f"({o},{i}) wgrad {a:.1f} us  mm {b:.1f} us  ({mb:.0f} MB operands: {mb / a * 1e-3:.2f} TB/s)")
