"""Weight-gradient GEMM formulations for the update's K = 131,072 reductions
(A/B probe): dW = dY^T X as mm(dY.t(), X) (current), mm(X.t(), dY) into the
transposed view, and both trunks as one bmm."""
import torch

m = 131072
shapes = [(256, 32), (128, 256), (64, 128), (8, 64)]  # (out, in)
def t(fn, reps=50):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps
tot = {}
for o, i in shapes:
    dy = torch.randn(2, m, o, device="cuda").to(torch.bfloat16)
    x = torch.randn(2, m, i, device="cuda").to(torch.bfloat16)
    out = torch.empty(2, o, i, device="cuda")
    outT = torch.empty(2, i, o, device="cuda")
    r = {}
    r["mm dY^T X (x2)"] = t(lambda: [torch.mm(dy[k].t(), x[k], out_dtype=torch.float32, out=out[k]) for k in (0, 1)])
    r["mm X^T dY (x2)"] = t(lambda: [torch.mm(x[k].t(), dy[k], out_dtype=torch.float32, out=outT[k]) for k in (0, 1)])
    try:
        r["bmm dY^T X"] = t(lambda: torch.bmm(dy.transpose(1, 2), x, out_dtype=torch.float32, out=out))
    except Exception as e:
        r["bmm dY^T X"] = float("nan")
    try:
        r["bmm fp32-out via bf16 + float"] = t(lambda: torch.bmm(dy.transpose(1, 2), x).float())
    except Exception:
        pass
    print((o, i), {k: round(v, 1) for k, v in r.items()})
    for k, v in r.items():
        tot[k] = tot.get(k, 0) + v
print("total per minibatch (both trunks):", {k: round(v, 1) for k, v in tot.items()})
