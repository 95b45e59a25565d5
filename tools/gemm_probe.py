import torch, time
B = 131072
shapes = [(256, 27), (128, 256), (64, 128), (7, 64)]
def t(f, reps=20):
    for _ in range(3): f()
    torch.cuda.synchronize(); e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): f()
    e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1)/reps*1000
for dt in (torch.float32, torch.bfloat16):
    torch.backends.cuda.matmul.allow_tf32 = True
    for N, K in shapes:
        gy = torch.randn(B, N, device='cuda', dtype=dt); x = torch.randn(B, K, device='cuda', dtype=dt)
        res = {}
        res['mm gyT x'] = t(lambda: gy.t() @ x)
        res['mm xT gy'] = t(lambda: x.t() @ gy)
        for ch in (2048, 4096, 16384):
            S = B // ch
            res[f'bmm{ch}'] = t(lambda: torch.bmm(gy.view(S, ch, N).transpose(1, 2), x.view(S, ch, K)).sum(0))
        W = torch.randn(N, K, device='cuda', dtype=dt)
        res['fwd addmm'] = t(lambda: torch.addmm(torch.zeros(N, device='cuda', dtype=dt), x, W.t()))
        res['bwd gx'] = t(lambda: gy @ W)
        print(dt, N, K, {k: round(v, 1) for k, v in res.items()})
