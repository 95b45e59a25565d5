import torch, time
B=131072
for (o,i) in ((256,32),(128,256),(64,128),(8,64)):
    gy=torch.randn(B,o,device='cuda',dtype=torch.bfloat16); x=torch.randn(B,i,device='cuda',dtype=torch.bfloat16)
    def a():
        S=B//4096; return torch.bmm(gy.view(S,4096,-1).transpose(1,2), x.view(S,4096,-1)).sum(0).float()
    def b(): return torch.mm(gy.t(), x, out_dtype=torch.float32)
    def c():
        S=B//4096; return torch.bmm(gy.view(S,4096,-1).transpose(1,2), x.view(S,4096,-1), out_dtype=torch.float32).sum(0)
    ref=(gy.float().t()@x.float())
    for name,f in (("bmm+sum",a),("mm fp32",b),("bmm fp32+sum",c)):
        try:
            for _ in range(3): r=f()
            torch.cuda.synchronize(); e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20): r=f()
            e1.record(); torch.cuda.synchronize()
            err=((r-ref).abs().max()/ref.abs().max()).item()
            print(o,i,name, round(e0.elapsed_time(e1)/20*1000,1),"us relerr",f"{err:.2e}")
        except Exception as ex: print(o,i,name,"ERR",str(ex)[:100])
