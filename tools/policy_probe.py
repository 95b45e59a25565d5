"""Policy forward timing probe (A/B only, not a product path):

  python tools/policy_probe.py [n_rows]

Times 200 back-to-back policy_fwd launches three ways -- a Python ctypes loop
(host-launch bound), the same loop behind a device-side spin gate, and one
CUDA graph of the 200 launches -- for the forward and for the fused act
(sampling) entry, so the kernel time can be separated from launch overhead."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_04676_b200 import sg  # noqa: E402


def timeit(fn, reps=200, gate=False, graph=False):
    torch.cuda.synchronize()
    if graph:
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            fn()
            s.synchronize()
            with torch.cuda.graph(g, stream=s):
                for _ in range(reps):
                    fn()
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) * 1e3 / reps
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if gate:
        torch.cuda._sleep(20_000_000)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
    pol = sg.Policy(27, 7)
    pol.load_params(torch.from_numpy(pol.init_params(0)).cuda())
    obs = torch.randn(n, 27, device="cuda")
    mean = torch.empty(n, 7, device="cuda")
    val = torch.empty(n, device="cuda")
    fwd = lambda: pol.forward(obs, mean, val)  # noqa: E731
    for _ in range(5):
        fwd()
    for name, kw in (("python loop", {}), ("gated loop", {"gate": True}), ("cuda graph", {"graph": True})):
        print(f"forward  {name:12s} {timeit(fwd, **kw):7.2f} us/launch  (n={n})")
    L = sg.lib()
    s0, inc = sg.make_stream(0, sg.TRAIN_STREAM)
    ls = torch.full((7,), -1.0, device="cuda")
    pos = torch.zeros(1, dtype=torch.int64, device="cuda")
    acts, logp = torch.empty(n, 7, device="cuda"), torch.empty(n, device="cuda")

    def act():
        st = torch.cuda.current_stream().cuda_stream
        sg._pcheck(L.sg_policy_act(pol._h, obs.data_ptr(), n, obs.stride(0), ls.data_ptr(), s0, inc, pos.data_ptr(),
                                   0, acts.data_ptr(), logp.data_ptr(), None, val.data_ptr(), st))
    for name, kw in (("gated loop", {"gate": True}), ("cuda graph", {"graph": True})):
        print(f"act      {name:12s} {timeit(act, **kw):7.2f} us/launch")


if __name__ == "__main__":
    main()
