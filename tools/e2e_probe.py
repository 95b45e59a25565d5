"""Where the host-buffer step (sg_env_step_host) spends its time: wall time
per call vs device time between events around it, pinned (zero-copy) vs
pageable (staged copies) buffers.  python tools/e2e_probe.py"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_04676_b200 import sg  # noqa: E402

n, steps = 16384, 300
env = sg.VecTaskEnv(robots=("psm",), n_envs=n, seed=0)
env.reset()
A, O = env.action_dim, env.obs_dim
for pinned in (True, False):
    mk = (lambda shape, dt: torch.empty(shape, dtype=dt).pin_memory()) if pinned else \
         (lambda shape, dt: torch.empty(shape, dtype=dt))
    act = mk((n, A), torch.float32)
    act.uniform_(-1, 1)
    outs = {k: mk(shape, dt) for k, shape, dt in (
        ("observations", (n, O), torch.float32), ("terminal_observations", (n, O), torch.float32),
        ("rewards", (n,), torch.float32), ("task_error", (n,), torch.float32),
        ("terminated", (n,), torch.uint8), ("timed_out", (n,), torch.uint8))}
    hr = sg.HostResult()
    for k, t in outs.items():
        setattr(hr, k, t.data_ptr())
    for _ in range(20):
        env.step_host_ptr(act.data_ptr(), hr)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for e0, e1 in evs:
        e0.record()
        env.step_host_ptr(act.data_ptr(), hr)
        e1.record()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / steps * 1e6
    dev = np.median([e0.elapsed_time(e1) * 1e3 for e0, e1 in evs])
    print(f"{'pinned (zero-copy)' if pinned else 'pageable (staged)'}: wall {wall:.1f} us/step, "
          f"device {dev:.1f} us/step, {n / wall:.1f} M env-steps/s")
