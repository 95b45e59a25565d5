"""N>1 path on CPU (gloo, world_size 2): bench.py's shard plan gives each rank
the global rows [r*N, (r+1)*N); stepping the shards independently (no
collective in the step) reproduces the single-device run bit for bit, and the
timing reduction is the max over ranks."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, steps, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist
    import bench
    from oracle import oracle as O
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    plan = bench.shard_plan(rank, world, n)
    m = O.resolve_robot("psm")
    e = O.Env(O.env_config(n_envs=plan["n_envs"], seed=7, row_offset=plan["row_offset"]), m)
    e.reset()
    ar = O.make_stream(7, 0xAC7104)
    for _ in range(steps):  # each rank slices its rows of the global bench stream
        a = O.fill_uniform_actions(ar, plan["global_n_envs"], m.dof)
        e.step(a[plan["row_offset"]: plan["row_offset"] + plan["n_envs"]])
    obs = torch.from_numpy(e.obs()[0])
    out = [torch.empty_like(obs) for _ in range(world)]
    dist.all_gather(out, obs)
    t = bench.max_over_ranks(float(rank + 1.5), dist, "cpu")
    if rank == 0:
        q.put((torch.cat(out).numpy(), t))
    dist.destroy_process_group()


def test_two_rank_shards_equal_single_run(oracle):
    n, steps, world = 48, 305, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, steps, q)) for r in range(world)]
    for p in procs:
        p.start()
    gathered, t = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    m = oracle.resolve_robot("psm")
    full = oracle.Env(oracle.env_config(n_envs=world * n, seed=7), m)
    full.reset()
    ar = oracle.make_stream(7, 0xAC7104)
    for _ in range(steps):
        full.step(oracle.fill_uniform_actions(ar, world * n, m.dof))
    assert np.array_equal(gathered, full.obs()[0])
    assert t == 2.5  # max over ranks of (rank + 1.5)
