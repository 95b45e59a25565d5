#!/usr/bin/env python3
"""Env-step throughput on B200 (BASELINE.json metric), one JSON line on rank 0.

Workload (BASELINE.json configs[1], bench_sim protocol proj/src/bench.cpp:97-135):
PSM TargetReaching, 16384 envs per GPU, actions U[-1,1) drawn from
make_stream(seed, 0xac7104) in the reference's row-major order (bench.cpp:31-35),
every step writes the full StepResult (observations, rewards, flags,
task_error, terminal observations on ended rows) and auto-resets ended envs.

  value  = env-steps/s with state resident in HBM: sg_env_bench_step launches
           of F fused steps (actions generated in-kernel), CUDA-event timed per
           launch on the env stream, L2 flushed (256 MiB write) between launches.
  e2e    = the same metric through the host C-ABI call sg_env_step_host:
           per step H2D of the actions from pinned memory and D2H of the full
           StepResult, one launch per step.
  --impl reference: the reference's CPU path (oracle port, all host cores).

Multi-GPU (torchrun): rank r owns global envs [r*N, (r+1)*N) with per-env
streams seeded by global id (weak scaling, no collective in the timed loop);
timing = max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "env-steps/sec at 1/2/4/8 B200 (PSM reach, 16K envs/GPU); % of HBM roofline"
CONFIGS = {
    "psm": dict(robot="psm", task="target_reaching", n_envs=16384, goal_sigma=0.05,
                workload="dVRK PSM reach, 16384 envs/GPU, random actions (BASELINE configs[1])"),
    "ecm": dict(robot="ecm", task="target_reaching", n_envs=65536, goal_sigma=0.05,
                workload="dVRK ECM camera reach, 65536 envs/GPU, random actions (BASELINE configs[2])"),
    "star": dict(robot="star", task="path_following", n_envs=16384, goal_sigma=0.15,
                 workload="STAR path following, 16384 envs/GPU, random actions (BASELINE configs[3])"),
    "multitool": dict(robots=("psm", "psm", "ecm"), task="multi_tool_reaching", n_envs=16384, goal_sigma=0.05,
                      workload="trimanual MultiToolReaching (PSM + PSM + ECM camera), 16384 envs/GPU, random "
                               "actions (SURVEY 8f rank 3; not a BASELINE config)"),
    "image": dict(robot="psm", task="image_matching", n_envs=16384, goal_sigma=0.05,
                  workload="PSM ImageMatching (32x32 camera render per env-step), 16384 envs/GPU, random actions "
                           "(SURVEY 8f rank 4; not a BASELINE config)"),
    "ppo": dict(robot="psm", task="target_reaching", n_envs=16384, goal_sigma=0.05,
                workload="full PPO rollout+update on PSM reach, 16384 envs/GPU, n_steps 32, 5 epochs x 4 "
                         "minibatches, 256/128/64 ELU MLP (BASELINE configs[4])"),
}

# Policy::forward FLOPs per env (PSM): 2 * MACs of actor + critic trunks
POLICY_FLOPS_PER_ENV = 2 * 2 * (27 * 256 + 256 * 128 + 128 * 64) + 2 * (64 * 7 + 64 * 1)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def step_bytes(A: int, O: int, fused: int, reset_frac: float, tools: int = 1, step_read: int = 0) -> dict:
    """Algorithmic HBM bytes of one fused launch per env.
    Per launch: joint state q/qdot/q_target read+write (3*A*4*2), goal read+write
    and tip write (3*4*3), step/hold counters r+w (16), bench stream state r+w (16).
    Per step: generated actions written (A*4), observation row (O*4), reward,
    task_error (4+4), terminated+timed_out (2).
    Per reset (amortised by reset_frac): terminal observation row (O*4), RNG
    state r+w (16), episode counter r+w (16), reset state write + reload
    (3*A*4*2 + 24)."""
    per_launch = 3 * A * 4 * 2 + 3 * tools * 4 * 3 + 16 + 16
    per_step = A * 4 + O * 4 + 8 + 2 + step_read
    per_reset = O * 4 + 16 * tools + 16 + 3 * A * 4 * 2 + 24 * tools
    total = per_launch + fused * (per_step + reset_frac * per_reset)
    return dict(per_launch=per_launch, per_step=per_step, per_reset=per_reset,
                per_env_launch=total, per_env_step=total / fused)


def shard_plan(rank: int, world: int, n_per_gpu: int) -> dict:
    """Env sharding across ranks (weak scaling): rank r owns global envs
    [r*N, (r+1)*N); per-env RNG streams and the bench action stream are
    indexed by global env id, so the union of the shards is bit-identical to
    one device stepping world*N envs. No collective touches the step."""
    return dict(row_offset=rank * n_per_gpu, n_envs=n_per_gpu, global_n_envs=world * n_per_gpu)


def max_over_ranks(value: float, dist, device) -> float:
    """Timing reduction: the job is as slow as its slowest rank."""
    if dist is None:
        return value
    import torch
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


class Clocks:
    """SM clock and throttle-reason sampling (NVML, the source nvidia-smi reads)
    on a background thread every 5 ms while the timed region runs."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.samples = []
        self._stop = None
        self._thread = None

    def _run(self):
        import pynvml
        h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
        self.max_sm = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        while not self._stop.is_set():
            try:
                sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append((sm, rs))
            except Exception:
                pass
            self._stop.wait(0.005)

    def __enter__(self):
        import threading
        self.max_sm = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._stop = threading.Event()
            self._thread = threading.Thread(target=self._run, daemon=True)
            self._thread.start()
            time.sleep(0.05)
        except Exception:
            self._thread = None
        return self

    def __exit__(self, *a):
        if self._thread:
            self._stop.set()
            self._thread.join(timeout=2)

    def summary(self) -> dict:
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_sm, "reasons": ["unavailable"], "samples": 0}
        sm = [s for s, _ in self.samples]
        reasons = sorted({k for _, r in self.samples for k, bit in self.REASONS.items() if r & bit})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": self.max_sm, "reasons": reasons,
                "samples": len(sm), "source": "NVML every 5 ms during the timed region"}


def cpu_reference(cfg: dict, steps: int, budget_s: float, threads: int = 0):
    """The reference's CPU path (oracle port of bench_sim) on the host cores.
    Returns (env-steps/s, lanes, sample description)."""
    from oracle import oracle as O
    O.build()
    if "robots" in cfg:
        return cpu_reference_multi(O, cfg, steps, budget_s, threads)
    m = O.resolve_robot(cfg["robot"])
    task = {"path_following": O.PATH_FOLLOWING, "image_matching": O.IMAGE_MATCHING}.get(cfg["task"], O.TARGET_REACHING)
    ocfg = O.env_config(n_envs=cfg["n_envs"], seed=0, task=task, goal_sigma=cfg["goal_sigma"])
    lanes = threads or os.cpu_count() or 1
    # calibrate, then size the sample to the time budget
    secs, st = O.bench_sim(ocfg, m, cfg["n_envs"] * 3, 1, lanes)
    rate = st[0] / secs[0]
    n_steps = max(3, min(steps, int(budget_s * rate / cfg["n_envs"])))
    secs, st = O.bench_sim(ocfg, m, cfg["n_envs"] * n_steps, 1, lanes)
    sample = (f"{cfg['n_envs']} envs x {int(st[0] // cfg['n_envs'])} steps after reset + 1 warm-up step "
              f"(bench_sim protocol, serial action fill and serial resets as in the reference), fp64, "
              f"{lanes} pool lanes")
    return float(st[0] / secs[0]), lanes, sample


def cpu_reference_multi(O, cfg: dict, steps: int, budget_s: float, threads: int = 0):
    """MultiToolReaching on the oracle (bench_sim protocol: serial action fill
    from make_stream(seed, 0xac7104), reset, warm-up step, timed steps)."""
    import time
    ms = [O.resolve_robot(r) for r in cfg["robots"]]
    n = cfg["n_envs"]
    lanes = threads or os.cpu_count() or 1
    e = O.MultiToolEnv(O.env_config(n_envs=n, seed=0, task=O.MULTI_TOOL, goal_sigma=cfg["goal_sigma"]), ms,
                       threads=lanes)
    ar = O.make_stream(0, 0xAC7104)
    e.reset()
    e.step(O.fill_uniform_actions(ar, n, e.action_dim))
    done, t0 = 0, time.perf_counter()
    while done < steps and time.perf_counter() - t0 < budget_s:
        e.step(O.fill_uniform_actions(ar, n, e.action_dim))
        done += 1
    dt = time.perf_counter() - t0
    sample = (f"{n} envs x {done} steps after reset + 1 warm-up step (bench_sim protocol, serial action fill "
              f"and serial resets), fp64, {lanes} pool lanes")
    return n * done / dt, lanes, sample


def bench_ppo(args, cfg, rank, world, local, dist):
    """Config 5: env-steps/s with learning (bench_learning, bench.cpp:137-174):
    whole trainer iterations (rollout of n_steps x N env steps with the tcgen05
    policy in the loop, GAE, 5 x 4 PPO minibatch updates, NCCL gradient
    all-reduce when world > 1) timed with CUDA events, max over ranks."""
    import torch
    from paper_2310_04676_b200 import ppo, sg
    n = cfg["n_envs"]
    plan = shard_plan(rank, world, n)
    robots = cfg.get("robots", (cfg.get("robot"),))
    env = sg.VecTaskEnv(robots=robots, device=local, n_envs=n, seed=0, task=cfg["task"],
                        goal_sigma=cfg["goal_sigma"], row_offset=plan["row_offset"])
    pol = sg.Policy(env.obs_dim, env.action_dim, device=local)
    tcfg = ppo.TrainConfig(seed=0, update_precision=args.update_precision)
    tr = ppo.Trainer(env, pol, tcfg, dist=dist)
    iters = max(1, -(-args.steps // tcfg.n_steps)) if args.steps else 4
    for _ in range(max(1, args.warmup // tcfg.n_steps + 1)):
        tr.iterate()
    torch.cuda.synchronize()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(iters)]
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    stats = None
    with Clocks(local) as clk:
        for e in ev:
            e[0].record()
            tr.rollout()
            e[1].record()
            tr.gae()
            e[2].record()
            tr.update()
            e[3].record()
        torch.cuda.synchronize()
    t_ms = sum(e[0].elapsed_time(e[3]) for e in ev)
    roll_ms = sum(e[0].elapsed_time(e[1]) for e in ev) / iters
    upd_ms = sum(e[2].elapsed_time(e[3]) for e in ev) / iters
    t_ms = max_over_ranks(t_ms, dist, f"cuda:{local}")
    steps = iters * tcfg.n_steps
    value = world * n * steps / (t_ms * 1e-3)
    # dominant tensor-core kernel: policy forward on the env's observation rows
    obs = env._result().observations
    mean = torch.empty(n, env.action_dim, device=f"cuda:{local}")
    val = torch.empty(n, device=f"cuda:{local}")
    for _ in range(5):
        pol.forward(obs, mean, val)
    reps = 200
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        pol.forward(obs, mean, val)
    e1.record()
    torch.cuda.synchronize()
    fwd_s = e0.elapsed_time(e1) * 1e-3 / reps
    peak = None
    try:
        peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops"])
        pk = "measured burst"
    except Exception:
        peak, pk = 1590.0, "fallback"
    achieved = n * POLICY_FLOPS_PER_ENV / fwd_s / 1e12
    if rank == 0:
        line = dict(
            metric=METRIC, value=value, unit="env-steps/s (with learning)", n_gpus=world, steps=steps,
            warmup=args.warmup, ms_per_step=t_ms / steps, higher_is_better=True, scaling="weak", vs_baseline=None,
            dtype="bf16 policy fwd / fp32 env / " + args.update_precision + " update", data="synthetic",
            config=dict(workload=cfg["workload"], n_envs_per_gpu=n, global_envs=world * n, iterations=iters,
                        parallelism=f"env-shard x{world} + NCCL grad all-reduce" if world > 1 else "1 GPU",
                        rollout_ms_per_iter=roll_ms, update_ms_per_iter=upd_ms,
                        l2="not flushed: the rollout buffer (80 MB) and weights are reused across steps by design"),
            roofline=dict(bound="tensor", achieved=achieved, peak=peak, unit="TFLOP/s", frac=achieved / peak,
                          traffic=None, peak_kind=pk, kernel="policy_fwd_kernel (tcgen05)",
                          flops_per_env=POLICY_FLOPS_PER_ENV, avg_launch_us=fwd_s * 1e6),
            cpu_baseline=None, e2e=None,
            # ours per iteration: rollout (policy fwd, sample, env step, bootstrap per step + last fwd), GAE,
            # per minibatch gather + 6 ELU fwd + 6 ELU bwd + loss (2) + Adam (2), policy repack
            gpu_launches=iters * (4 * tcfg.n_steps + 1 + 1 + tcfg.epochs * tcfg.minibatch_count * 17 + 1),
            clocks=clk.summary(),
        )
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None, help="timed env steps (default 64000; ppo: 320)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="psm", choices=sorted(CONFIGS))
    ap.add_argument("--fuse", type=int, default=250, help="steps per fused launch")
    ap.add_argument("--e2e-steps", type=int, default=400)
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--envs", type=int, default=None,
                    help="override envs per GPU (scaling studies; the headline uses the BASELINE config)")
    ap.add_argument("--update-precision", default="bf16", choices=["fp32", "tf32", "bf16"])
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config])
    if args.envs:
        cfg["n_envs"] = args.envs
        cfg["workload"] += f" [override: {args.envs} envs/GPU]"
    if args.steps is None:
        args.steps = 320 if args.config == "ppo" else 64000

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank != 0:
            return
        total = max(args.steps, 3)
        rate, lanes, sample = cpu_reference(cfg, total, budget_s=120.0)
        line = dict(metric=METRIC, value=rate, unit="env-steps/s", n_gpus=args.gpus, steps=args.steps,
                    warmup=args.warmup, ms_per_step=1e3 * cfg["n_envs"] / rate, higher_is_better=True,
                    scaling="weak", vs_baseline=None, dtype="f64", data="synthetic", impl="reference",
                    config=dict(workload=cfg["workload"], n_envs=cfg["n_envs"]),
                    cpu_baseline=dict(value=rate, unit="env-steps/s", cores=lanes, kind="port", sample=sample),
                    e2e=dict(value=rate, unit="env-steps/s", h2d_bytes_per_step=0, d2h_bytes_per_step=0))
        print(json.dumps(line), flush=True)
        return

    import numpy as np
    import torch
    from paper_2310_04676_b200 import sg

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    if args.config == "ppo":
        bench_ppo(args, cfg, rank, world, local, dist)
        if dist:
            dist.destroy_process_group()
        return

    n = cfg["n_envs"]
    plan = shard_plan(rank, world, n)
    robots = cfg.get("robots", (cfg.get("robot"),))
    env = sg.VecTaskEnv(robots=robots, device=local, n_envs=n, seed=0, task=cfg["task"],
                        goal_sigma=cfg["goal_sigma"], row_offset=plan["row_offset"])
    A, O = env.action_dim, env.obs_dim
    env.reset()
    env.bench_begin(0, first_step=0, global_n_envs=plan["global_n_envs"])
    F = max(1, min(args.fuse, args.steps))
    # warm-up: W untimed steps (first is the bench_sim warm-up step), plus one
    # untimed fused launch so the timed launches see a warm instruction cache
    for _ in range(max(args.warmup, 1)):
        env.bench_step(1)
    env.bench_step(F)
    steps_done = max(args.warmup, 1) + F
    torch.cuda.synchronize()

    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=f"cuda:{local}")  # 256 MiB > L2
    launches = []
    k = args.steps
    while k > 0:
        launches.append(min(F, k))
        k -= launches[-1]
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in launches]
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with Clocks(local) as clk:
        for (e0, e1), kf in zip(ev, launches):
            flush.zero_()
            e0.record()
            env.bench_step(kf)
            e1.record()
        torch.cuda.synchronize()
    env.synchronize()
    steps_done += args.steps
    launch_ms = [e0.elapsed_time(e1) for e0, e1 in ev]
    t_ms = sum(launch_ms)
    t_ms = max_over_ranks(t_ms, dist, f"cuda:{local}")
    if dist:
        dist.barrier()
    value = world * n * args.steps / (t_ms * 1e-3)

    # ---- roofline of the dominant kernel (env_step_kernel, fused bench variant)
    resets = (steps_done // 300) - ((steps_done - args.steps) // 300)
    # ImageMatching reads the env's target image every step (reward + observation copy)
    wh = (O - 3 * A - 3) // 2 if cfg["task"] == "image_matching" else 0
    b = step_bytes(A, O, F, resets / max(args.steps, 1), tools=len(robots), step_read=4 * wh)
    full = [ms for ms, kf in zip(launch_ms, launches) if kf == F]
    avg_launch_s = (sum(full) / len(full)) * 1e-3 if full else t_ms * 1e-3 / len(launches)
    peak, peak_kind = peaks()
    achieved = n * b["per_env_launch"] / avg_launch_s / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", f"traffic_{args.config}.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    # ---- e2e through the host C-ABI call (pinned host buffers) --------------
    e2e = None
    if args.e2e_steps > 0:
        E = args.e2e_steps
        h_act = torch.empty((E, n, A), dtype=torch.float32).pin_memory()
        for s in range(E):  # pre-generate the bench stream (device generator), outside timing
            env.bench_step(1)
            h_act[s].copy_(env.bench_actions())
        outs = {k2: torch.empty(shape, dtype=dt).pin_memory() for k2, shape, dt in (
            ("observations", (n, O), torch.float32), ("terminal_observations", (n, O), torch.float32),
            ("rewards", (n,), torch.float32), ("task_error", (n,), torch.float32),
            ("terminated", (n,), torch.uint8), ("timed_out", (n,), torch.uint8))}
        hr = sg.HostResult()
        for k2, t in outs.items():
            setattr(hr, k2, t.data_ptr())
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        # the timed region spans a synchronized reset burst (every 300 steps),
        # so the conditional terminal-observation copy is exercised
        for s in range(E):
            env.step_host_ptr(h_act[s].data_ptr(), hr)
            if s == 0:
                ended0 = env.host_counters()[0]
                e0.record()
        e1.record()
        torch.cuda.synchronize()
        e2e_ms = e0.elapsed_time(e1)
        E -= 1
        burst_steps = -(-(env.host_counters()[0] - ended0) // n)
        e2e_ms = max_over_ranks(e2e_ms, dist, f"cuda:{local}")
        tobs_b = outs["terminal_observations"].numel() * 4
        d2h = sum(t.numel() * t.element_size() for k2, t in outs.items() if k2 != "terminal_observations") + 16
        d2h += tobs_b * burst_steps / max(E, 1)
        e2e = dict(value=world * n * E / (e2e_ms * 1e-3), unit="env-steps/s", h2d_bytes_per_step=n * A * 4,
                   d2h_bytes_per_step=d2h, steps=E, reset_burst_steps=burst_steps,
                   path="sg_env_step_host (C-ABI), 1 launch/step; terminal observations copied on steps "
                        "where rows ended")

    # ---- per-step API in a CUDA graph (1 launch per step, no fusion) --------
    single = None
    try:
        G = 64
        g = torch.cuda.CUDAGraph()
        s_ = torch.cuda.Stream()
        env.set_stream(s_)
        with torch.cuda.graph(g, stream=s_):
            for _ in range(G):
                env.bench_step(1)
        env.set_stream(None)
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        reps = 10
        tot = 0.0
        for _ in range(reps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            tot += e0.elapsed_time(e1)
        single = dict(value=n * G * reps / (tot * 1e-3), unit="env-steps/s",
                      how=f"CUDA graph of {G} single-step launches, L2 flushed between replays")
    except Exception as ex:  # informational only
        single = dict(error=str(ex)[:200])

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rate, lanes, sample = cpu_reference(cfg, 10_000, budget_s=args.cpu_budget)
        cpu = dict(value=rate, unit="env-steps/s", cores=lanes, kind="port", sample=sample)
        # HostInfo-style (bench.hpp:41-45): hardware threads, and the same
        # protocol on one pool lane (all lanes and 1 lane)
        rate1, _, sample1 = cpu_reference(cfg, 10_000, budget_s=min(5.0, args.cpu_budget), threads=1)
        cpu.update(hardware_threads=os.cpu_count(), value_1_lane=rate1, sample_1_lane=sample1)

    if rank == 0:
        line = dict(
            metric=METRIC, value=value, unit="env-steps/s", n_gpus=world, steps=args.steps, warmup=args.warmup,
            ms_per_step=t_ms / args.steps, higher_is_better=True, scaling="weak", vs_baseline=None,
            dtype="fp32", data="synthetic",
            config=dict(workload=cfg["workload"], n_envs_per_gpu=n, global_envs=world * n,
                        fused_steps_per_launch=F, parallelism=f"env-shard x{world}",
                        l2="256 MiB flush between timed launches; per-launch state read cold from HBM"),
            roofline=dict(bound="hbm", achieved=achieved, peak=peak, unit="GB/s", frac=achieved / peak,
                          traffic=traffic, peak_kind=peak_kind, kernel=(f"mt_step_kernel<T={len(robots)}, GEN> ({F} fused steps/launch)" if len(robots) > 1 else
                                  f"im_step_kernel<{cfg['robot'].upper()} chain, GEN> ({F} fused steps/launch)" if wh else
                                  f"env_step_kernel<{cfg['robot'].upper()} chain, 2 team warps, GEN> ({F} fused steps/launch)"),
                          bytes_per_env_step=b["per_env_step"], bytes_per_launch=n * b["per_env_launch"],
                          avg_launch_us=avg_launch_s * 1e6),
            cpu_baseline=cpu, e2e=e2e, single_step_launches=single,
            gpu_launches=len(launches), clocks=clk.summary(),
        )
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
