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
import math
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
    "policy": dict(robot="psm", task="target_reaching", n_envs=16384, goal_sigma=0.05,
                   workload="random-init-policy rollout on PSM reach, 16384 envs/GPU: tcgen05 policy forward + "
                            "Gaussian sampling + env step per step, no update (north_star; ppo.cpp:258-313)"),
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


def _np_policy(O: int, A: int, seed: int = 0):
    """Random-init fp64 MLP weights for the CPU rollout baseline with the
    reference's init law (policy.cpp:87-102: N(0, 2/fan_in), last layer x0.01,
    zero biases; drawn with numpy here -- the values do not change the cost)."""
    import numpy as np
    rng = np.random.default_rng(seed)
    dims = [O, 256, 128, 64]
    trunks = []
    for out_last in (A, 1):
        layers = []
        for l in range(4):
            i, o = dims[l], (dims[l + 1] if l < 3 else out_last)
            W = rng.normal(0.0, (2.0 / i) ** 0.5, size=(o, i)) * (0.01 if l == 3 else 1.0)
            layers.append((W, np.zeros(o)))
        trunks.append(layers)
    return trunks


def _np_forward(trunks, x):
    """Policy::forward / trunk_forward (policy.cpp:110-161): x W^T + b, ELU
    (expm1, policy.cpp:33) on the hidden layers, fp64. Runs on torch's CPU
    kernels (multithreaded BLAS GEMM + vectorised ELU over all host threads)
    as the stand-in for the reference's Eigen GEMMs on its thread pool."""
    import torch
    h0 = torch.from_numpy(x)
    outs = []
    for layers in trunks:
        h = h0
        for l, (W, b) in enumerate(layers):
            h = torch.addmm(torch.from_numpy(b), h, torch.from_numpy(W).t())
            if l < 3:
                h = torch.nn.functional.elu(h)
        outs.append(h.numpy())
    return outs[0], outs[1][:, 0]


def cpu_policy_reference(cfg: dict, steps: int, budget_s: float, threads: int = 0):
    """The reference's rollout step on the host cores (ppo.cpp:258-313 without
    the update): Policy::forward in fp64, one serial trainer stream for the
    Gaussian noise (make_stream(seed, 0x7261696e)), log-probs, env step on the
    oracle's pool, bootstrap forward of the timed-out rows. Returns
    (env-steps/s, lanes, sample description)."""
    import numpy as np
    from oracle import oracle as O
    O.build()
    m = O.resolve_robot(cfg["robot"])
    n = cfg["n_envs"]
    lanes = threads or os.cpu_count() or 1
    import torch
    torch.set_num_threads(lanes)
    e = O.Env(O.env_config(n_envs=n, seed=0, goal_sigma=cfg["goal_sigma"]), m, threads=lanes)
    obs = e.reset()
    A, Od = m.dof, obs.shape[1]
    trunks = _np_policy(Od, A)
    log_std = np.full(A, -1.0)
    sigma = np.exp(log_std)
    rs = O.make_stream(0, 0x7261696E)
    half_log_2pi = 0.9189385332046727

    def one_step(obs):
        mean, value = _np_forward(trunks, obs)
        z = O.fill_normals(rs, n, A)
        act = mean + sigma * z
        logp = (-0.5 * z * z - log_std - half_log_2pi).sum(1)
        e.step(act)
        r = e.result()
        boot = r["timed_out"].astype(bool) & ~r["terminated"].astype(bool)
        if boot.any():
            _np_forward(trunks, e.obs()[1][boot])
        return e.obs()[0], logp, value

    obs = one_step(obs)[0]  # warm-up step (timing starts after the first step)
    done, t0 = 0, time.perf_counter()
    while done < steps and time.perf_counter() - t0 < budget_s:
        obs = one_step(obs)[0]
        done += 1
    dt = time.perf_counter() - t0
    sample = (f"{n} envs x {done} rollout steps after a warm-up step (fp64 Policy::forward on torch CPU kernels, "
              f"serial trainer-stream noise, oracle env step on {lanes} pool lanes, bootstrap forward)")
    return n * done / dt, lanes, sample


def cpu_ppo_reference(cfg: dict, budget_s: float, n_envs: int = 2048, threads: int = 0):
    """Config 5 on the host cores (bench_learning, bench.cpp:137-174): whole
    trainer iterations (ppo.cpp:243-341) of a bounded sample -- n_envs envs
    instead of the GPU's 16,384; rollout and update costs are per sample, so
    env-steps/s with learning does not depend on N -- in fp64: rollout of
    n_steps (Policy::forward, trainer-stream noise, log-probs, oracle env step
    on the pool, bootstrap forward of timed-out rows), GAE (rollout.cpp:42-76,
    global advantage normalisation), epochs x minibatches of the PPO loss
    (ppo.cpp:90-154; gradients by torch autograd on CPU instead of the
    reference's hand-written backward), global-norm clip and Adam
    (ppo.cpp:50-64, 157-224). The minibatch shuffle uses torch.randperm, not
    the trainer stream (same cost class). Returns (env-steps/s, lanes, sample)."""
    import numpy as np
    import torch
    import torch.nn.functional as F
    from oracle import oracle as O
    from paper_2310_04676_b200.ppo import HALF_LOG_2PI, LOG_STD_MAX, LOG_STD_MIN, TrainConfig
    O.build()
    lanes = threads or os.cpu_count() or 1
    torch.set_num_threads(lanes)
    tc = TrainConfig(seed=0)
    m = O.resolve_robot(cfg["robot"])
    n, T, A = n_envs, tc.n_steps, m.dof
    e = O.Env(O.env_config(n_envs=n, seed=0, goal_sigma=cfg["goal_sigma"]), m, threads=lanes)
    obs = e.reset()
    Od = obs.shape[1]
    params = [torch.from_numpy(x).clone().requires_grad_(True)
              for trunk in _np_policy(Od, A) for W, b in trunk for x in (W, b)]
    log_std = torch.full((A,), tc.init_log_std, dtype=torch.float64, requires_grad=True)
    params.append(log_std)
    adam_m = [torch.zeros_like(p) for p in params]
    adam_v = [torch.zeros_like(p) for p in params]
    rs = O.make_stream(0, 0x7261696E)

    def forward(x):
        outs = []
        for t in range(2):
            h = x
            for l in range(4):
                h = F.linear(h, params[8 * t + 2 * l], params[8 * t + 2 * l + 1])
                if l < 3:
                    h = F.elu(h)
            outs.append(h)
        return outs[0], outs[1][:, 0]

    def iteration(obs, step_no):
        buf = dict(obs=np.zeros((T, n, Od)), act=np.zeros((T, n, A)), logp=np.zeros((T, n)),
                   val=np.zeros((T, n)), rew=np.zeros((T, n)), term=np.zeros((T, n), bool),
                   tout=np.zeros((T, n), bool), boot=np.zeros((T, n)))
        ls = log_std.detach().clamp(LOG_STD_MIN, LOG_STD_MAX).numpy()
        with torch.no_grad():
            for t in range(T):
                mean, value = forward(torch.from_numpy(obs))
                z = O.fill_normals(rs, n, A)
                act = mean.numpy() + np.exp(ls) * z
                buf["obs"][t], buf["act"][t], buf["val"][t] = obs, act, value.numpy()
                buf["logp"][t] = (-0.5 * z * z - ls - HALF_LOG_2PI).sum(1)
                e.step(act)
                r = e.result()
                buf["rew"][t], buf["term"][t], buf["tout"][t] = r["rewards"], r["terminated"], r["timed_out"]
                bmask = buf["tout"][t] & ~buf["term"][t]
                if bmask.any():
                    buf["boot"][t][bmask] = forward(torch.from_numpy(e.obs()[1][bmask]))[1].numpy()
                obs = e.obs()[0]
            last = forward(torch.from_numpy(obs))[1].numpy()
        adv, ret = np.zeros((T, n)), np.zeros((T, n))
        running = np.zeros(n)
        for t in range(T - 1, -1, -1):  # rollout.cpp:42-66, vectorised over envs
            vn = last if t == T - 1 else buf["val"][t + 1]
            ended = buf["term"][t] | buf["tout"][t]
            nxt = np.where(buf["term"][t], 0.0, np.where(buf["tout"][t], buf["boot"][t], vn))
            delta = buf["rew"][t] + tc.gamma * nxt - buf["val"][t]
            running = np.where(ended, delta, delta + tc.gamma * tc.lam * running)
            adv[t], ret[t] = running, running + buf["val"][t]
        adv = (adv - adv.mean()) / (adv.std() + 1e-8)
        flat = {k: torch.from_numpy(v.reshape(T * n, *v.shape[2:])) for k, v in
                (("obs", buf["obs"]), ("act", buf["act"]), ("logp", buf["logp"]), ("adv", adv), ("ret", ret))}
        mb = (T * n) // tc.minibatch_count
        for _ in range(tc.epochs):
            perm = torch.randperm(T * n)
            for k in range(tc.minibatch_count):
                idx = perm[k * mb:(k + 1) * mb]
                mean, value = forward(flat["obs"][idx])
                lsc = log_std.clamp(LOG_STD_MIN, LOG_STD_MAX)
                logp = (-0.5 * ((flat["act"][idx] - mean) * torch.exp(-lsc)) ** 2 - lsc - HALF_LOG_2PI).sum(1)
                ratio = torch.exp(logp - flat["logp"][idx])
                a_ = flat["adv"][idx]
                surr = torch.minimum(ratio * a_, ratio.clamp(1 - tc.clip_eps, 1 + tc.clip_eps) * a_)
                loss = (-surr.mean() + tc.value_coef * 0.5 * ((value - flat["ret"][idx]) ** 2).mean()
                        - tc.entropy_coef * (lsc + 0.5 + HALF_LOG_2PI).sum())
                grads = torch.autograd.grad(loss, params)
                gn = math.sqrt(sum(float((g * g).sum()) for g in grads))
                if not math.isfinite(gn):
                    raise RuntimeError("cpu_ppo_reference: non-finite gradient")
                sc = min(1.0, tc.max_grad_norm / (gn + 1e-6))
                step_no += 1
                with torch.no_grad():
                    for p, g, m1, v1 in zip(params, grads, adam_m, adam_v):
                        g = g * sc
                        m1.mul_(0.9).add_(g, alpha=0.1)
                        v1.mul_(0.999).addcmul_(g, g, value=0.001)
                        mh = m1 / (1 - 0.9 ** step_no)
                        vh = v1 / (1 - 0.999 ** step_no)
                        p.sub_(tc.learning_rate * mh / (vh.sqrt() + 1e-8))
        return obs, step_no

    obs, step_no = iteration(obs, 0)  # warm-up iteration
    done, t0 = 0, time.perf_counter()
    while True:
        obs, step_no = iteration(obs, step_no)
        done += 1
        if time.perf_counter() - t0 >= budget_s:
            break
    dt = time.perf_counter() - t0
    sample = (f"{n} envs x {done} PPO iterations ({T} rollout steps + {tc.epochs} x {tc.minibatch_count} minibatch "
              f"updates) after a warm-up iteration: fp64 policy / loss / Adam on torch CPU kernels (autograd "
              f"backward), oracle env step on {lanes} pool lanes")
    return n * T * done / dt, lanes, sample


def policy_fwd_seconds(pol, obs, mean, val, dev, reps=200):
    """Average duration of one policy_fwd launch: CUDA events around one
    replay of a CUDA graph of `reps` back-to-back launches on the launching
    stream (the graph removes the per-call host launch path; a Python loop of
    launches measures ~2 us more per launch)."""
    import torch
    s = torch.cuda.Stream(dev)
    s.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(s):
        for _ in range(5):
            pol.forward(obs, mean, val)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                pol.forward(obs, mean, val)
        g.replay()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        g.replay()
        e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e-3 / reps


def bench_policy(args, cfg, rank, world, local, dist):
    """north_star's random-init-policy workload: rollout-only env-steps/s with
    the tcgen05 policy in the loop (ppo.cpp:258-313: policy forward -> Gaussian
    sample on the trainer stream -> env step -> rollout buffer + timeout
    bootstrap), no PPO update. Whole 32-step rollouts (one CUDA-graph replay
    each) are timed with CUDA events, L2 flushed before each, gated like the
    env bench; max over ranks."""
    import torch
    from paper_2310_04676_b200 import ppo, sg
    n = cfg["n_envs"]
    dev = f"cuda:{local}"
    plan = shard_plan(rank, world, n)
    env = sg.VecTaskEnv(robots=(cfg["robot"],), device=local, n_envs=n, seed=0, task=cfg["task"],
                        goal_sigma=cfg["goal_sigma"], row_offset=plan["row_offset"])
    pol = sg.Policy(env.obs_dim, env.action_dim, device=local)
    tcfg = ppo.TrainConfig(seed=0)
    tr = ppo.Trainer(env, pol, tcfg, dist=dist)
    T = tcfg.n_steps
    rollouts = max(1, -(-args.steps // T))
    for _ in range(max(2, -(-args.warmup // T))):  # the 2nd rollout captures the graph the timed ones replay
        tr.rollout()
    torch.cuda.synchronize()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)

    class _Roll:
        def bench_step(self, k):
            tr.rollout()

    runs = max(1, args.runs)
    with Clocks(local) as clk:
        res = timed_runs(_Roll(), [T] * rollouts, flush, runs, not args.no_gate, dist, dev, gate_us=1000.0)
    tr.env.synchronize()
    t_runs = [r["t_ms"] for r in res]
    t_ms = statistics.mean(t_runs)
    steps = rollouts * T
    value = world * n * steps / (t_ms * 1e-3)
    vals = [world * n * steps / (t * 1e-3) for t in t_runs]

    # dominant tensor-core kernel: policy_fwd on the env's observation rows,
    # CUDA events on the launching stream
    obs = env._result().observations
    mean = torch.empty(n, env.action_dim, device=dev)
    val = torch.empty(n, device=dev)
    fwd_s = policy_fwd_seconds(pol, obs, mean, val, dev)
    try:
        peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops"])
        pk = "measured burst"
    except Exception:
        peak, pk = 1590.0, "fallback"
    achieved = n * POLICY_FLOPS_PER_ENV / fwd_s / 1e12

    # e2e: the same rollout through the public per-call API (3 C-ABI calls per
    # step: policy forward, sample, env step) with the step's result read back
    # to pinned host memory every step (observations, rewards, flags: what the
    # reference's host trainer loop consumes), synchronised per step
    e2e = None
    E = min(args.e2e_steps or steps, 2000)
    if E > 0:
        h_obs = torch.empty((n, env.obs_dim), dtype=torch.float32).pin_memory()
        h_rew = torch.empty(n, dtype=torch.float32).pin_memory()
        h_flags = torch.empty((2, n), dtype=torch.uint8).pin_memory()
        acts = torch.empty(n, env.action_dim, device=dev)
        logp = torch.empty(n, device=dev)
        L = sg.lib()
        st = torch.cuda.current_stream().cuda_stream
        d_pos = torch.zeros(1, dtype=torch.int64, device=dev)
        ls = tr.log_std_c
        o = env._result().observations

        def host_step(o):
            # one fused tensor-core launch: forward + Gaussian sampling + log-prob
            sg._pcheck(L.sg_policy_act(pol._h, o.data_ptr(), n, o.stride(0), ls.data_ptr(), tr.stream_state,
                                       tr.stream_inc, d_pos.data_ptr(), 0, acts.data_ptr(), logp.data_ptr(), None,
                                       val.data_ptr(), st))
            r = env.step(acts)
            h_obs.copy_(r.observations, non_blocking=True)
            h_rew.copy_(r.rewards, non_blocking=True)
            h_flags[0].copy_(r.terminated, non_blocking=True)
            h_flags[1].copy_(r.timed_out, non_blocking=True)
            torch.cuda.current_stream().synchronize()
            return r.observations

        o = host_step(o)
        if dist:
            dist.barrier()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record()
        for _ in range(E):
            o = host_step(o)
        a1.record()
        torch.cuda.synchronize()
        e_ms = max_over_ranks(a0.elapsed_time(a1), dist, dev)
        e2e = dict(value=world * n * E / (e_ms * 1e-3), unit="env-steps/s", h2d_bytes_per_step=0,
                   d2h_bytes_per_step=n * (env.obs_dim * 4 + 4 + 2), steps=E,
                   path="sg_policy_act (forward + sampling, one launch) + sg_env_step per step, observations / "
                        "rewards / flags copied to pinned host buffers and synchronised every step (no host inputs: "
                        "the actions are the policy's)")

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rate, lanes, sample = cpu_policy_reference(cfg, 10_000, budget_s=args.cpu_budget)
        cpu = dict(value=rate, unit="env-steps/s", cores=lanes, kind="port", sample=sample)
    if rank == 0:
        line = dict(
            metric=METRIC, value=value, unit="env-steps/s (random-init policy rollout)", n_gpus=world, steps=steps,
            warmup=args.warmup, ms_per_step=t_ms / steps, higher_is_better=True, scaling="weak", vs_baseline=None,
            dtype="bf16 policy fwd / fp32 env", data="synthetic",
            config=dict(workload=cfg["workload"], n_envs_per_gpu=n, global_envs=world * n, rollouts=rollouts,
                        rollout_steps=T, parallelism=f"env-shard x{world}",
                        l2="256 MiB flush before every timed rollout"),
            runs=dict(n=runs, value_mean=statistics.mean(vals), value_std=statistics.pstdev(vals),
                      gate_held=[r["gate_held"] for r in res]),
            roofline=dict(bound="tensor", achieved=achieved, peak=peak, unit="TFLOP/s", frac=achieved / peak,
                          traffic=None, peak_kind=pk, kernel="policy_fwd_kernel (tcgen05)",
                          flops_per_env=POLICY_FLOPS_PER_ENV, avg_launch_us=fwd_s * 1e6),
            cpu_baseline=cpu, e2e=e2e,
            # per rollout step: one policy launch (act; + the previous step's bootstrap from step 1 on)
            # and one env step; per rollout: the last step's bootstrap and the last-value forward
            gpu_launches=runs * rollouts * (2 * T + 2),
            clocks=clk.summary(),
        )
        print(json.dumps(line), flush=True)


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
    # e2e: the public call a training loop makes, Trainer.iterate(): rollout,
    # GAE, update, then one synchronisation that reads the iteration's
    # statistics and metrics back to the host (and checks the device error
    # word and the non-finite flag); no host inputs (actions are the policy's)
    e2e_iters = max(2, iters // 2)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a0.record()
    for _ in range(e2e_iters):
        tr.iterate()
    a1.record()
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(a0.elapsed_time(a1), dist, f"cuda:{local}")
    e2e_val = world * n * tcfg.n_steps * e2e_iters / (e2e_ms * 1e-3)
    # bytes iterate() reads back: stats (4 x f64), metrics (5 x f32), the
    # non-finite flag and the log-std mean (f32 each)
    d2h_iter = 4 * 8 + 5 * 4 + 4 + 4
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rate, lanes, sample = cpu_ppo_reference(cfg, budget_s=args.cpu_budget)
        cpu = dict(value=rate, unit="env-steps/s (with learning)", cores=lanes, kind="port", sample=sample)
    upd_ms = sum(e[2].elapsed_time(e[3]) for e in ev) / iters
    t_ms = max_over_ranks(t_ms, dist, f"cuda:{local}")
    steps = iters * tcfg.n_steps
    value = world * n * steps / (t_ms * 1e-3)
    # dominant tensor-core kernel: policy forward on the env's observation rows
    obs = env._result().observations
    mean = torch.empty(n, env.action_dim, device=f"cuda:{local}")
    val = torch.empty(n, device=f"cuda:{local}")
    fwd_s = policy_fwd_seconds(pol, obs, mean, val, f"cuda:{local}")
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
            cpu_baseline=cpu,
            e2e=dict(value=e2e_val, unit="env-steps/s (with learning)", h2d_bytes_per_step=0,
                     d2h_bytes_per_step=d2h_iter / tcfg.n_steps, iterations=e2e_iters,
                     path="Trainer.iterate() per iteration (rollout + GAE + update + one synchronisation "
                          f"reading {d2h_iter} B of statistics / metrics); a step = one rollout step of N envs"),
            # ours per iteration: rollout (policy fwd, sample, env step, bootstrap per step + last fwd), GAE,
            # per minibatch gather + 6 ELU fwd + 6 ELU bwd + loss (2) + Adam (2), policy repack
            gpu_launches=iters * (4 * tcfg.n_steps + 1 + 1 + tcfg.epochs * tcfg.minibatch_count * 17 + 1),
            clocks=clk.summary(),
        )
        print(json.dumps(line), flush=True)


def contract_bytes(A: int, O: int, tools: int = 1, step_read: int = 0) -> int:
    """SURVEY.md 8(d) algorithmic bytes per env-step (the fp32 SoA per-call step
    contract): read actions 4A + q, qdot 8A + goal 12 per tool + counters 16;
    write q, qdot, q_target 12A + observation row 4O + reward, task_error 8 +
    two flags 2. PSM 314 B, ECM 278 B, STAR 350 B. `step_read`: per-step task
    inputs beyond that (the ImageMatching target image)."""
    return 24 * A + 4 * O + 12 * tools + 26 + step_read


def spawn_ranks(args) -> int:
    """`bench.py --gpus N` outside torchrun: launch N ranks on this node the
    way the driver does (torch.distributed.run, 127.0.0.1 rendezvous, NCCL
    comm-init logging on) and return their exit code."""
    import socket
    import subprocess
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.run(cmd, env=env).returncode


def init_dist(world: int, local: int, backend: str | None = None):
    if world <= 1:
        return None
    import torch
    import torch.distributed as dist
    if backend is None:
        backend = "nccl" if torch.cuda.is_available() else "gloo"
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    else:
        dist.init_process_group("gloo")
    return dist


def dry_run(args, cfg, rank, world, local) -> None:
    """The N-rank plumbing without a GPU (CPU tests): process group, shard
    plan, gathered plans and the max-over-ranks reduction of a per-rank time."""
    dist = init_dist(world, local, backend="gloo")
    plan = shard_plan(rank, world, cfg["n_envs"])
    plans = [plan]
    if dist:
        plans = [None] * world
        dist.all_gather_object(plans, plan)
    t = max_over_ranks(1.0 + rank, dist, "cpu")
    if rank == 0:
        print(json.dumps(dict(dry_run=True, n_gpus=world, plans=plans, max_time=t, backend="gloo" if dist else None)),
              flush=True)
    if dist:
        dist.destroy_process_group()


def gate_cycles(n_launches: int, us_per_launch: float = 200.0) -> int:
    """Length of the device-side gate: long enough for the host to enqueue every
    flush / event / launch of one timed run behind it (generous: 200 us per
    launch on top of 10 ms; a whole rollout graph replay gets more), and long
    enough for the SM clocks to be up when the first timed launch starts."""
    return int((10000 + us_per_launch * n_launches) * 1e-6 * 2.0e9)


def timed_runs(env, launches, flush, runs: int, gate: bool, dist, device, retries: int = 3, do_flush: bool = True,
               gate_us: float = 200.0):
    """`runs` independent timed runs of the same launch sequence. Each run is
    bracketed by barrier + synchronize; every launch is preceded by an L2
    flush (256 MiB write) and timed by CUDA events on the env's stream (the
    current stream). With `gate`, a spin kernel (torch.cuda._sleep) heads the
    run so the host has enqueued the whole sequence before the GPU reaches the
    first event: the events then see only device time, never host-enqueue
    latency (with one launch per run there is nothing else to hide it). An
    untimed rehearsal of one gated launch first loads every kernel module the
    run uses (lazy loading) and creates the events. A run whose gate had
    already opened when the host finished enqueueing is repeated (up to
    `retries` times; the flag is reported). Returns per run: summed launch ms
    (max over ranks), per-launch ms, and whether the gate held."""
    import torch
    if gate:  # rehearsal (untimed): spin kernel, flush, events, one launch
        torch.cuda._sleep(gate_cycles(0) // 10)
        flush.zero_()
        r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        r0.record()
        env.bench_step(launches[0])
        r1.record()
        torch.cuda.synchronize()
    out = []
    for _ in range(runs):
        for attempt in range(retries + 1):
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in launches]
            if dist:
                dist.barrier()
            torch.cuda.synchronize()
            g = None
            if gate:
                torch.cuda._sleep(gate_cycles(len(launches), gate_us))
                g = torch.cuda.Event()
                g.record()
            for (e0, e1), kf in zip(ev, launches):
                if do_flush:
                    flush.zero_()
                e0.record()
                env.bench_step(kf)
                e1.record()
            held = (not g.query()) if g is not None else None
            torch.cuda.synchronize()
            ok = held is not False
            if dist:  # every rank repeats together
                t = torch.tensor([0.0 if ok else 1.0], device=device)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                ok = t.item() == 0.0
            if ok or attempt == retries:
                break
        ms = [e0.elapsed_time(e1) for e0, e1 in ev]
        t = max_over_ranks(sum(ms), dist, device)
        if dist:
            dist.barrier()
        out.append(dict(t_ms=t, launch_ms=ms, gate_held=held, attempts=attempt + 1))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None, help="timed env steps per run (default 25000; policy: 6400; ppo: 320)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="psm", choices=sorted(CONFIGS))
    ap.add_argument("--fuse", type=int, default=250, help="steps per fused launch")
    ap.add_argument("--runs", type=int, default=5, help="independent timed runs of --steps steps (mean +- std)")
    ap.add_argument("--no-gate", action="store_true",
                    help="enqueue the timed launches without the device-side gate (round-1 protocol; "
                         "host-enqueue latency lands inside the events)")
    ap.add_argument("--e2e-steps", type=int, default=None, help="host-API steps (default: --steps, <= 4000)")
    ap.add_argument("--no-flush", action="store_true", help="experiments only: keep L2 warm between launches")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dry-run", action="store_true", help="rank plumbing only (CPU, gloo)")
    ap.add_argument("--envs", type=int, default=None,
                    help="override envs per GPU (scaling studies; the headline uses the BASELINE config)")
    ap.add_argument("--update-precision", default="bf16", choices=["fp32", "tf32", "bf16"])
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config])
    if args.envs:
        cfg["n_envs"] = args.envs
        cfg["workload"] += f" [override: {args.envs} envs/GPU]"
    if args.steps is None:
        # default run lengths keep every launch of a run behind the device gate
        # (the command queue holds ~1000 entries: 100 fused launches or 200
        # rollouts with their flushes and events; longer runs stall the host
        # mid-run and let host latency into the timed intervals)
        args.steps = {"ppo": 320, "policy": 6400}.get(args.config, 25000)

    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(spawn_ranks(args))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")

    if args.dry_run:
        dry_run(args, cfg, rank, world, local)
        return

    if args.impl == "reference":
        if rank != 0:
            return
        total = max(args.steps, 3)
        if args.config == "policy":
            rate, lanes, sample = cpu_policy_reference(cfg, total, budget_s=120.0)
        elif args.config == "ppo":
            rate, lanes, sample = cpu_ppo_reference(cfg, budget_s=60.0)
        else:
            rate, lanes, sample = cpu_reference(cfg, total, budget_s=120.0)
        line = dict(metric=METRIC, value=rate, unit="env-steps/s", n_gpus=args.gpus, steps=args.steps,
                    warmup=args.warmup, ms_per_step=1e3 * cfg["n_envs"] / rate, higher_is_better=True,
                    scaling="weak", vs_baseline=None, dtype="f64", data="synthetic", impl="reference",
                    config=dict(workload=cfg["workload"], n_envs_per_gpu=cfg["n_envs"]),
                    cpu_baseline=dict(value=rate, unit="env-steps/s", cores=lanes, kind="port", sample=sample),
                    e2e=dict(value=rate, unit="env-steps/s", h2d_bytes_per_step=0, d2h_bytes_per_step=0))
        print(json.dumps(line), flush=True)
        return

    import torch
    torch.cuda.set_device(local)
    dist = init_dist(world, local, backend="nccl")
    try:
        if args.config == "ppo":
            bench_ppo(args, cfg, rank, world, local, dist)
        elif args.config == "policy":
            bench_policy(args, cfg, rank, world, local, dist)
        else:
            bench_env(args, cfg, rank, world, local, dist)
    finally:
        if dist:
            dist.destroy_process_group()


def load_profile_counters(config: str, fused: int) -> dict:
    """ncu numbers of the dominant kernel at THIS run's fused-step count
    (profiles/r2/traffic_<config>_k<F>.json, written by tools/profile_r2.sh
    from one `ncu --set full` capture): DRAM and L2 bytes per launch and the
    issue-slot utilisation."""
    p = os.path.join(ROOT, "profiles", "r2", f"traffic_{config}_k{fused}.json")
    if not os.path.exists(p):
        return {}
    try:
        return json.load(open(p))
    except Exception:
        return {}


def bench_env(args, cfg, rank, world, local, dist):
    import torch
    from paper_2310_04676_b200 import sg

    n = cfg["n_envs"]
    dev = f"cuda:{local}"
    plan = shard_plan(rank, world, n)
    robots = cfg.get("robots", (cfg.get("robot"),))
    env = sg.VecTaskEnv(robots=robots, device=local, n_envs=n, seed=0, task=cfg["task"],
                        goal_sigma=cfg["goal_sigma"], row_offset=plan["row_offset"])
    A, O = env.action_dim, env.obs_dim
    env.reset()
    env.bench_begin(0, first_step=0, global_n_envs=plan["global_n_envs"])
    F = max(1, min(args.fuse, args.steps))
    # warm-up: W untimed steps (the first is bench_sim's warm-up step), plus one
    # untimed fused launch so the timed launches see a warm instruction cache
    torch.cuda.nvtx.range_push("warmup")
    for _ in range(max(args.warmup, 1)):
        env.bench_step(1)
    env.bench_step(F)
    torch.cuda.nvtx.range_pop()
    steps_done = max(args.warmup, 1) + F
    torch.cuda.synchronize()

    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MiB > L2
    launches = []
    k = args.steps
    while k > 0:
        launches.append(min(F, k))
        k -= launches[-1]
    runs = max(1, args.runs)
    with Clocks(local) as clk:
        torch.cuda.nvtx.range_push("timed")
        res = timed_runs(env, launches, flush, runs, not args.no_gate, dist, dev, do_flush=not args.no_flush)
        torch.cuda.nvtx.range_pop()
    env.synchronize()
    steps_done += runs * args.steps
    t_runs = [r["t_ms"] for r in res]
    t_ms = statistics.mean(t_runs)
    value = world * n * args.steps / (t_ms * 1e-3)
    vals = [world * n * args.steps / (t * 1e-3) for t in t_runs]

    # ---- roofline of the dominant kernel (SURVEY 8(d) per-call contract bytes)
    wh = (O - 3 * A - 3) // 2 if cfg["task"] == "image_matching" else 0
    cb = contract_bytes(A, O, tools=len(robots), step_read=4 * wh)
    full = [ms for r in res for ms, kf in zip(r["launch_ms"], launches) if kf == F]
    avg_launch_s = (sum(full) / len(full)) * 1e-3
    peak, peak_kind = peaks()
    achieved = n * F * cb / avg_launch_s / 1e9
    # the same launch with state read / written once per launch (fused amortised bytes)
    resets = (steps_done // 300) - ((steps_done - runs * args.steps) // 300)
    b = step_bytes(A, O, F, resets / max(runs * args.steps, 1), tools=len(robots), step_read=4 * wh)
    prof = load_profile_counters(args.config, F)

    # ---- e2e through the host C-ABI call (pinned host buffers) --------------
    E = min(args.e2e_steps or args.steps, 4000)
    e2e = bench_e2e(env, E, n, A, O, dist, dev, world, torch, sg) if E > 0 else None

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
        # protocol on one pool lane and at config 1's 64 envs
        rate1, _, sample1 = cpu_reference(cfg, 10_000, budget_s=min(5.0, args.cpu_budget), threads=1)
        cpu.update(hardware_threads=os.cpu_count(), value_1_lane=rate1, sample_1_lane=sample1)
        rate64, l64, sample64 = cpu_reference(dict(cfg, n_envs=64), 100_000, budget_s=min(3.0, args.cpu_budget))
        cpu.update(value_64_envs=rate64, sample_64_envs=sample64)

    kname = (f"mt_step_kernel<T={len(robots)}, GEN>" if len(robots) > 1 else
             f"im_step_kernel<{cfg['robot'].upper()} chain, GEN>" if wh else
             f"env_step_kernel<{cfg['robot'].upper()} chain, 2 team warps, GEN>")
    if rank == 0:
        roof = dict(bound="hbm", achieved=achieved, peak=peak, unit="GB/s", frac=achieved / peak,
                    traffic=prof.get("dram_bytes_per_launch"), peak_kind=peak_kind,
                    kernel=f"{kname} ({F} fused steps/launch)", bytes_per_env_step=cb,
                    bytes_per_env_step_source="SURVEY.md 8(d) per-call step contract (24A + 4O + 12 + 26)",
                    bytes_per_launch=n * F * cb, avg_launch_us=avg_launch_s * 1e6,
                    fused_amortised=dict(bytes_per_env_step=b["per_env_step"],
                                         frac=n * b["per_env_launch"] / avg_launch_s / 1e9 / peak,
                                         note="state read/written once per fused launch"),
                    l2_bytes_per_launch=prof.get("lts_bytes_per_launch"),
                    issue_active_pct=prof.get("issue_active_pct"),
                    profile=prof.get("source"))
        line = dict(
            metric=METRIC, value=value, unit="env-steps/s", n_gpus=world, steps=args.steps, warmup=args.warmup,
            ms_per_step=t_ms / args.steps, higher_is_better=True, scaling="weak", vs_baseline=None,
            dtype="fp32", data="synthetic",
            config=dict(workload=cfg["workload"], n_envs_per_gpu=n, global_envs=world * n,
                        fused_steps_per_launch=F, parallelism=f"env-shard x{world}",
                        l2=("256 MiB flush before every timed launch; per-launch state read cold from HBM"
                            if not args.no_flush else "NOT flushed (experiment)"),
                        timing=("device-gated: a spin kernel heads each run so every launch is enqueued "
                                "before the GPU reaches it" if not args.no_gate else "host-enqueued (no gate)")),
            runs=dict(n=runs, value_mean=statistics.mean(vals), value_std=statistics.pstdev(vals),
                      ms_per_step_mean=t_ms / args.steps,
                      ms_per_step_std=statistics.pstdev([t / args.steps for t in t_runs]),
                      gate_held=[r["gate_held"] for r in res], attempts=[r["attempts"] for r in res],
                      ms_per_run=[r["t_ms"] for r in res]),
            roofline=roof, cpu_baseline=cpu, e2e=e2e, single_step_launches=single,
            gpu_launches=runs * len(launches) * (2 if cfg["task"] == "path_following" and F > 1 else 1),
            clocks=clk.summary(),
        )
        print(json.dumps(line), flush=True)


def bench_e2e(env, E, n, A, O, dist, dev, world, torch, sg):
    """`E` steps through the host C-ABI call sg_env_step_host: per step the
    action rows come from pinned host memory and the full StepResult goes back
    to pinned host buffers (terminal rows on steps where envs ended). Actions
    are the bench stream, pre-generated into a ring of up to 300 steps."""
    ring = min(E + 1, 300)
    # host buffers from the library's pinned allocator (sg_host_alloc)
    keep = [sg.HostBuffer((ring, n, A), torch.float32)]
    h_act = keep[0].tensor
    for s in range(ring):  # pre-generate the bench stream (device generator), outside timing
        env.bench_step(1)
        h_act[s].copy_(env.bench_actions())
    spec = (("observations", (n, O), torch.float32), ("terminal_observations", (n, O), torch.float32),
            ("rewards", (n,), torch.float32), ("task_error", (n,), torch.float32),
            ("terminated", (n,), torch.uint8), ("timed_out", (n,), torch.uint8))
    keep += [sg.HostBuffer(shape, dt) for _, shape, dt in spec]
    outs = {k2: buf.tensor for (k2, _, _), buf in zip(spec, keep[1:])}
    hr = sg.HostResult()
    for k2, t in outs.items():
        setattr(hr, k2, t.data_ptr())
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.nvtx.range_push("e2e")
    env.step_host_ptr(h_act[0].data_ptr(), hr)  # untimed first host step
    ended0 = env.host_counters()[0]
    e0.record()
    for s in range(E):
        env.step_host_ptr(h_act[(s + 1) % ring].data_ptr(), hr)
    e1.record()
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1), dist, dev)
    burst_steps = -(-(env.host_counters()[0] - ended0) // n)
    tobs_b = outs["terminal_observations"].numel() * 4
    d2h = sum(t.numel() * t.element_size() for k2, t in outs.items() if k2 != "terminal_observations") + 16
    d2h += tobs_b * burst_steps / max(E, 1)
    return dict(value=world * n * E / (e2e_ms * 1e-3), unit="env-steps/s", h2d_bytes_per_step=n * A * 4,
                d2h_bytes_per_step=d2h, steps=E, reset_burst_steps=burst_steps,
                path="sg_env_step_host (C-ABI), 1 launch + 1 synchronisation per step; terminal observations "
                     "copied on steps where rows ended")


if __name__ == "__main__":
    main()
