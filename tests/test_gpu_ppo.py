"""GPU: rollout sampling on the reference trainer stream, the GAE kernel, and
a short on-device PPO run (config 5 path: tcgen05 policy -> env step ->
GAE -> update)."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from tests.test_ppo_cpu import _gae_reference  # noqa: E402


def test_sample_kernel_uses_reference_stream(sg, oracle):
    from paper_2310_04676_b200 import ppo
    n, A, seed = 300, 7, 4
    L = sg.lib()
    s0, inc = ppo.make_stream(seed, ppo.TRAIN_STREAM)
    mean = torch.zeros(n, A, device="cuda")
    log_std = torch.tensor([0.0, 0.0, 0.0, 0.0, -7.0, 3.0, -1.0], device="cuda")  # two clamped
    act = torch.empty(n, A, device="cuda")
    logp = torch.empty(n, device="cuda")
    skip = 2 * n * A * 3 + 999  # three earlier rollout steps + an update's draws
    pos = torch.tensor([skip], dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    sg._pcheck(L.sg_policy_sample(mean.data_ptr(), n, A, log_std.data_ptr(), s0, inc, pos.data_ptr(), 2 * n * A,
                                  act.data_ptr(), logp.data_ptr(), st))
    torch.cuda.synchronize()
    r = oracle.make_stream(seed, ppo.TRAIN_STREAM)
    for _ in range(skip + 2 * n * A):
        oracle.next_u32(r)
    ls = np.clip(log_std.cpu().numpy().astype(np.float64), -5, 2)
    ref_a = np.zeros((n, A)); ref_lp = np.zeros(n)
    for e in range(n):
        for i in range(A):
            z = oracle.normal(r)
            ref_a[e, i] = np.exp(ls[i]) * z
            ref_lp[e] += -0.5 * z * z - ls[i] - 0.9189385332046727
    np.testing.assert_allclose(act.cpu().numpy(), ref_a, rtol=2e-7, atol=1e-30)
    np.testing.assert_allclose(logp.cpu().numpy(), ref_lp, rtol=1e-6)


def test_gae_kernel_matches_reference(sg):
    rng = np.random.default_rng(7)
    T, n = 32, 2000
    rew = rng.normal(size=(T, n)).astype(np.float32)
    val = rng.normal(size=(T, n)).astype(np.float32)
    term = (rng.random((T, n)) < 0.02).astype(np.uint8)
    tout = ((rng.random((T, n)) < 0.03) & (term == 0)).astype(np.uint8)
    boot = (rng.normal(size=(T, n)) * tout).astype(np.float32)
    last = rng.normal(size=n).astype(np.float32)
    terr = rng.random((T, n)).astype(np.float32)
    d = lambda x: torch.from_numpy(x).cuda()
    adv = torch.empty(T, n, device="cuda"); ret = torch.empty(T, n, device="cuda")
    ep_acc = torch.zeros(n, device="cuda"); stats = torch.zeros(4, dtype=torch.float64, device="cuda")
    args = [d(rew), d(val), d(term), d(tout), d(boot), d(last), d(terr)]
    sg._pcheck(sg.lib().sg_compute_gae(*[a.data_ptr() for a in args], T, n, 0.99, 0.95, adv.data_ptr(),
                                       ret.data_ptr(), ep_acc.data_ptr(), stats.data_ptr(),
                                       torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    ra, rr = _gae_reference(rew.astype(np.float64), val.astype(np.float64), term, tout, boot.astype(np.float64),
                            last.astype(np.float64), 0.99, 0.95)
    np.testing.assert_allclose(adv.cpu().numpy(), ra, rtol=1e-4, atol=1e-4)
    np.testing.assert_allclose(ret.cpu().numpy(), rr, rtol=1e-4, atol=1e-4)
    ends = (term | tout).astype(bool)
    assert stats[3].item() == ends.sum()
    assert abs(stats[0].item() - rew.astype(np.float64).sum()) < 1e-2


def test_ppo_trainer_runs_and_learns_signal(sg):
    from paper_2310_04676_b200 import ppo
    env = sg.VecTaskEnv(robots=("psm",), n_envs=4096, seed=0, episode_len=60)
    pol = sg.Policy(env.obs_dim, env.action_dim)
    tr = ppo.Trainer(env, pol, ppo.TrainConfig(seed=0, n_steps=32))
    hist = [tr.iterate() for _ in range(4)]
    for h in hist:
        for k in ("policy_loss", "value_loss", "kl", "mean_step_reward"):
            assert math.isfinite(h[k]), (k, h)
    assert hist[-1]["env_steps"] == 4 * 32 * 4096
    assert hist[-1]["episodes_completed"] > 0  # episode_len 60 -> timeouts inside the run
    assert -5.0 <= hist[-1]["log_std_mean"] <= 2.0
    # the critic fits returns: value loss falls from the first to the last iteration
    assert hist[-1]["value_loss"] < hist[0]["value_loss"]


def test_fused_adam_step_matches_reference_formulas(sg):
    """sg_adam_step == ppo.cpp:199-207 (clip to max_grad_norm when the norm
    exceeds it) + Adam::step (ppo.cpp:56-64) + log-std projection, restated in
    fp64 numpy, over steps with gradients above and below the clip norm;
    the gradient is zeroed and the bf16 mirror refreshed."""
    rng = np.random.default_rng(3)
    n, ls_off, ls_n = 5000, 4990, 7
    p = rng.normal(size=n)
    p[ls_off: ls_off + ls_n] = [-4.9, 1.95, 0.0, -1.0, 1.99, -4.99, 0.5]
    m = np.zeros(n); v = np.zeros(n)
    P = torch.tensor(p, dtype=torch.float32, device="cuda")
    G = torch.zeros(n, device="cuda")
    M, V = torch.zeros(n, device="cuda"), torch.zeros(n, device="cuda")
    mirror = torch.zeros(n, dtype=torch.bfloat16, device="cuda")
    t = torch.zeros(1, dtype=torch.int32, device="cuda")
    gsq = torch.zeros(2, device="cuda")
    lr, b1, b2, eps, max_norm = 1e-2, 0.9, 0.999, 1e-8, 1.0
    for step, gscale in enumerate((0.001, 1.0, 0.003, 5.0), start=1):
        g = rng.normal(size=n) * gscale
        G.copy_(torch.tensor(g, dtype=torch.float32))
        sg._pcheck(sg.lib().sg_adam_step(P.data_ptr(), G.data_ptr(), M.data_ptr(), V.data_ptr(), mirror.data_ptr(),
                                         n, gsq.data_ptr(), t.data_ptr(), lr, b1, b2, eps, max_norm, ls_off, ls_n,
                                         -5.0, 2.0, torch.cuda.current_stream().cuda_stream))
        torch.cuda.synchronize()
        g = g.astype(np.float32).astype(np.float64)
        norm = np.linalg.norm(g)
        if norm > max_norm:
            g *= max_norm / norm
        m = b1 * m + (1 - b1) * g
        v = b2 * v + (1 - b2) * g * g
        p = p - lr * (m / (1 - b1 ** step)) / (np.sqrt(v / (1 - b2 ** step)) + eps)
        p[ls_off: ls_off + ls_n] = np.clip(p[ls_off: ls_off + ls_n], -5.0, 2.0)
        assert t.item() == step
        np.testing.assert_allclose(P.cpu().numpy(), p, rtol=2e-5, atol=2e-6)
        assert not G.any()
        assert torch.equal(mirror, P.to(torch.bfloat16))
        p = P.cpu().numpy().astype(np.float64)  # continue from the device's fp32 state
        m = M.cpu().numpy().astype(np.float64)
        v = V.cpu().numpy().astype(np.float64)
    assert gsq[1].item() == 0.0
    # a non-finite gradient (ppo.cpp:193-199 throws): parameters and moments
    # untouched, gradient cleared, sticky flag raised
    before = [x.clone() for x in (P, M, V)]
    G.copy_(torch.tensor(rng.normal(size=n), dtype=torch.float32))
    G[17] = float("nan")
    sg._pcheck(sg.lib().sg_adam_step(P.data_ptr(), G.data_ptr(), M.data_ptr(), V.data_ptr(), mirror.data_ptr(),
                                     n, gsq.data_ptr(), t.data_ptr(), lr, b1, b2, eps, max_norm, ls_off, ls_n,
                                     -5.0, 2.0, torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    assert gsq[1].item() == 1.0
    for a, b in zip((P, M, V), before):
        assert torch.equal(a, b)
    assert not G.any()


def test_ppo_trainer_bf16_update_runs(sg):
    """The bench's update precision: bf16 GEMMs on the fused-Adam bf16 mirror,
    captured in a CUDA graph."""
    from paper_2310_04676_b200 import ppo
    env = sg.VecTaskEnv(robots=("psm",), n_envs=4096, seed=0, episode_len=60)
    pol = sg.Policy(env.obs_dim, env.action_dim)
    tr = ppo.Trainer(env, pol, ppo.TrainConfig(seed=0, n_steps=32, update_precision="bf16"))
    hist = [tr.iterate() for _ in range(4)]
    for h in hist:
        for k in ("policy_loss", "value_loss", "kl", "mean_step_reward"):
            assert math.isfinite(h[k]), (k, h)
    assert torch.equal(tr.mirror, tr.params.to(torch.bfloat16))
    assert hist[-1]["value_loss"] < hist[0]["value_loss"]


def test_trainer_checkpoint_round_trip(sg, tmp_path):
    """Trainer.save_checkpoint writes the reference format; a second trainer
    loading it has the same reference-layout parameters and policy outputs."""
    from paper_2310_04676_b200 import ppo
    env = sg.VecTaskEnv(robots=("psm",), n_envs=1024, seed=1)
    a = ppo.Trainer(env, sg.Policy(env.obs_dim, env.action_dim), ppo.TrainConfig(seed=3))
    a.iterate()
    path = str(tmp_path / "psm.ckpt")
    a.save_checkpoint(path, "psm")
    env2 = sg.VecTaskEnv(robots=("psm",), n_envs=1024, seed=1)
    pol2 = sg.Policy(env2.obs_dim, env2.action_dim)
    b = ppo.Trainer(env2, pol2, ppo.TrainConfig(seed=9))
    meta = b.load_checkpoint(path)
    assert meta["robot"] == "psm" and meta["hidden"] == (256, 128, 64)
    assert torch.equal(a.ref_params(), b.ref_params())
    obs = env.reset()
    m1, v1 = torch.empty(1024, 7, device="cuda"), torch.empty(1024, device="cuda")
    m2, v2 = torch.empty_like(m1), torch.empty_like(v1)
    a.policy.forward(obs, m1, v1)
    pol2.forward(obs, m2, v2)
    torch.cuda.synchronize()
    assert torch.equal(m1, m2) and torch.equal(v1, v2)


def test_update_kernels_elu_and_gather(sg):
    """train.cu: device ELU forward / backward vs torch (fp32: within 2 ulp of
    expm1; bf16: one rounding of the fp32 result), and the fused minibatch
    gather vs index_select; the PPO loss gradients with the device ELU path
    equal the torch-ELU path."""
    from paper_2310_04676_b200 import ppo
    g = torch.Generator(device="cuda").manual_seed(0)
    z = torch.randn(4096, 64, device="cuda", generator=g) * 3
    h = sg.elu_forward(z)
    torch.testing.assert_close(h, torch.nn.functional.elu(z), rtol=3e-7, atol=1e-7)
    dh = torch.randn_like(z)
    zr = z.clone().requires_grad_(True)
    torch.nn.functional.elu(zr).backward(dh)
    torch.testing.assert_close(sg.elu_backward(h, dh), zr.grad, rtol=1e-6, atol=1e-6)
    zb = z.bfloat16()
    hb = sg.elu_forward(zb)
    torch.testing.assert_close(hb.float(), torch.nn.functional.elu(zb.float()).bfloat16().float(), rtol=8e-3,
                               atol=1e-6)
    assert sg.elu_forward(zb, out=zb) is zb  # in place
    # gather
    cap, O, A, m = 5000, 32, 7, 1200
    obs, act = torch.randn(cap, O, device="cuda"), torch.randn(cap, A, device="cuda")
    logp, adv, ret = (torch.randn(cap, device="cuda") for _ in range(3))
    idx = torch.randperm(cap, device="cuda")[:m]
    for dt in (torch.float32, torch.bfloat16):
        out = [torch.empty(m, O, device="cuda", dtype=dt), torch.empty(m, A, device="cuda")] + \
              [torch.empty(m, device="cuda") for _ in range(3)]
        sg.ppo_gather(idx, obs, act, logp, adv, ret, *out)
        assert torch.equal(out[0], obs[idx].to(dt)) and torch.equal(out[1], act[idx])
        for o, src in zip(out[2:], (logp, adv, ret)):
            assert torch.equal(o, src[idx])
    # unpadded rows (the env's obs_dim-wide rows) -> zero-padded bf16 / fp32 rows; A > 8
    for ow, A2 in ((27, 9), (30, 3)):
        obs2, act2 = torch.randn(cap, ow, device="cuda"), torch.randn(cap, A2, device="cuda")
        for dt in (torch.float32, torch.bfloat16):
            out = [torch.full((m, O), 5.0, device="cuda", dtype=dt), torch.empty(m, A2, device="cuda")] + \
                  [torch.empty(m, device="cuda") for _ in range(3)]
            sg.ppo_gather(idx, obs2, act2, logp, adv, ret, *out)
            ref = torch.zeros(m, O, device="cuda")
            ref[:, :ow] = obs2[idx]
            assert torch.equal(out[0], ref.to(dt)) and torch.equal(out[1], act2[idx])
            for o, src in zip(out[2:], (logp, adv, ret)):
                assert torch.equal(o, src[idx])
    # loss gradients: device-ELU layers == torch-ELU layers (fp32)
    torch.manual_seed(1)
    layout, ls_off, total, _ = ppo.padded_layout(27, 7)
    params = torch.randn(total, device="cuda") * 0.1
    x = torch.randn(512, 32, device="cuda")
    grads = []
    for dev_elu in (False, True):
        p = params.clone().requires_grad_(True)
        layers = [(p[w0: w0 + o * i].view(o, i), p[b0: b0 + ob]) for (w0, o, i), (b0, ob) in layout]
        mean, value = ppo.mlp_layers(layers, x, device_elu=dev_elu)
        (mean.square().sum() + value.sum()).backward()
        grads.append(p.grad.clone())
    torch.testing.assert_close(grads[1], grads[0], rtol=1e-4, atol=1e-5)  # h + 1 vs exp(z), GEMM order


def test_fused_ppo_loss_matches_reference_formulas(sg):
    """sg_ppo_loss (ppo.cpp:90-154 in one kernel) == the autograd loss head
    (tests/test_ppo_cpu.py pins that one to the reference's analytic
    gradients): loss, metrics, dmean, dvalue, dlog_std, with clipped ratios,
    both surrogate branches and a log-std outside the box."""
    from paper_2310_04676_b200 import ppo
    g = torch.Generator(device="cuda").manual_seed(5)
    B, A, P = 3000, 7, 8
    mean_full = torch.randn(B, P, device="cuda", generator=g) * 0.3
    value_full = torch.randn(B, P, device="cuda", generator=g)
    log_std = torch.tensor([-1.0, -0.5, 0.2, -6.0, 2.5, -1.2, 0.0], device="cuda")  # two outside [-5, 2]
    lsc = log_std.clamp(ppo.LOG_STD_MIN, ppo.LOG_STD_MAX)
    # actions drawn from the policy (as in a rollout): moderate log-probs
    act = mean_full[:, :A] + torch.exp(lsc) * torch.randn(B, A, device="cuda", generator=g)
    logp = (-0.5 * ((act - mean_full[:, :A]) * torch.exp(-lsc)) ** 2 - lsc - ppo.HALF_LOG_2PI).sum(1)
    old_logp = logp + 0.3 * torch.randn(B, device="cuda", generator=g)  # ratios around 1 +- 30 %
    adv = torch.randn(B, device="cuda", generator=g)
    ret = torch.randn(B, device="cuda", generator=g)
    cfg = ppo.TrainConfig(entropy_coef=0.01)
    m_ref = mean_full[:, :A].clone().requires_grad_(True)
    v_ref = value_full[:, 0].clone().requires_grad_(True)
    ls_ref = log_std.clone().requires_grad_(True)
    loss_ref, met_ref = ppo.loss_head(m_ref, v_ref, ls_ref, act, old_logp, adv, ret, cfg)
    loss_ref.backward()
    mf = mean_full.clone().requires_grad_(True)
    vf = value_full.clone().requires_grad_(True)
    ls = log_std.clone().requires_grad_(True)
    loss, met = ppo._PPOLossDevice.apply(mf, vf, ls, act, old_logp, adv, ret, A, cfg.clip_eps, cfg.value_coef,
                                         cfg.entropy_coef)
    loss.backward()
    assert 0.05 < float(met_ref[4]) < 0.95  # both surrogate branches present
    torch.testing.assert_close(loss, loss_ref, rtol=1e-4, atol=1e-5)
    # metrics: kl is a mean of near-cancelling terms, clip_fraction may flip a
    # sample whose ratio sits on the clip boundary (fp32 exp)
    torch.testing.assert_close(met, met_ref, rtol=1e-3, atol=1e-3)
    torch.testing.assert_close(mf.grad[:, :A], m_ref.grad, rtol=1e-4, atol=1e-8)
    assert (mf.grad[:, A:] == 0).all() and (vf.grad[:, 1:] == 0).all()
    torch.testing.assert_close(vf.grad[:, 0], v_ref.grad, rtol=1e-5, atol=1e-9)
    torch.testing.assert_close(ls.grad, ls_ref.grad, rtol=1e-4, atol=1e-6)
    assert ls.grad[3] == 0 and ls.grad[4] == 0


def test_update_graph_with_captured_nccl_allreduce(sg):
    """The multi-GPU update path on one GPU: a world-1 NCCL group with the
    gradient all-reduce forced on is captured inside the update's CUDA graph
    (ppo.cpp:201-204 all-reduce before clipping); all-reduce-mean over one
    rank is the identity, so the parameters match a trainer without any
    collective (to the run-to-run noise of the atomically reduced gradient
    norm)."""
    import socket
    import torch.distributed as dist
    from paper_2310_04676_b200 import ppo
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda:0"))
    try:
        res = []
        for use_dist in (False, True):
            env = sg.VecTaskEnv(robots=("psm",), n_envs=2048, seed=2, episode_len=40)
            tr = ppo.Trainer(env, sg.Policy(env.obs_dim, env.action_dim),
                             ppo.TrainConfig(seed=1, n_steps=32, update_precision="fp32"),
                             dist=dist if use_dist else None)
            tr.force_collectives = use_dist
            for _ in range(3):
                tr.iterate()
            assert tr.graph is not None  # the update ran as a graph replay
            res.append(tr.params.clone())
        torch.testing.assert_close(res[0], res[1], rtol=1e-2, atol=1e-3)
    finally:
        dist.destroy_process_group()


def test_trainer_raises_on_nonfinite_training(sg):
    """A diverged policy (non-finite parameters) is a SimError at the next
    iteration's synchronisation -- non-finite actions reach the env
    (dynamics.cpp:198-200) and the loss / gradient check (ppo.cpp:193-199) --
    instead of training on silently."""
    from paper_2310_04676_b200 import ppo
    env = sg.VecTaskEnv(robots=("psm",), n_envs=1024, seed=0)
    tr = ppo.Trainer(env, sg.Policy(env.obs_dim, env.action_dim), ppo.TrainConfig(seed=0))
    tr.iterate()
    with torch.no_grad():
        tr.params[5] = float("nan")
    tr.policy.load_params(tr.ref_params())
    with pytest.raises(sg.SimError):
        tr.iterate()


def test_shard_sampling_takes_its_rows_of_the_global_stream(sg):
    """ppo.cpp:264-270 draws each rollout step's noise from ONE stream over all
    global rows. A shard owning global rows [r*N, (r+1)*N) of world*N
    (Trainer: step_offset = 2A (t*world*N + row_offset)) gets exactly those
    rows' draws -- shards never share noise."""
    torch.manual_seed(0)
    world, N, A, t = 4, 300, 7, 3
    mean = torch.randn(world * N, A, device="cuda")
    pol = sg.Policy(27, A)
    full, lp_full = pol.sample(mean, seed=5, step_offset=2 * A * t * world * N)
    for r in range(world):
        part, lp = pol.sample(mean[r * N:(r + 1) * N].contiguous(), seed=5,
                              step_offset=2 * A * (t * world * N + r * N))
        assert torch.equal(part, full[r * N:(r + 1) * N])
        assert torch.equal(lp, lp_full[r * N:(r + 1) * N])
    assert not torch.equal(full[:N], full[N:2 * N])


def test_rollout_noise_ahead_equals_fused_sampling(sg):
    """The trainer's default rollout draws step t+1's noise on a side stream
    during env step t (sg_policy_noise + sg_policy_act_noise, CUDA-graphed
    with a fork/join per step); it must leave the rollout buffer bit-identical
    to the fused per-step sg_policy_act path, including across the graph
    replays of later rollouts and an episode boundary."""
    from paper_2310_04676_b200 import ppo
    bufs = []
    for ahead in (True, False):
        env = sg.VecTaskEnv(robots=("psm",), n_envs=2048, seed=1, episode_len=40)
        tr = ppo.Trainer(env, sg.Policy(env.obs_dim, env.action_dim), ppo.TrainConfig(seed=2, noise_ahead=ahead))
        out = []
        for _ in range(3):  # eager rollout, graph capture, graph replay
            tr.rollout()
            torch.cuda.synchronize()
            out.append({k: tr.buf[k].clone() for k in ("obs", "actions", "logp", "values", "rewards", "boot")})
        bufs.append(out)
    for a, b in zip(*bufs):
        for k in a:
            assert torch.equal(a[k], b[k]), k


def test_rollout_folded_bootstrap_equals_separate_launch(sg):
    """The default rollout computes step t-1's timeout bootstrap inside step
    t's policy launch (sg_policy_act_bootstrap); the rollout buffer --
    bootstrap values included, across timeouts and graph replays -- is
    bit-identical to a separate sg_policy_bootstrap launch per step."""
    from paper_2310_04676_b200 import ppo
    bufs = []
    for fold in (True, False):
        env = sg.VecTaskEnv(robots=("psm",), n_envs=2048, seed=3, episode_len=37)
        tr = ppo.Trainer(env, sg.Policy(env.obs_dim, env.action_dim), ppo.TrainConfig(seed=5, fold_bootstrap=fold))
        out = []
        for _ in range(3):  # eager rollout, graph capture, graph replay
            tr.rollout()
            torch.cuda.synchronize()
            out.append({k: tr.buf[k].clone() for k in ("obs", "actions", "logp", "values", "boot", "timed_out")})
        bufs.append(out)
    n_boot = sum(int((o["boot"] != 0).sum()) for o in bufs[0])
    assert n_boot > 0  # timeouts inside the rollouts exercised the folded path
    for a, b in zip(*bufs):
        for k in a:
            assert torch.equal(a[k], b[k]), k


@pytest.mark.parametrize("m,n", [(131072, 256), (1000, 128), (257, 64), (131072, 8)])
def test_elu_backward_colsum_matches_reference(sg, m, n):
    """sg_elu_backward_colsum: dz = dh * ELU'(h) (bit-identical to
    sg_elu_backward) and the fp32 column sums of dz accumulated into the
    bias gradient (what 1^T dZ gives, to fp32 summation-order noise); h = NULL
    gives the plain column sums of dh."""
    torch.manual_seed(3)
    h = torch.where(torch.rand(m, n, device="cuda") < 0.5, torch.rand(m, n, device="cuda"),
                    -torch.rand(m, n, device="cuda")).to(torch.bfloat16)
    dh = (torch.randn(m, n, device="cuda") * 0.3).to(torch.bfloat16)
    acc = torch.full((n,), 0.25, device="cuda")  # accumulates on top of what is there
    dz = sg.elu_backward_colsum(h, dh, acc)
    ref_dz = sg.elu_backward(h, dh)
    acc2 = torch.zeros(n, device="cuda")
    sg.elu_backward_colsum(None, dh, acc2, out=False)
    torch.cuda.synchronize()
    assert torch.equal(dz, ref_dz)
    ref = ref_dz.double().sum(0) + 0.25
    assert torch.allclose(acc.double(), ref, rtol=1e-4, atol=1e-3)
    assert torch.allclose(acc2.double(), dh.double().sum(0), rtol=1e-4, atol=1e-3)


@pytest.mark.parametrize("out_dim,in_dim,m", [(256, 32, 131072), (128, 256, 131072), (64, 128, 1000), (8, 64, 77)])
def test_wgrad_matches_reference(sg, out_dim, in_dim, m):
    """sg_policy_wgrad (dW = dY^T X over the minibatch rows on the tensor cores,
    MN-major UMMA operands streamed with cp.async, per-CTA partials + one sum)
    == the fp64 product of the same bf16 operands to fp32 accumulation noise,
    including a ragged row count and CTAs with empty slices."""
    torch.manual_seed(5)
    dy = (torch.randn(m, out_dim, device="cuda") * 0.3).to(torch.bfloat16)
    x = (torch.randn(m, in_dim, device="cuda") * 0.5).to(torch.bfloat16)
    partial = torch.empty(148 * 128 * 256, device="cuda")
    out = torch.full((out_dim, in_dim), 7.0, device="cuda")  # overwritten, not accumulated
    sg.wgrad(dy, x, partial, out)
    torch.cuda.synchronize()
    ref = dy.double().t() @ x.double()
    err = (out.double() - ref).abs().max().item()
    assert err <= 1e-3 * ref.abs().max().item() + 1e-4, err
