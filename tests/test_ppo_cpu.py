"""PPO host logic on CPU: the loss head's autograd gradients equal the
reference's analytic gradients (ppo.cpp:101-145), GAE restatement, the
trainer stream seeding, and the multi-rank reductions (gloo, world 2)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_2310_04676_b200 import ppo


def test_loss_head_gradients_match_reference_formulas():
    rng = np.random.default_rng(0)
    n, A = 64, 7
    cfg = ppo.TrainConfig()
    mean = rng.normal(size=(n, A))
    value = rng.normal(size=n)
    log_std = np.array([-1.0, -0.5, 0.3, -6.0, 2.5, 0.0, -2.0])  # two outside the clamp box
    actions = mean + rng.normal(size=(n, A)) * 0.5
    old_logp = rng.normal(size=n) - 5.0
    adv = rng.normal(size=n)
    ret = rng.normal(size=n)
    t = lambda x: torch.tensor(x, dtype=torch.float64, requires_grad=True)
    m_t, v_t, ls_t = t(mean), t(value), t(log_std)
    loss, _ = ppo.loss_head(m_t, v_t, ls_t, torch.tensor(actions), torch.tensor(old_logp), torch.tensor(adv),
                            torch.tensor(ret), cfg)
    loss.backward()
    # reference analytic gradients (ppo.cpp:90-145)
    ls = np.clip(log_std, -5.0, 2.0)
    inv_var = np.exp(-2 * ls)
    dmean = np.zeros((n, A)); dls = np.zeros(A); dval = np.zeros(n)
    for j in range(n):
        diff = actions[j] - mean[j]
        logp = (-0.5 * diff * diff * inv_var - ls - ppo.HALF_LOG_2PI).sum()
        ratio = np.exp(logp - old_logp[j])
        unc = ratio * adv[j]
        clo = np.clip(ratio, 1 - cfg.clip_eps, 1 + cfg.clip_eps) * adv[j]
        d = -(1.0 / n) * (unc if unc <= clo else 0.0)
        dmean[j] = d * diff * inv_var
        dls += d * (diff * diff * inv_var - 1.0)
        dval[j] = cfg.value_coef * (value[j] - ret[j]) / n
    dls -= cfg.entropy_coef
    dls[(log_std < -5.0) | (log_std > 2.0)] = 0.0
    # policy loss gradient wrt mean is -(1/n)*dsurr/dmean: the reference's dmean is d(loss)/d(mean) w/ sign folded
    np.testing.assert_allclose(m_t.grad.numpy(), dmean, rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(ls_t.grad.numpy(), dls, rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(v_t.grad.numpy(), dval, rtol=1e-9, atol=1e-12)


def _gae_reference(rew, val, term, tout, boot, last, gamma, lam):
    # rollout.cpp:42-66
    T, n = rew.shape
    adv = np.zeros((T, n)); ret = np.zeros((T, n))
    for e in range(n):
        running = 0.0
        for t in range(T - 1, -1, -1):
            if term[t, e]:
                delta = rew[t, e] - val[t, e]
            elif tout[t, e]:
                delta = rew[t, e] + gamma * boot[t, e] - val[t, e]
            else:
                vn = last[e] if t == T - 1 else val[t + 1, e]
                delta = rew[t, e] + gamma * vn - val[t, e]
            running = delta if (term[t, e] or tout[t, e]) else delta + gamma * lam * running
            adv[t, e] = running
            ret[t, e] = running + val[t, e]
    return adv, ret


def test_gae_reference_restatement_properties():
    """Sanity of the numpy restatement used by the GPU GAE test: with no
    episode ends, GAE(lambda=1, gamma=1) returns = reward-to-go + last value."""
    rng = np.random.default_rng(1)
    T, n = 8, 5
    rew, val, last = rng.normal(size=(T, n)), rng.normal(size=(T, n)), rng.normal(size=n)
    z = np.zeros((T, n), bool)
    adv, ret = _gae_reference(rew, val, z, z, np.zeros((T, n)), last, 1.0, 1.0)
    np.testing.assert_allclose(ret[0], rew.sum(0) + last, rtol=1e-12)


def test_trainer_stream_matches_oracle(oracle):
    for seed in (0, 3, 2024):
        s, inc = ppo.make_stream(seed, ppo.TRAIN_STREAM)
        r = oracle.make_stream(seed, ppo.TRAIN_STREAM)
        assert (s, inc) == (r.state, r.inc)


def _port():
    s = socket.socket(); s.bind(("127.0.0.1", 0)); p = s.getsockname()[1]; s.close(); return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = torch.full((5,), float(rank + 1))
    ppo.allreduce_mean_(g, dist)
    adv = torch.arange(4, dtype=torch.float32) + 10 * rank
    mean, std = ppo.global_adv_stats(adv, dist)
    if rank == 0:
        q.put((g.tolist(), float(mean), float(std)))
    dist.destroy_process_group()


def test_gradient_and_advantage_reductions_two_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    g, mean, std = q.get(timeout=120)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert g == [1.5] * 5
    allv = np.concatenate([np.arange(4), np.arange(4) + 10]).astype(np.float64)
    assert abs(mean - allv.mean()) < 1e-6 and abs(std - allv.std()) < 1e-5


def test_padded_training_layout_is_equivalent():
    """The padded training copy (odd widths rounded up to 8 for the GEMMs)
    computes the same MLP as the reference layout, and padded entries get
    zero gradient."""
    torch.manual_seed(0)
    O, A = 27, 7
    _, ls_ref = ppo.param_layout(O, A)
    flat = torch.randn(ls_ref + A, dtype=torch.float64)
    layout, ls_pad, total, r2p = ppo.padded_layout(O, A)
    r2p = torch.from_numpy(r2p)
    assert len(set(r2p.tolist())) == r2p.numel()
    pad = torch.zeros(total, dtype=torch.float64)
    pad[r2p] = flat
    obs = torch.randn(64, O, dtype=torch.float64)
    m_ref, v_ref, _ = ppo.mlp_forward(flat, obs, O, A)
    pad = pad.requires_grad_(True)
    layers = [(pad[w0: w0 + o * i].view(o, i), pad[b0: b0 + ob]) for (w0, o, i), (b0, ob) in layout]
    obs_p = torch.zeros(64, 32, dtype=torch.float64)
    obs_p[:, :O] = obs
    m_pad, v_pad = ppo.mlp_layers(layers, obs_p)
    assert torch.allclose(m_pad[:, :A], m_ref, atol=1e-12) and torch.allclose(v_pad, v_ref, atol=1e-12)
    (m_pad[:, :A].sum() + v_pad.sum()).backward()
    mask = torch.ones(total, dtype=torch.bool)
    mask[r2p] = False
    assert pad.grad[mask].abs().max().item() == 0.0
