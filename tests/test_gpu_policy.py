"""Tensor-core policy forward (tcgen05, BF16 in / FP32 accumulate) vs a plain
PyTorch fp32 reference of Policy::forward (proj/src/policy.cpp:110-161).

Two references: (a) bf16-emulating (inputs, weights and each hidden
activation rounded to bf16 exactly where the kernel rounds) — must agree to
fp32 accumulation-order noise; (b) the full-fp32 reference — agrees within
the stated bf16 tolerance."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _layers(flat, obs_dim, act_dim):
    dims = [obs_dim, 256, 128, 64]
    off = 0
    out = {}
    for trunk in (0, 1):
        o_last = act_dim if trunk == 0 else 1
        for l in range(4):
            i, o = dims[l], (dims[l + 1] if l < 3 else o_last)
            W = flat[off: off + o * i].reshape(o, i)
            off += o * i
            b = flat[off: off + o]
            off += o
            out[(trunk, l)] = (W, b)
    return out


def _ref_forward(flat, obs, act_dim, emulate_bf16):
    L = _layers(flat, obs.shape[1], act_dim)
    r = (lambda t: t.to(torch.bfloat16).float()) if emulate_bf16 else (lambda t: t)
    outs = []
    for trunk in (0, 1):
        h = r(obs)
        for l in range(4):
            W, b = L[(trunk, l)]
            z = h @ r(W).T + b
            h = r(torch.where(z > 0, z, torch.expm1(z))) if l < 3 else z
        outs.append(h)
    return outs[0], outs[1][:, 0]


@pytest.mark.parametrize("n,act_dim,obs_dim", [(16384, 7, 27), (1000, 6, 24), (130, 8, 30)])
def test_policy_forward_matches_torch(sg, n, act_dim, obs_dim):
    torch.manual_seed(0)
    pol = sg.Policy(obs_dim, act_dim)
    flat = pol.init_params(seed=3)
    flat = torch.from_numpy(flat).cuda()
    # non-zero biases and an un-shrunk last layer so every path is exercised
    flat = flat + 0.05 * torch.randn_like(flat)
    pol.load_params(flat)
    obs = torch.randn(n, obs_dim, device="cuda") * 0.5
    mean, value = pol.forward(obs)
    torch.cuda.synchronize()
    m_e, v_e = _ref_forward(flat, obs, act_dim, emulate_bf16=True)
    m_f, v_f = _ref_forward(flat, obs, act_dim, emulate_bf16=False)
    scale = max(m_f.abs().max().item(), v_f.abs().max().item(), 1e-3)
    # (a) same rounding points: fp32 accumulation order + __expf ELU only
    assert (mean - m_e).abs().max().item() <= 2e-2 * scale
    assert (value - v_e).abs().max().item() <= 2e-2 * scale
    # (b) bf16 tolerance vs the fp32 reference
    assert (mean - m_f).abs().max().item() <= 5e-2 * scale
    assert (value - v_f).abs().max().item() <= 5e-2 * scale


def test_policy_forward_reads_env_observation_rows(sg):
    """The kernel consumes the env's row-major observation view directly."""
    env = sg.VecTaskEnv(robots=("psm",), n_envs=512, seed=1)
    obs = env.reset()
    pol = sg.Policy(env.obs_dim, env.action_dim)
    flat = torch.from_numpy(pol.init_params(seed=0)).cuda()
    pol.load_params(flat)
    mean, value = pol.forward(obs)
    torch.cuda.synchronize()
    m_f, v_f = _ref_forward(flat, obs.clone(), env.action_dim, emulate_bf16=False)
    assert torch.isfinite(mean).all() and torch.isfinite(value).all()
    assert (mean - m_f).abs().max().item() < 5e-2 * max(m_f.abs().max().item(), 1e-4) + 1e-5


def test_init_params_matches_reference_stream(sg, oracle):
    """Policy::init_params: first weights are scale * normal() of
    make_stream(seed, 0x9019) (policy.cpp:87-102)."""
    pol = sg.Policy(27, 7)
    flat = pol.init_params(seed=5)
    r = oracle.make_stream(5, 0x9019)
    scale = np.sqrt(2.0 / 27)
    first = [scale * oracle.normal(r) for _ in range(10)]
    assert np.allclose(flat[:10], np.float32(first))
    assert np.all(flat[pol.log_std_offset:] == -1.0)


@pytest.mark.parametrize("n,act_dim,obs_dim", [(16384, 7, 27), (1000, 6, 24), (130, 8, 30)])
def test_fused_forward_sampling_equals_separate_calls(sg, n, act_dim, obs_dim):
    """sg_policy_act (forward + trainer-stream sampling + log-prob in the
    tensor-core kernel's epilogue) == sg_policy_forward then sg_policy_sample,
    bit for bit: mean, value, actions and log-probs, at an arbitrary stream
    position and a non-default log-std (one dim outside the clamp box)."""
    torch.manual_seed(1)
    pol = sg.Policy(obs_dim, act_dim)
    flat = torch.from_numpy(pol.init_params(seed=4)).cuda()
    flat = flat + 0.05 * torch.randn_like(flat)
    pol.load_params(flat)
    obs = torch.randn(n, obs_dim, device="cuda") * 0.5
    ls = torch.linspace(-1.5, 0.5, act_dim, device="cuda")
    ls[0] = -7.0
    mean, value = pol.forward(obs)
    acts, logp = pol.sample(mean, seed=9, log_std=ls, draw_pos=123456, step_offset=2 * act_dim * 777)
    a2, lp2, v2, m2 = pol.act(obs, seed=9, log_std=ls, draw_pos=123456, step_offset=2 * act_dim * 777,
                              want_mean=True)
    torch.cuda.synchronize()
    assert torch.equal(m2, mean) and torch.equal(v2, value)
    assert torch.equal(a2, acts) and torch.equal(lp2, logp)


@pytest.mark.parametrize("n,act_dim,obs_dim", [(16384, 7, 27), (1000, 6, 24), (130, 16, 30)])
def test_precomputed_noise_equals_fused_sampling(sg, n, act_dim, obs_dim):
    """sg_policy_noise (the sampling's stream part, ahead of the forward) +
    sg_policy_act_noise == sg_policy_act bit for bit: actions, log-probs,
    mean and value, at an arbitrary stream position and log-std."""
    torch.manual_seed(2)
    pol = sg.Policy(obs_dim, act_dim)
    flat = torch.from_numpy(pol.init_params(seed=5)).cuda()
    pol.load_params(flat + 0.05 * torch.randn_like(flat))
    obs = torch.randn(n, obs_dim, device="cuda") * 0.5
    ls = torch.linspace(-1.5, 0.5, act_dim, device="cuda")
    ls[-1] = 3.0
    kw = dict(seed=11, log_std=ls, draw_pos=98765, step_offset=2 * act_dim * 31)
    a1, lp1, v1, m1 = pol.act(obs, want_mean=True, **kw)
    sz, lp2 = pol.noise(n, **kw)
    a2, v2, m2 = pol.act_noise(obs, sz, want_mean=True)
    torch.cuda.synchronize()
    assert torch.equal(m2, m1) and torch.equal(v2, v1)
    assert torch.equal(lp2, lp1)
    assert torch.equal(a2, a1)
