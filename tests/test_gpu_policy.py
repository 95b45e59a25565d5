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


@pytest.mark.parametrize("n", [131072, 1000, 129])
def test_train_forward_matches_bf16_reference(sg, n):
    """sg_policy_train_forward (the PPO update's minibatch forward: persistent
    tensor-core kernel, bf16 obs rows in, every hidden activation stored) ==
    the bf16-emulating fp32 reference, for the activations h1..h3 of both
    trunks and the padded outputs, with the trainer's padded layout (obs width
    27 -> 32, last layers 7 -> 8 and 1 -> 8 rows)."""
    from paper_2310_04676_b200 import ppo
    torch.manual_seed(3)
    O, A = 27, 7
    layout, ls_pad, total, ref_to_pad = ppo.padded_layout(O, A)
    pol = sg.Policy(O, A)
    ref = torch.from_numpy(pol.init_params(seed=6)).cuda()
    ref = ref + 0.05 * torch.randn_like(ref)
    flat = torch.zeros(total, device="cuda")
    flat[torch.from_numpy(ref_to_pad).cuda()] = ref
    tp = sg.Policy(O, A)
    tp.set_param_layout(layout, [32, 256, 128, 64])
    tp.load_params(flat)
    obs = torch.zeros(n, 32, device="cuda", dtype=torch.bfloat16)
    obs[:, :O] = (torch.randn(n, O, device="cuda") * 0.5).to(torch.bfloat16)
    h1 = torch.empty(2, n, 256, device="cuda", dtype=torch.bfloat16)
    h2 = torch.empty(2, n, 128, device="cuda", dtype=torch.bfloat16)
    h3 = torch.empty(2, n, 64, device="cuda", dtype=torch.bfloat16)
    out = torch.empty(2, n, 8, device="cuda", dtype=torch.bfloat16)
    tp.train_forward(obs, h1, h2, h3, out)
    torch.cuda.synchronize()
    r = lambda t: t.to(torch.bfloat16).float()  # noqa: E731
    for t in (0, 1):
        h = obs.float()
        for l, got in enumerate((h1[t], h2[t], h3[t], out[t])):
            (w0, o, i), (b0, ob) = layout[4 * t + l]
            W = flat[w0: w0 + o * i].view(o, i)
            b = flat[b0: b0 + ob]
            z = h @ r(W).T + b
            h = r(torch.where(z > 0, z, torch.expm1(z))) if l < 3 else r(z)
            err = (got.float() - h).abs().max().item()
            scale = h.abs().max().item() + 1e-6
            # one bf16 rounding of an fp32 value that differs by accumulation order
            assert err <= 1.6e-2 * scale, (t, l, err, scale)
            h = got.float()  # continue from the kernel's own activations
    # padded output columns are exact zeros (zero weights and biases)
    assert torch.all(out[0][:, A:] == 0) and torch.all(out[1][:, 1:] == 0)


def test_fused_update_forward_matches_library_gradients(sg):
    """One PPO minibatch gradient with the fused tensor-core forward ==
    the library forward (bf16 GEMMs + ELU kernels) within bf16 tolerance, and
    a whole bf16 iteration learns (finite metrics)."""
    from paper_2310_04676_b200 import ppo
    grads = []
    for fused in (True, False):
        env = sg.VecTaskEnv(robots=("psm",), n_envs=2048, seed=1, episode_len=50)
        tr = ppo.Trainer(env, sg.Policy(env.obs_dim, env.action_dim),
                         ppo.TrainConfig(seed=4, update_precision="bf16", fused_forward=fused, cuda_graph=False))
        assert (tr.train_policy is not None) == fused
        tr.rollout()
        tr.gae()
        cap = tr.T * tr.N
        idx = torch.randperm(cap, device="cuda", generator=torch.Generator(device="cuda").manual_seed(0))[: cap // 4]
        b, g = tr.buf, tr.mb_buf
        m = idx.numel()
        sg.ppo_gather(idx, b["obs"][:tr.T].reshape(cap, tr.O), b["actions"].view(cap, tr.A), b["logp"].view(cap),
                      b["adv"].view(cap), b["ret"].view(cap), g["obs"][:m], g["act"][:m], g["logp"][:m],
                      g["adv"][:m], g["ret"][:m])
        tr.grad.zero_()
        if fused:
            mean_f, value_f = ppo._FusedMLP.apply(tr, g["obs"][:m], tr.layers[0][0])
        else:
            with torch.autocast("cuda", dtype=torch.bfloat16):
                mean_f, value_f = ppo.mlp_layers(tr.layers, g["obs"][:m], device_elu=True, full=True)
        loss, _ = ppo._PPOLossDevice.apply(mean_f.contiguous(), value_f.contiguous(), tr.log_std, g["act"][:m],
                                           g["logp"][:m], g["adv"][:m], g["ret"][:m], tr.A, tr.cfg.clip_eps,
                                           tr.cfg.value_coef, tr.cfg.entropy_coef, True)
        loss.backward()
        torch.cuda.synchronize()
        grads.append(tr.grad.clone())
    a, b2 = grads
    rel = ((a - b2).norm() / b2.norm()).item()
    assert rel < 3e-2, rel
    env = sg.VecTaskEnv(robots=("psm",), n_envs=2048, seed=1, episode_len=50)
    tr = ppo.Trainer(env, sg.Policy(env.obs_dim, env.action_dim), ppo.TrainConfig(seed=4, update_precision="bf16"))
    h = tr.iterate()
    assert all(np.isfinite(h[k]) for k in ("policy_loss", "value_loss", "kl"))


@pytest.mark.parametrize("n_in,k,m", [(256, 128, 131072), (256, 128, 300), (128, 64, 1000), (64, 8, 129),
                                       (64, 8, 100000), (128, 64, 5)])
def test_layer_backward_matches_reference(sg, n_in, k, m):
    """sg_policy_layer_backward (dZ, the next layer's db and this layer's dW in
    one launch): dZ as in sg_policy_dgrad_elu, ragged tails included (rows
    past m neither read nor written: a guard row after the output stays
    untouched); colsum += the column sums of the bf16 dZ it wrote; wgrad +=
    dY^T h against fp64 of the same bf16 operands (fp32 accumulation over
    the rows: relative 1e-3 of the row-norm product)."""
    from paper_2310_04676_b200 import ppo
    torch.manual_seed(11)
    layout, ls_pad, total, _ = ppo.padded_layout(27, 7)
    flat = torch.randn(total, device="cuda") * 0.1
    imgs = sg.WtImages(layout, 0)
    imgs.pack(flat)
    l = {256: 1, 128: 2, 64: 3}[n_in]
    (w0, o, i), _ = layout[l]
    W = flat[w0: w0 + o * i].view(o, i).to(torch.bfloat16).float()
    dy = (torch.randn(m, k, device="cuda") * 0.5).to(torch.bfloat16)
    h = torch.where(torch.rand(m, n_in, device="cuda") < 0.5, torch.rand(m, n_in, device="cuda"),
                    -torch.rand(m, n_in, device="cuda")).to(torch.bfloat16)
    buf = torch.full((m + 1, n_in), 7.0, device="cuda", dtype=torch.bfloat16)
    colsum = torch.full((n_in,), 0.5, device="cuda")
    wg = torch.full((k + 1, n_in), 0.25, device="cuda")  # + a guard row
    dz = sg.layer_backward(dy, imgs.image(0, l), n_in, h, colsum, wg[:k], out=buf[:m])
    torch.cuda.synchronize()
    assert torch.all(buf[m] == 7.0)
    hf = h.float()
    ref = (dy.float() @ W) * torch.where(hf > 0, torch.ones_like(hf), hf + 1)
    err = (dz.float() - ref).abs()
    assert torch.all(err <= 8e-3 * ref.abs() + 1e-4 * ref.abs().max()), err.max().item()
    cs_ref = dz.double().sum(0) + 0.5
    assert torch.allclose(colsum.double(), cs_ref, rtol=1e-4, atol=1e-3 * (1 + m ** 0.5) * 1e-2)
    wg_ref = dy.double().t() @ h.double() + 0.25
    scale = dy.double().norm(dim=0)[:, None] * h.double().norm(dim=0)[None, :]
    assert torch.all((wg[:k].double() - wg_ref).abs() <= 1e-3 * scale + 1e-5), \
        ((wg[:k].double() - wg_ref).abs() / scale).max().item()
    assert torch.all(wg[k] == 0.25)
    # without colsum / wgrad: the same dZ
    dz2 = sg.layer_backward(dy, imgs.image(0, l), n_in, h)
    torch.cuda.synchronize()
    assert torch.equal(dz2, dz)


@pytest.mark.parametrize("m,k3", [(131072, 8), (300, 8), (5, 8), (100000, 1)])
def test_backward_tail_matches_layer_backward(sg, m, k3):
    """sg_policy_backward_tail (layers 3 and 2 in one launch, dZ_2 on chip)
    == the two sg_policy_layer_backward launches it replaces, plus db_3 =
    column sums of dY_3: dZ_1 bit-exact up to the accumulation order (bf16
    within 1 ulp), gradients within fp32 summation-order tolerance."""
    from paper_2310_04676_b200 import ppo
    torch.manual_seed(17)
    layout, ls_pad, total, _ = ppo.padded_layout(27, 7)
    flat = torch.randn(total, device="cuda") * 0.1
    imgs = sg.WtImages(layout, 0)
    imgs.pack(flat)
    dy3 = torch.zeros(m, 8, device="cuda", dtype=torch.bfloat16)
    dy3[:, :k3] = (torch.randn(m, k3, device="cuda") * 0.5).to(torch.bfloat16)

    def act(n):
        return torch.where(torch.rand(m, n, device="cuda") < 0.5, torch.rand(m, n, device="cuda"),
                           -torch.rand(m, n, device="cuda")).to(torch.bfloat16)
    h3, h2 = act(64), act(128)
    z = lambda *s: torch.zeros(*s, device="cuda")  # noqa: E731
    db3, dw3, db2, dw2, db1 = z(k3), z(k3, 64), z(64), z(64, 128), z(128)
    rdw3, rdb2, rdw2, rdb1 = z(8, 64), z(64), z(64, 128), z(128)
    dz1 = sg.backward_tail(dy3[:, :k3] if k3 < 8 else dy3, imgs.image(0, 3), imgs.image(0, 2), h3, h2,
                           db3, dw3, db2, dw2, db1)
    dz2 = sg.layer_backward(dy3, imgs.image(0, 3), 64, h3, rdb2, rdw3)
    rdz1 = sg.layer_backward(dz2, imgs.image(0, 2), 128, h2, rdb1, rdw2)
    torch.cuda.synchronize()
    d = (dz1.float() - rdz1.float()).abs()
    assert torch.all(d <= 2 ** -7 * rdz1.float().abs() + 1e-6), d.max().item()
    assert torch.allclose(db3.double(), dy3[:, :k3].double().sum(0), rtol=1e-4, atol=1e-2)
    assert torch.allclose(dw3, rdw3[:k3], rtol=1e-4, atol=1e-3)
    assert torch.allclose(db2, rdb2, rtol=1e-4, atol=1e-3)
    assert torch.allclose(dw2, rdw2, rtol=1e-3, atol=1e-2)
    assert torch.allclose(db1, rdb1, rtol=1e-3, atol=1e-2)


@pytest.mark.parametrize("m", [131072, 300, 5])
def test_layer_backward_first_layer_weight_gradient(sg, m):
    """sg_policy_layer_backward with x0 (the 256-wide layer): the first
    layer's weight gradient dW_0 += dZ_0^T x0 from the dZ_0 tiles it keeps
    (fp64 of the kernel's own bf16 dZ_0, recomputed by the dZ-writing
    variant, within 1e-3 of the row-norm product), db_0 and dW_1 as without
    x0, and no dZ written."""
    from paper_2310_04676_b200 import ppo
    torch.manual_seed(13)
    layout, ls_pad, total, _ = ppo.padded_layout(27, 7)
    flat = torch.randn(total, device="cuda") * 0.1
    imgs = sg.WtImages(layout, 0)
    imgs.pack(flat)
    dy = (torch.randn(m, 128, device="cuda") * 0.5).to(torch.bfloat16)
    h = torch.where(torch.rand(m, 256, device="cuda") < 0.5, torch.rand(m, 256, device="cuda"),
                    -torch.rand(m, 256, device="cuda")).to(torch.bfloat16)
    x0 = torch.randn(m, 32, device="cuda").to(torch.bfloat16)
    cs_a, cs_b = torch.zeros(256, device="cuda"), torch.zeros(256, device="cuda")
    wg_a, wg_b = torch.zeros(128, 256, device="cuda"), torch.zeros(128, 256, device="cuda")
    wg0 = torch.full((256, 32), 0.5, device="cuda")
    dz = sg.layer_backward(dy, imgs.image(0, 1), 256, h, cs_a, wg_a)
    assert sg.layer_backward(dy, imgs.image(0, 1), 256, h, cs_b, wg_b, x0=x0, wgrad0=wg0) is None
    torch.cuda.synchronize()
    assert torch.allclose(cs_a, cs_b, rtol=1e-4, atol=1e-3)  # (two fp32 summation orders)
    assert torch.allclose(wg_a, wg_b, rtol=1e-4, atol=1e-3)
    ref = dz.double().t() @ x0.double() + 0.5
    scale = dz.double().norm(dim=0)[:, None] * x0.double().norm(dim=0)[None, :]
    assert torch.all((wg0.double() - ref).abs() <= 1e-3 * scale + 1e-5), \
        ((wg0.double() - ref).abs() / scale).max().item()


@pytest.mark.parametrize("n_in,k,m", [(256, 128, 131072), (128, 64, 1000), (64, 8, 129)])
def test_dgrad_elu_matches_reference(sg, n_in, k, m):
    """sg_policy_dgrad_elu (backward through a hidden layer: (dY W) * ELU'(h),
    ELU'(h) = h > 0 ? 1 : h + 1, one tensor-core launch) == the fp32 product of
    the same bf16 operands, rounded once to bf16; W^T packed by
    sg_policy_pack_wt from a padded flat layout."""
    from paper_2310_04676_b200 import ppo
    torch.manual_seed(7)
    layout, ls_pad, total, _ = ppo.padded_layout(27, 7)
    flat = torch.randn(total, device="cuda") * 0.1
    imgs = sg.WtImages(layout, 0)
    imgs.pack(flat)
    l = {256: 1, 128: 2, 64: 3}[n_in]
    for t in (0, 1):
        (w0, o, i), _ = layout[4 * t + l]
        assert (o, i) == (k, n_in)
        W = flat[w0: w0 + o * i].view(o, i).to(torch.bfloat16).float()
        dy = (torch.randn(m, k, device="cuda") * 0.5).to(torch.bfloat16)
        h = torch.where(torch.rand(m, n_in, device="cuda") < 0.5, torch.rand(m, n_in, device="cuda"),
                        -torch.rand(m, n_in, device="cuda")).to(torch.bfloat16)
        dz = sg.dgrad_elu(dy, imgs.image(t, l), n_in, h)
        torch.cuda.synchronize()
        hf = h.float()
        ref = (dy.float() @ W) * torch.where(hf > 0, torch.ones_like(hf), hf + 1)
        err = (dz.float() - ref).abs()
        tol = 8e-3 * ref.abs() + 1e-4 * ref.abs().max()
        assert torch.all(err <= tol), (t, err.max().item())
