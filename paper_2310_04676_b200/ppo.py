"""On-device PPO trainer closing the rollout loop (BASELINE config 5).

Reference: Trainer::iterate / ppo_update / ppo_loss_and_grad / Adam
(proj/src/ppo.cpp:56-341), compute_gae (proj/src/rollout.cpp:42-77),
RolloutBuffer (proj/include/scalpel/rollout.hpp:28-48).

Device mapping (everything stays in HBM; the host only sequences launches):
  rollout step t   sg_policy_forward (tcgen05 BF16 MLP) -> sg_policy_sample
                   (reference trainer stream, bit-exact u32 draws) -> env step
                   (fused sm_100a kernel) -> sg_policy_bootstrap (only tiles
                   with timed-out rows do work) -> D2D copies into the
                   time-major rollout buffer.
  after rollout    sg_policy_forward(last obs) -> sg_compute_gae (+ episode
                   statistics) -> advantage normalisation (global over ranks).
  update           epochs x minibatches of the clipped-surrogate loss on the
                   same MLP in PyTorch (library GEMMs, autograd), gradient
                   all-reduce over ranks (NCCL), global-norm clip, Adam with
                   the reference's bias correction, log-std clamp, then
                   sg_policy_load_params repacks the bf16 tensor-core images.

Documented deviations: the minibatch permutation is a
device permutation (torch.randperm) instead of the reference's Fisher-Yates
over the shared stream; the trainer stream position is still advanced by the
Fisher-Yates draw count so every rollout's z draws match the reference's
stream. With world_size > 1 each rank shuffles its own shard and gradients
are averaged (PPO is not bit-identical across world sizes).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import math
import os

import torch
import torch.nn.functional as F

from . import sg

HALF_LOG_2PI = 0.9189385332046727  # ppo.cpp:28
LOG_STD_MIN, LOG_STD_MAX = -5.0, 2.0  # policy.hpp:28-29
TRAIN_STREAM = 0x7261696E  # ppo.cpp:233

make_stream = sg.make_stream  # rng.hpp:69-83 (host side; PCG32 (state, inc))


@dataclass
class TrainConfig:  # ppo.hpp:25-45
    gamma: float = 0.99
    lam: float = 0.95
    clip_eps: float = 0.2
    learning_rate: float = 3e-4
    epochs: int = 5
    minibatch_count: int = 4
    value_coef: float = 1.0
    entropy_coef: float = 0.0
    max_grad_norm: float = 1.0
    n_steps: int = 32
    init_log_std: float = -1.0
    timeout_bootstrap: bool = True
    seed: int = 0
    update_precision: str = "tf32"  # fp32 | tf32 | bf16 (autocast) for the update GEMMs
    cuda_graph: bool = True  # capture the update in a CUDA graph (single rank)
    # draw step t+1's sampling noise on a side stream during env step t
    # (sg_policy_noise + sg_policy_act_noise, bit-identical to the fused
    # sg_policy_act); measured slower on B200 (rollout 725 vs 788 M
    # env-steps/s: the fp64 noise kernel outlasts the K = 1 env step it
    # overlaps and the fork / join adds graph edges), so off by default
    noise_ahead: bool = False
    # bf16 update: the minibatch forward on the tensor cores
    # (sg_policy_train_forward) instead of library GEMMs + ELU passes
    fused_forward: bool = True
    # the timeout bootstrap of step t-1 inside step t's policy launch
    # (sg_policy_act_bootstrap) instead of its own launch per step
    fold_bootstrap: bool = True

    def validate(self):  # ppo.cpp:31-48 (subset relevant on device)
        if not 0.0 <= self.gamma <= 1.0:
            raise sg.ConfigError("train.gamma must be in [0, 1]")
        if not 0.0 <= self.lam <= 1.0:
            raise sg.ConfigError("train.lambda must be in [0, 1]")
        if not self.clip_eps > 0.0:
            raise sg.ConfigError("train.clip_eps must be > 0")
        if not self.learning_rate > 0.0:
            raise sg.ConfigError("train.learning_rate must be > 0")
        if self.epochs < 1 or self.minibatch_count < 1:
            raise sg.ConfigError("train.epochs and minibatch_count must be >= 1")
        if self.n_steps < 25:
            raise sg.ConfigError("train.n_steps must be >= 25 (GAE horizon floor)")


class _Linear(torch.autograd.Function):
    """y = x W^T + b with every gradient a GEMM (_linear_grads); the bias
    gradient is ones^T dy (a GEMV) instead of a column reduction."""

    _ones: dict = {}

    @staticmethod
    def forward(ctx, x, W, b, Wc=None, bc=None):
        # Wc / bc: compute copies (the bf16 mirror the fused Adam step keeps
        # current); gradients still flow to the fp32 leaves W / b
        Wc = W if Wc is None else Wc
        bc = b if bc is None else bc
        ctx.w_dtype = W.dtype
        ctx.direct = _direct_grads(W, b)
        ctx.save_for_backward(x, Wc)
        return torch.addmm(bc, x, Wc.t())

    @staticmethod
    def backward(ctx, gy):
        x, W = ctx.saved_tensors
        return _linear_grads(ctx, gy, x, W)


_DIRECT_GRADS = os.environ.get("SG_NO_DIRECT_GRAD") != "1"  # A/B switch


def _direct_grads(W, b):
    """(W.grad, b.grad) when the trainer owns them (zeroed before every
    minibatch, each layer used once per forward): the backward GEMMs then
    write the gradients straight into the flat gradient buffer instead of
    returning them for autograd to accumulate (one add kernel per tensor)."""
    if _DIRECT_GRADS and getattr(W, "_sg_direct_grad", False) and W.grad is not None and b.grad is not None:
        return W.grad, b.grad
    return None


def _linear_grads(ctx, gy, x, W):
    """dX = dY W; dW = dY^T X and db = 1^T dY reduce over the whole minibatch
    (K = 131072) straight into fp32 (out_dtype: one GEMM, fp32 accumulation
    and output; tools/gw_probe.py: 24-31 us per layer vs 42-45 us for the
    earlier bf16 split-K batched GEMM + sum, at 1/100 of its rounding error)."""
    gx = gy @ W if ctx.needs_input_grad[0] else None
    B = gy.shape[0]
    out_dt = torch.float32 if gy.dtype in (torch.bfloat16, torch.float16) else None
    key = (B, gy.dtype, gy.device)
    ones = _Linear._ones.get(key)
    if ones is None:
        ones = _Linear._ones[key] = torch.ones(1, B, dtype=gy.dtype, device=gy.device)
    if ctx.direct is not None and (out_dt is not None or gy.dtype == ctx.w_dtype):
        gW_buf, gb_buf = ctx.direct
        skip_gb = getattr(ctx, "gb_done", False)  # the bias gradient came from a column-sum pass
        if getattr(ctx, "gw_done", False):  # the weight gradient came from sg_policy_wgrad
            pass
        elif out_dt:
            torch.mm(gy.t(), x, out_dtype=out_dt, out=gW_buf)
            if not skip_gb:
                torch.mm(ones, gy, out_dtype=out_dt, out=gb_buf.view(1, -1))
        else:
            torch.mm(gy.t(), x, out=gW_buf)
            if not skip_gb:
                torch.mm(ones, gy, out=gb_buf.view(1, -1))
        return gx, None, None, None, None
    gW = torch.mm(gy.t(), x, out_dtype=out_dt) if out_dt else gy.t() @ x
    gb = (torch.mm(ones, gy, out_dtype=out_dt) if out_dt else ones @ gy).view(-1)
    return gx, gW.to(ctx.w_dtype), gb.to(ctx.w_dtype), None, None


class _LinearELU(torch.autograd.Function):
    """h = ELU(x W^T + b) (policy.cpp:120-128): the GEMM in the library, the
    activation in place on the device ELU kernel (train.cu). Only h is kept:
    the derivative exp(z) = h + 1 on the negative side comes from the output."""

    @staticmethod
    def forward(ctx, x, W, b, Wc=None, bc=None):
        Wc = W if Wc is None else Wc
        bc = b if bc is None else bc
        ctx.w_dtype = W.dtype
        ctx.direct = _direct_grads(W, b)
        h = sg.elu_forward(torch.addmm(bc, x, Wc.t()), out=None)
        ctx.save_for_backward(x, Wc, h)
        return h

    @staticmethod
    def backward(ctx, gh):
        x, W, h = ctx.saved_tensors
        return _linear_grads(ctx, sg.elu_backward(h, gh.contiguous()), x, W)


def _linear(x, W, b, Wm=None, bm=None, elu: bool = False):
    fn = _LinearELU if elu else _Linear
    if torch.is_autocast_enabled():
        dt = torch.get_autocast_dtype("cuda")
        with torch.autocast("cuda", enabled=False):
            if Wm is not None and Wm.dtype == dt:
                return fn.apply(x.to(dt), W, b, Wm, bm)
            return fn.apply(x.to(dt), W.to(dt), b.to(dt))
    return fn.apply(x, W, b)


class _FusedMLP(torch.autograd.Function):
    """The update's minibatch Policy::forward (bf16) as ONE tensor-core launch
    (sg_policy_train_forward: both trunks, every hidden activation stored as
    it is packed for the next layer) instead of 8 library GEMMs + 6 ELU passes;
    the backward pass is the library one (_linear_grads per layer, direct
    gradient writes, the train.cu ELU derivative from the stored outputs).
    `leaf` is any trainer parameter, passed only so autograd calls backward."""

    @staticmethod
    def forward(ctx, trainer, obs, leaf):
        m = obs.shape[0]
        h1, h2, h3, out = trainer.fused_buffers(m)
        trainer.train_policy.load_params(trainer.params)  # this minibatch's weights (Adam ran since)
        if trainer.wt_images is not None:
            trainer.wt_images.pack(trainer.params)  # W^T for the fused backward
        trainer.train_policy.train_forward(obs, h1, h2, h3, out)
        ctx.trainer, ctx.obs, ctx.acts = trainer, obs, (h1, h2, h3)
        return out[0], out[1]

    @staticmethod
    def backward(ctx, g_mean, g_value):
        tr, obs = ctx.trainer, ctx.obs
        h1, h2, h3 = ctx.acts
        colsum = tr.colsum_bias
        for t, gy in ((0, g_mean), (1, g_value)):
            ins = (obs, h1[t], h2[t], h3[t])
            g = gy.contiguous().to(torch.bfloat16)
            l0_done = False
            L = [tr.layers[4 * t + j] for j in range(4)]
            tail = (tr.wt_images is not None and tr.fuse_tail and colsum and tr.wgrad_partial is not None
                    and g.shape[1] <= 8 and all(_direct_grads(L[j][0], L[j][1]) is not None for j in (1, 2, 3)))
            if tail:  # layers 3 and 2 (dZ_2 kept on chip) and db_1 in one launch
                g = sg.backward_tail(g, tr.wt_images.image(t, 3), tr.wt_images.image(t, 2), h3[t], h2[t],
                                     L[3][1].grad, L[3][0].grad, L[2][1].grad, L[2][0].grad, L[1][1].grad)
            for l in ((1, 0) if tail else (3, 2, 1, 0)):
                if l0_done:  # (dW_0 and db_0 came with layer 1's backward)
                    break
                W, b, Wm, _ = tr.layers[4 * t + l]
                direct = _direct_grads(W, b)
                cs = colsum and direct is not None
                if cs and l == 3:  # the last layer's db: one column-sum pass over dY
                    sg.elu_backward_colsum(None, g, b.grad, out=False)
                fused = tr.wt_images is not None and l > 0
                # (tensor-core reductions beat the split-K GEMMs on every layer:
                # 256x32 23.7 vs 30.8 us, 128x256 26.7 vs 32.0, 64x128 19.4 vs
                # 27.5 (TMA-fed), 8x64 18.7 vs 24.6; tools/wgrad_probe.py)
                gw = tr.wgrad_partial is not None and direct is not None
                if gw and not fused:  # dW = dY^T X on the tensor cores (per-CTA row slices + one sum)
                    sg.wgrad(g, ins[l], tr.wgrad_partial, W.grad)
                lctx = _LayerCtx(needs_gx=l > 0 and not fused, direct=direct, w_dtype=W.dtype, gb_done=cs,
                                 gw_done=gw)
                gx, gW, gb, _, _ = _linear_grads(lctx, g, ins[l], Wm)
                if lctx.direct is None:  # (only without the trainer-owned gradient views)
                    W.grad.add_(gW)
                    b.grad.add_(gb)
                if fused:  # dZ = (dY W) * ELU'(h), the next db and this dW in one launch
                    W0 = tr.layers[4 * t][0]
                    l0 = (l == 1 and cs and gw and tr.fuse_l0 and obs.dtype == torch.bfloat16 and obs.shape[1] == 32
                          and obs.is_contiguous() and _direct_grads(W0, tr.layers[4 * t][1]) is not None)
                    g = sg.layer_backward(g, tr.wt_images.image(t, l), ins[l].shape[1], ins[l],
                                          tr.layers[4 * t + l - 1][1].grad if cs else None, W.grad if gw else None,
                                          x0=obs if l0 else None, wgrad0=W0.grad if l0 else None)
                    l0_done = l0
                elif l > 0 and cs:  # ELU' and the next-lower layer's db in one pass
                    g = sg.elu_backward_colsum(ins[l], gx.contiguous(), tr.layers[4 * t + l - 1][1].grad)
                elif l > 0:
                    g = sg.elu_backward(ins[l], gx.contiguous())
        return None, None, None


class _LayerCtx:
    """The attributes _linear_grads reads from an autograd ctx."""

    def __init__(self, needs_gx: bool, direct, w_dtype, gb_done: bool = False, gw_done: bool = False):
        self.needs_input_grad = (needs_gx,)
        self.direct = direct
        self.w_dtype = w_dtype
        self.gb_done = gb_done
        self.gw_done = gw_done


def param_layout(obs_dim: int, act_dim: int):
    """Flat offsets of (W_l, b_l) per trunk and of log_std (policy.cpp:42-63)."""
    dims = [obs_dim, 256, 128, 64]
    off = 0
    out = []
    for trunk in (0, 1):
        o_last = act_dim if trunk == 0 else 1
        for l in range(4):
            i, o = dims[l], (dims[l + 1] if l < 3 else o_last)
            out.append(((off, o, i), (off + o * i, o)))
            off += o * i + o
    return out, off


def _up8(x: int) -> int:
    return (x + 7) // 8 * 8


def padded_layout(obs_dim: int, act_dim: int):
    """Training copy of the parameters with GEMM-friendly shapes: the obs
    width and the output widths padded to multiples of 8 (odd leading
    dimensions such as 27 and 7 push cuBLAS onto 4-8x slower kernels; see
    tools/gemm_probe.py). Padded weights / biases start at zero and receive
    zero gradients (padded inputs are zero, padded outputs are unused), so
    Adam keeps them at zero. Returns (layout, log_std offset, total size,
    reference index -> padded index map)."""
    import numpy as np
    ref_layout, ls_ref = param_layout(obs_dim, act_dim)
    dims_p = [_up8(obs_dim), 256, 128, 64]
    layout = []
    ref_to_pad = np.zeros(ls_ref + act_dim, dtype=np.int64)
    off = 0
    for k, ((w0, o, i), (b0, ob)) in enumerate(ref_layout):
        l = k % 4
        ip = dims_p[l]
        op = _up8(o) if l == 3 else o
        rows = np.arange(o)[:, None]
        cols = np.arange(i)[None, :]
        ref_to_pad[w0: w0 + o * i] = (off + rows * ip + cols).reshape(-1)
        bo = off + op * ip
        ref_to_pad[b0: b0 + ob] = bo + np.arange(ob)
        layout.append(((off, op, ip), (bo, op)))
        off = bo + op
    ls_pad = off
    ref_to_pad[ls_ref: ls_ref + act_dim] = ls_pad + np.arange(act_dim)
    return layout, ls_pad, ls_pad + _up8(act_dim), ref_to_pad


def mlp_forward(params: torch.Tensor, obs: torch.Tensor, obs_dim: int, act_dim: int):
    """Policy::forward (policy.cpp:110-161) on a flat parameter view."""
    layout, ls_off = param_layout(obs_dim, act_dim)
    layers = [(params[w0: w0 + o * i].view(o, i), params[b0: b0 + ob]) for (w0, o, i), (b0, ob) in layout]
    mean, value = mlp_layers(layers, obs)
    return mean, value, ls_off


def mlp_layers(layers, obs, device_elu: bool = False, full: bool = False):
    """layers[k] = (W, b) or (W, b, W_bf16_mirror, b_bf16_mirror).
    device_elu: hidden activations on the train.cu ELU kernels (CUDA tensors).
    full: return the whole (padded) critic output instead of its column 0."""
    outs = []
    for trunk in (0, 1):
        h = obs
        for l in range(4):
            if device_elu and l < 3:
                h = _linear(h, *layers[4 * trunk + l], elu=True)
            else:
                h = _linear(h, *layers[4 * trunk + l])
                if l < 3:
                    h = F.elu(h)
        outs.append(h)
    return (outs[0], outs[1]) if full else (outs[0], outs[1][:, 0])


def loss_head(mean, value, log_std_raw, actions, old_logp, adv, ret, cfg: TrainConfig):
    """The data part of ppo_loss_and_grad (ppo.cpp:90-154) on (mean, value,
    raw log-std); autograd reproduces the reference's analytic gradients."""
    log_std = log_std_raw.clamp(LOG_STD_MIN, LOG_STD_MAX)  # projection: no gradient outside the box
    inv_std = torch.exp(-log_std)
    diff = actions - mean
    logp = (-0.5 * (diff * inv_std) ** 2 - log_std - HALF_LOG_2PI).sum(1)
    ratio = torch.exp(logp - old_logp)
    unclipped = ratio * adv
    clipped = ratio.clamp(1.0 - cfg.clip_eps, 1.0 + cfg.clip_eps) * adv
    # d(-surr)/dlogp follows the unclipped branch when it is the min (ties included)
    surr = torch.where(unclipped <= clipped, unclipped, clipped.detach())
    policy_loss = -surr.mean()
    value_loss = 0.5 * ((value - ret) ** 2).mean()
    entropy = (log_std + 0.5 + HALF_LOG_2PI).sum()
    loss = policy_loss + cfg.value_coef * value_loss - cfg.entropy_coef * entropy
    with torch.no_grad():
        metrics = torch.stack([policy_loss.detach(), value_loss.detach(), entropy.detach(),
                               (old_logp - logp).mean().detach(),
                               ((ratio - 1.0).abs() > cfg.clip_eps).float().mean()])
    return loss, metrics


class _PPOLossDevice(torch.autograd.Function):
    """The data part of ppo_loss_and_grad (ppo.cpp:90-154) on one fused device
    kernel (train.cu sg_ppo_loss): it forms the loss, the metrics and, like the
    reference, the analytic gradients in the same pass; backward only scales
    them by the incoming gradient. mean_full / value_full are the padded
    last-layer outputs (columns >= A, resp. >= 1, get zero gradient)."""

    @staticmethod
    def forward(ctx, mean_full, value_full, log_std_raw, act, old_logp, adv, ret, A, clip_eps, value_coef,
                entropy_coef, unit_grad=False):
        ctx.unit_grad = unit_grad
        dmean = torch.empty_like(mean_full)
        dvalue = torch.empty_like(value_full)
        dls = torch.empty_like(log_std_raw)
        acc = torch.empty(4 + A, device=mean_full.device)
        out = torch.empty(6, device=mean_full.device)
        sg.ppo_loss(mean_full, value_full, log_std_raw, act, old_logp, adv, ret, A, clip_eps, value_coef,
                    entropy_coef, LOG_STD_MIN, LOG_STD_MAX, dmean, dvalue, dls, acc, out)
        ctx.save_for_backward(dmean, dvalue, dls)
        metrics = out[1:6]
        ctx.mark_non_differentiable(metrics)
        return out[0], metrics

    @staticmethod
    def backward(ctx, g_loss, g_metrics):
        # the trainer backpropagates the loss itself (loss.backward(): g_loss
        # == 1), so the analytic gradients pass through unscaled (no extra
        # elementwise launches); other callers get them scaled
        dmean, dvalue, dls = ctx.saved_tensors
        if ctx.unit_grad:
            return dmean, dvalue, dls, None, None, None, None, None, None, None, None, None
        g = g_loss.to(dmean.dtype)
        return dmean * g, dvalue * g, dls * g_loss, None, None, None, None, None, None, None, None, None


def ppo_loss(params, obs, actions, old_logp, adv, ret, cfg: TrainConfig, obs_dim, act_dim):
    """ppo_loss_and_grad (ppo.cpp:76-155): MLP forward + loss head."""
    mean, value, ls_off = mlp_forward(params, obs, obs_dim, act_dim)
    return loss_head(mean.float(), value.float(), params[ls_off: ls_off + act_dim], actions, old_logp, adv, ret,
                     cfg)


def allreduce_mean_(t: torch.Tensor, dist, force: bool = False) -> torch.Tensor:
    """Gradient all-reduce (sum, then / world) before clipping (ppo.cpp:201).
    force: issue the collective even at world size 1 (tests of the captured
    NCCL path on a single GPU)."""
    if dist is not None and dist.is_initialized() and (dist.get_world_size() > 1 or force):
        dist.all_reduce(t)
        t /= dist.get_world_size()
    return t


def global_adv_stats(adv: torch.Tensor, dist) -> tuple[torch.Tensor, torch.Tensor]:
    """rollout.cpp:70-76 normalisation statistics over every rank's buffer."""
    s = torch.stack([adv.sum(), (adv * adv).sum(), torch.tensor(float(adv.numel()), device=adv.device)]).double()
    if dist is not None and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(s)
    mean = s[0] / s[2]
    var = (s[1] / s[2] - mean * mean).clamp_min(0.0)
    return mean.float(), var.sqrt().float()


class Trainer:
    def __init__(self, env: "sg.VecTaskEnv", policy: "sg.Policy", cfg: TrainConfig, dist=None):
        cfg.validate()
        self.env, self.policy, self.cfg, self.dist = env, policy, cfg, dist
        dev = torch.device(f"cuda:{env.device}")
        self.dev = dev
        N, A, O, T = env.n_envs, env.action_dim, env.obs_dim, cfg.n_steps
        self.N, self.A, self.O, self.T = N, A, O, T
        # fp32 master parameters in the padded training layout (padded_layout)
        # plus one flat gradient; per-layer leaves alias slices of both, so
        # autograd writes straight into the flat gradient (no slice-backward
        # graph) and the all-reduce / clip / Adam run on single flat tensors.
        # The reference-layout vector the tensor-core kernel packs from is a
        # gather of the master (self.ref_params).
        layout, ls_pad, total, ref_to_pad = padded_layout(O, A)
        self.ref_to_pad = torch.from_numpy(ref_to_pad).to(dev)
        self.params = torch.zeros(total, device=dev)
        self.params[self.ref_to_pad] = torch.from_numpy(policy.init_params(cfg.seed, cfg.init_log_std)).to(dev)
        self.grad = torch.zeros_like(self.params)
        self.params.grad = self.grad
        self.ls_off = ls_pad
        self.O_pad = _up8(O)
        self.layers = []
        # bf16 update: the fused Adam step (sg_adam_step) keeps a bf16 mirror
        # of the master parameters for the GEMMs (no per-call weight casts)
        self.mirror = (torch.zeros(total, device=dev, dtype=torch.bfloat16)
                       if cfg.update_precision == "bf16" else None)
        for (w0, o, i), (b0, ob) in layout:
            W = self.params[w0: w0 + o * i].view(o, i).detach().requires_grad_(True)
            b = self.params[b0: b0 + ob].detach().requires_grad_(True)
            W.grad = self.grad[w0: w0 + o * i].view(o, i)
            b.grad = self.grad[b0: b0 + ob]
            W._sg_direct_grad = True  # the backward GEMMs write these views directly
            if self.mirror is not None:
                self.layers.append((W, b, self.mirror[w0: w0 + o * i].view(o, i), self.mirror[b0: b0 + ob]))
            else:
                self.layers.append((W, b))
        self.log_std = self.params[self.ls_off: self.ls_off + A].detach().requires_grad_(True)
        # the fused minibatch forward packs its weights from the padded copy
        self.train_policy = None
        self.wt_images = None
        self.fuse_l0 = False
        self.fuse_tail = False
        # bias gradients from column-sum passes (fused into the ELU backward)
        # instead of M = 1 split-K GEMMs; SG_NO_COLSUM_BIAS=1 for the GEMMs
        self.colsum_bias = os.environ.get("SG_NO_COLSUM_BIAS") != "1"
        # weight gradients on the tensor cores (sg_policy_wgrad) instead of
        # split-K library GEMMs; SG_NO_WGRAD=1 for the GEMMs
        self.wgrad_partial = None
        self._fused_buf = None
        if cfg.fused_forward and cfg.update_precision == "bf16" and os.environ.get("SG_NO_FUSED_FWD") != "1":
            self.train_policy = sg.Policy(O, A, device=policy.device)
            self.train_policy.set_param_layout(layout, [_up8(O), 256, 128, 64])
            # the fused backward through the hidden layers: (dY W) * ELU'(h) and
            # the next layer's bias sums in one tensor-core launch with h / dZ
            # moved by TMA (sg_policy_dgrad_elu_colsum): 39.5 / 22.8 / 16.5 us
            # vs 61.2 / 31.5 / 24.0 for library GEMM + ELU pass at m = 131072
            # (tools/dgrad_probe.py); update 11.41 -> 10.28 ms. SG_NO_FUSED_BWD=1
            # for the library path
            if os.environ.get("SG_NO_FUSED_BWD") != "1":
                self.wt_images = sg.WtImages(layout, dev)
            # layer 1's backward also takes the first layer's weight gradient
            # from the dZ_0 tile it holds (dZ_0 never written); SG_NO_FUSE_L0=1
            # for a separate sg_policy_wgrad over a written dZ_0
            self.fuse_l0 = os.environ.get("SG_NO_FUSE_L0") != "1"
            # the last two layers' backward as one launch (sg_policy_backward_tail);
            # SG_NO_FUSE_TAIL=1 for one sg_policy_layer_backward per layer
            self.fuse_tail = os.environ.get("SG_NO_FUSE_TAIL") != "1"
            if os.environ.get("SG_NO_WGRAD") != "1":
                self.wgrad_partial = torch.empty(148 * 128 * 256, device=dev)
        self.log_std.grad = self.grad[self.ls_off: self.ls_off + A]
        # The whole update is one CUDA-graph replay at any world size: the NCCL
        # gradient all-reduce of every minibatch is captured with the GEMMs
        # (the communicator is created by the warm-up updates before capture).
        self.use_graph = cfg.cuda_graph
        self.force_collectives = False
        # Adam state (ppo.cpp:50-64) for the fused optimizer step
        self.adam_m = torch.zeros_like(self.params)
        self.adam_v = torch.zeros_like(self.params)
        self.adam_t = torch.zeros(1, device=dev, dtype=torch.int32)
        self.grad_sq = torch.zeros(2, device=dev)  # [squared norm scratch, sticky non-finite flag]
        if self.mirror is not None:
            self.mirror.copy_(self.params)
        policy.load_params(self.ref_params())
        self.perms = torch.empty(cfg.epochs, T * N, dtype=torch.int64, device=dev)
        self.g_metrics = torch.zeros(5, device=dev)
        self.graph = None
        z = lambda *s, dt=torch.float32: torch.zeros(*s, device=dev, dtype=dt)
        # obs slot t = the policy input of rollout step t; the env writes step
        # t's observations straight into slot t + 1 (sg_env_step_into), and
        # slot T carries over to the next rollout's slot 0
        self.buf = dict(obs=z(T + 1, N, O), actions=z(T, N, A), logp=z(T, N), values=z(T, N), rewards=z(T, N),
                        terminated=z(T, N, dt=torch.uint8), timed_out=z(T, N, dt=torch.uint8), boot=z(T, N),
                        task_error=z(T, N), adv=z(T, N), ret=z(T, N), last_values=z(N))
        mb = (T * N + cfg.minibatch_count - 1) // cfg.minibatch_count
        obs_dt = torch.bfloat16 if cfg.update_precision == "bf16" else torch.float32
        self.mb_buf = dict(obs=z(mb, _up8(O), dt=obs_dt), act=z(mb, A), logp=z(mb), adv=z(mb), ret=z(mb))
        self.mean = z(N, A)
        # scaled sampling noise of the current / next rollout step (sg_policy_noise)
        self.noise = [z(N, A, dt=torch.float64), z(N, A, dt=torch.float64)]
        self.noise_stream = torch.cuda.Stream(dev)
        self.log_std_c = z(A)
        self.rollout_graph = None
        self.ep_acc = z(N)
        self.stats = z(4, dt=torch.float64)
        self.stream_state, self.stream_inc = make_stream(cfg.seed, TRAIN_STREAM)
        # The reference draws every rollout step's noise from ONE stream over
        # all global rows (ppo.cpp:264-270) and shuffles the global buffer
        # (:175-178). A shard of global rows [row_off, row_off + N) of
        # world * N takes its rows' slice of each step's draws, and the stream
        # advances by the global draw counts.
        multi = dist is not None and dist.is_initialized()
        self.world = dist.get_world_size() if multi else 1
        self.global_n = self.world * N
        self.row_off = int(env.cfg.row_offset)
        self.draw_pos = 0  # u32 draws consumed from the trainer stream
        self.d_pos = torch.zeros(1, dtype=torch.int64, device=dev)
        self.obs = None
        self.env_steps = 0
        self.iteration = 0
        self._perm_stream = (torch.cuda.Stream(dev) if os.environ.get("SG_NO_PERM_PREFETCH") != "1" else None)
        self._perms_ready = None
        self.gen = torch.Generator(device=dev)
        self.gen.manual_seed(cfg.seed * 1000003 + (dist.get_rank() if dist is not None and dist.is_initialized() else 0))

    def fused_buffers(self, m: int):
        """bf16 activation buffers of the fused minibatch forward, [2][m][width]
        views of one allocation sized for the largest minibatch (fixed
        addresses: the update is graph-captured)."""
        if self._fused_buf is None:
            mb = (self.T * self.N + self.cfg.minibatch_count - 1) // self.cfg.minibatch_count
            self._fused_buf = torch.empty(2 * mb * (256 + 128 + 64 + 8), dtype=torch.bfloat16, device=self.dev)
        buf, out = self._fused_buf, []
        off = 0
        for w in (256, 128, 64, 8):
            out.append(buf[off: off + 2 * m * w].view(2, m, w))
            off += 2 * m * w
        return out

    # -- rollout -----------------------------------------------------------
    def _stream(self):
        return torch.cuda.current_stream(self.dev).cuda_stream

    def rollout(self):
        """n_steps of policy forward -> sample -> env step -> bootstrap into the
        rollout buffer (ppo.cpp:258-313). From the second iteration on the whole
        rollout is one CUDA-graph replay (every buffer pointer is fixed; the
        trainer-stream position lives in device memory), so ~8 launches per
        env step no longer pace the host (tools/rollout_probe.py: 2.9 ->
        1.2 ms per 32-step rollout)."""
        env, b = self.env, self.buf
        N, A, T = self.N, self.A, self.T
        if self.obs is None:  # first rollout: the reset observations enter through slot T
            self.obs = env.reset()
            b["obs"][T].copy_(self.obs)
        self.d_pos.fill_(self.draw_pos)
        if self.rollout_graph is not None:
            self.rollout_graph.replay()
        else:
            self._rollout_body()
            if self.use_graph:  # record (not run) the graph the next rollouts replay
                self._capture_rollout()
        self.draw_pos += 2 * T * self.global_n * A
        self.env_steps += N * T

    def _capture_rollout(self) -> None:
        side = torch.cuda.Stream(self.dev)
        side.wait_stream(torch.cuda.current_stream(self.dev))
        self.rollout_graph = torch.cuda.CUDAGraph()
        self.env.set_stream(side)
        try:
            with torch.cuda.graph(self.rollout_graph, stream=side):
                self._rollout_body()
        finally:
            self.env.set_stream(None)
        torch.cuda.current_stream(self.dev).wait_stream(side)

    def _rollout_body(self):
        env, pol, b = self.env, self.policy, self.buf
        N, A, T = self.N, self.A, self.T
        L = sg.lib()
        st = self._stream()
        log_std = self.log_std_c
        log_std.copy_(self.params[self.ls_off: self.ls_off + A])
        b["obs"][0].copy_(b["obs"][T])
        ahead = self.cfg.noise_ahead
        fold = self.cfg.fold_bootstrap and self.cfg.timeout_bootstrap and not ahead
        tobs = None
        main = torch.cuda.current_stream(self.dev)

        def noise(t, stream):  # step t's draws: scaled noise + log-probs (ppo.cpp:262-277)
            sg._pcheck(L.sg_policy_noise(pol._h, N, log_std.data_ptr(), self.stream_state, self.stream_inc,
                                         self.d_pos.data_ptr(), 2 * A * (t * self.global_n + self.row_off),
                                         self.noise[t % 2].data_ptr(), b["logp"][t].data_ptr(), stream))
        if ahead:
            noise(0, st)
        for t in range(T):
            obs = b["obs"][t]
            if ahead:
                # policy forward + actions from the noise drawn during the
                # previous env step: one tcgen05 launch
                sg._pcheck(L.sg_policy_act_noise(pol._h, obs.data_ptr(), N, obs.stride(0),
                                                 self.noise[t % 2].data_ptr(), b["actions"][t].data_ptr(), None,
                                                 b["values"][t].data_ptr(), st))
                if t + 1 < T:  # the next step's draws (fp64 pipe) overlap this env step (fp32 SIMT)
                    self.noise_stream.wait_stream(main)
                    with torch.cuda.stream(self.noise_stream):
                        noise(t + 1, self.noise_stream.cuda_stream)
            elif fold and t > 0:
                # policy forward + sampling + log-prob, and step t-1's timeout
                # bootstrap (its terminal rows are still in the env's buffer):
                # one tcgen05 launch
                sg._pcheck(L.sg_policy_act_bootstrap(
                    pol._h, obs.data_ptr(), N, obs.stride(0), log_std.data_ptr(), self.stream_state, self.stream_inc,
                    self.d_pos.data_ptr(), 2 * A * (t * self.global_n + self.row_off), b["actions"][t].data_ptr(),
                    b["logp"][t].data_ptr(), None, b["values"][t].data_ptr(), tobs.data_ptr(), self.O,
                    b["timed_out"][t - 1].data_ptr(), b["terminated"][t - 1].data_ptr(), b["boot"][t - 1].data_ptr(),
                    st))
            else:
                # policy forward + Gaussian sampling + log-prob: one tcgen05 launch
                sg._pcheck(L.sg_policy_act(pol._h, obs.data_ptr(), N, obs.stride(0), log_std.data_ptr(),
                                           self.stream_state, self.stream_inc, self.d_pos.data_ptr(),
                                           2 * A * (t * self.global_n + self.row_off), b["actions"][t].data_ptr(),
                                           b["logp"][t].data_ptr(), None, b["values"][t].data_ptr(), st))
            # the env writes the step's observations / rewards / flags / errors
            # into the rollout buffer itself (ppo.cpp:280-299)
            direct = (N * self.O) % 4 == 0  # slots 16-byte aligned: the kernel's row stores go straight in
            res = env.step_into(b["actions"][t], observations=b["obs"][t + 1] if direct else None,
                                rewards=b["rewards"][t], task_error=b["task_error"][t],
                                terminated=b["terminated"][t], timed_out=b["timed_out"][t])
            if not direct:
                b["obs"][t + 1].copy_(res.observations)
            tobs = res.terminal_observations
            if not self.cfg.timeout_bootstrap:
                b["boot"][t].zero_()
            elif not fold or t == T - 1:
                sg._pcheck(L.sg_policy_bootstrap(pol._h, tobs.data_ptr(), N, self.O, res.timed_out.data_ptr(),
                                                 res.terminated.data_ptr(), b["boot"][t].data_ptr(), st))
            if ahead and t + 1 < T:
                main.wait_stream(self.noise_stream)
        pol.forward(b["obs"][T], self.mean, b["last_values"])

    def gae(self):
        b = self.buf
        self.stats.zero_()
        sg._pcheck(sg.lib().sg_compute_gae(
            b["rewards"].data_ptr(), b["values"].data_ptr(), b["terminated"].data_ptr(), b["timed_out"].data_ptr(),
            b["boot"].data_ptr(), b["last_values"].data_ptr(), b["task_error"].data_ptr(), self.T, self.N,
            self.cfg.gamma, self.cfg.lam, b["adv"].data_ptr(), b["ret"].data_ptr(), self.ep_acc.data_ptr(),
            self.stats.data_ptr(), self._stream()))
        mean, std = global_adv_stats(b["adv"], self.dist)
        b["adv"].sub_(mean).div_(std + 1e-8)

    # -- update ------------------------------------------------------------
    def ref_params(self) -> torch.Tensor:
        """The reference's flat parameter layout (policy.cpp:42-63), fp32."""
        return self.params[self.ref_to_pad]

    def _update_body(self, perms: torch.Tensor, metrics: torch.Tensor):
        """epochs x minibatches of ppo_update (ppo.cpp:157-224) on device
        tensors only (no host synchronisation, so it can be graph-captured)."""
        cfg, b = self.cfg, self.buf
        cap = self.T * self.N
        mb = (cap + cfg.minibatch_count - 1) // cfg.minibatch_count
        obs = b["obs"][:self.T].reshape(cap, self.O)
        act = b["actions"].view(cap, self.A)
        logp, adv, ret = b["logp"].view(cap), b["adv"].view(cap), b["ret"].view(cap)
        g = self.mb_buf
        for e in range(cfg.epochs):
            for start in range(0, cap, mb):
                idx = perms[e, start: start + mb]
                m_rows = idx.numel()
                # one launch gathers the minibatch rows (obs straight to the GEMM dtype)
                sg.ppo_gather(idx, obs, act, logp, adv, ret, g["obs"][:m_rows], g["act"][:m_rows],
                              g["logp"][:m_rows], g["adv"][:m_rows], g["ret"][:m_rows])
                # (self.grad is zero here: initially, and after every fused Adam step)
                if self.train_policy is not None:  # one tensor-core launch (bf16 obs rows in)
                    mean_f, value_f = _FusedMLP.apply(self, g["obs"][:m_rows], self.layers[0][0])
                else:
                    with torch.autocast("cuda", dtype=torch.bfloat16, enabled=cfg.update_precision == "bf16"):
                        mean_f, value_f = mlp_layers(self.layers, g["obs"][:m_rows], device_elu=True, full=True)
                loss, m = _PPOLossDevice.apply(mean_f.contiguous(), value_f.contiguous(), self.log_std,
                                               g["act"][:m_rows], g["logp"][:m_rows], g["adv"][:m_rows],
                                               g["ret"][:m_rows], self.A, cfg.clip_eps, cfg.value_coef,
                                               cfg.entropy_coef, True)
                loss.backward()  # d loss = 1: the loss head's gradients pass through unscaled
                allreduce_mean_(self.grad, self.dist, force=self.force_collectives)
                self._adam_step()
                metrics += m

    def _adam_step(self) -> None:
        """Global-norm clip (ppo.cpp:201-204), Adam::step (ppo.cpp:56-64),
        log-std box projection (:206-207), gradient reset and bf16 mirror
        refresh in two kernels (sg_adam_step), no host synchronisation."""
        cfg = self.cfg
        sg._pcheck(sg.lib().sg_adam_step(
            self.params.data_ptr(), self.grad.data_ptr(), self.adam_m.data_ptr(), self.adam_v.data_ptr(),
            self.mirror.data_ptr() if self.mirror is not None else None, self.params.numel(),
            self.grad_sq.data_ptr(), self.adam_t.data_ptr(), cfg.learning_rate, 0.9, 0.999, 1e-8,
            cfg.max_grad_norm, self.ls_off, self.A, LOG_STD_MIN, LOG_STD_MAX, self._stream()))

    def _new_perms(self) -> None:
        cap = self.T * self.N
        for e in range(self.cfg.epochs):
            self.perms[e].copy_(torch.randperm(cap, device=self.dev, generator=self.gen))

    def _capture_update(self) -> None:
        """Capture the whole update (5 epochs x 4 minibatches: gathers, forward,
        backward, clip, Adam, log-std clamp) in one CUDA graph so the host no
        longer paces ~2000 small launches. Warm-up runs on saved copies of the
        parameters / optimizer state, which are restored before training."""
        saved = [t.clone() for t in (self.params, self.adam_m, self.adam_v, self.adam_t)]
        side = torch.cuda.Stream(self.dev)
        side.wait_stream(torch.cuda.current_stream(self.dev))
        with torch.cuda.stream(side):
            self._new_perms()
            for _ in range(2):
                self._update_body(self.perms, self.g_metrics)
        torch.cuda.current_stream(self.dev).wait_stream(side)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self._update_body(self.perms, self.g_metrics)
        with torch.no_grad():
            for t, v in zip((self.params, self.adam_m, self.adam_v, self.adam_t), saved):
                t.copy_(v)
            if self.mirror is not None:
                self.mirror.copy_(self.params)
        self.grad.zero_()

    def update(self):
        cfg = self.cfg
        cap = self.T * self.N
        prev_tf32 = torch.backends.cuda.matmul.allow_tf32
        torch.backends.cuda.matmul.allow_tf32 = cfg.update_precision == "tf32"
        try:
            if self.use_graph:
                if self.graph is None:
                    self._capture_update()
                cur = torch.cuda.current_stream(self.dev)
                if self._perms_ready is not None:  # drawn after the previous update, beside the rollout
                    cur.wait_event(self._perms_ready)
                else:
                    self._new_perms()
                self.g_metrics.zero_()
                self.graph.replay()
                metrics = self.g_metrics.clone()
                if self._perm_stream is not None:
                    # the next update's permutations (same generator, same draw order) on a
                    # side stream once this update has read its own: the sorts overlap the
                    # next rollout's latency-bound launches instead of heading the update
                    self._perm_stream.wait_stream(cur)
                    with torch.cuda.stream(self._perm_stream):
                        self._new_perms()
                    self._perms_ready = torch.cuda.Event()
                    self._perms_ready.record(self._perm_stream)
            else:
                metrics = torch.zeros(5, device=self.dev)
                self._new_perms()
                self._update_body(self.perms, metrics)
        finally:
            torch.backends.cuda.matmul.allow_tf32 = prev_tf32
        # the reference's Fisher-Yates consumed (global buffer size - 1) draws per epoch
        self.draw_pos += cfg.epochs * (self.T * self.global_n - 1)
        self.policy.load_params(self.ref_params())
        return metrics / (cfg.epochs * cfg.minibatch_count)

    def save_checkpoint(self, path: str, robot: str, task: str = "target_reaching") -> None:
        """The current policy as a reference checkpoint (policy.cpp:220-242),
        readable by the reference's load_checkpoint / evaluate_policy."""
        sg.save_checkpoint(path, self.ref_params().double().cpu().numpy(), self.O, self.A, robot, task)

    def load_checkpoint(self, path: str) -> dict:
        """Initialise the policy from a reference checkpoint (load_checkpoint,
        policy.cpp:244-295); Adam state restarts (the reference does not store it)."""
        meta, p = sg.load_checkpoint(path)
        if (meta["obs_dim"], meta["action_dim"], meta["hidden"]) != (self.O, self.A, (256, 128, 64)):
            raise sg.ConfigError(f"checkpoint '{path}' shape {meta} does not match this trainer")
        with torch.no_grad():
            self.params[self.ref_to_pad] = torch.from_numpy(p).float().to(self.dev)
            self.adam_m.zero_()
            self.adam_v.zero_()
            self.adam_t.zero_()
            if self.mirror is not None:
                self.mirror.copy_(self.params)
        self.policy.load_params(self.ref_params())
        return meta

    def iterate(self) -> dict:
        self.rollout()
        self.gae()
        m = self.update()
        self.iteration += 1
        # one synchronisation per iteration: device-detected env errors
        # (non-finite action / reward, goal-sampling exhaustion) raise here,
        # and a non-finite minibatch loss or gradient (ppo.cpp:193-199)
        self.env.synchronize()
        s = self.stats.tolist()
        pm = m.tolist()
        nonfinite = self.grad_sq[1].item() != 0.0 or not all(math.isfinite(x) for x in pm)
        if nonfinite:
            self.grad_sq[1] = 0.0
            raise sg.SimError(f"ppo_update: non-finite loss (iteration {self.iteration}, metrics {pm})")
        return dict(iteration=self.iteration, env_steps=self.env_steps, episodes_completed=int(s[3]),
                    mean_episode_reward=s[1] / s[3] if s[3] else float("nan"),
                    mean_final_error=s[2] / s[3] if s[3] else float("nan"),
                    mean_step_reward=s[0] / (self.N * self.T), policy_loss=pm[0], value_loss=pm[1],
                    entropy=pm[2], kl=pm[3], clip_fraction=pm[4],
                    log_std_mean=float(self.params[self.ls_off: self.ls_off + self.A]
                                       .clamp(LOG_STD_MIN, LOG_STD_MAX).mean()))
