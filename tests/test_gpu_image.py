"""GPU parity for ImageMatching (envs.cpp:269-295, 333-335, 464-473, 513-523;
renderer render.cpp:34-67) against the fp64 oracle
(tests/test_oracle_image.py pins the oracle with the reference's render tests).

Bit-exact: timed_out / terminated, step / episode counters, PCG32 streams,
the per-env scenes (fp64 draws rounded once). Tolerances: joint state and tip
as in tests/test_gpu_parity.py; image pixels 1e-3 except at silhouette /
occlusion boundaries, where a ray that grazes a sphere can hit in one
precision and miss in the other (the fp32 oracle shows ~1e-6 of the pixels
beyond 1e-3, tests/test_oracle_image.py drift figures in DESIGN.md): at most
PIXEL_FLIP_FRAC of the pixels may exceed the tolerance, and the reward may
differ by no more than those pixels' mean difference plus 2e-5.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

TOL = dict(q=1e-5, qdot=1e-4, q_target=1e-5, pos=2e-5, pixel=1e-3, reward=2e-5)
PIXEL_FLIP_FRAC = 1e-4


def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")


def _check_obs(o_dev, o_ref, A, wh, what):
    head = 3 * A + 3
    tol = np.concatenate([np.full(A, TOL["q"]), np.full(A, TOL["qdot"]), np.full(3, TOL["pos"]),
                          np.full(A, TOL["q_target"])])
    assert (np.abs(o_dev[:, :head] - o_ref[:, :head]) <= tol).all(), f"{what}: joint/tip columns"
    d = np.abs(o_dev[:, head:] - o_ref[:, head:])
    flips = int((d > TOL["pixel"]).sum())
    assert flips <= PIXEL_FLIP_FRAC * d.size + 1, f"{what}: {flips} pixels beyond {TOL['pixel']}"
    return d


def _run(sg, oracle, robot, n, steps, seed):
    _cuda()
    m = oracle.resolve_robot(robot)
    ref = oracle.Env(oracle.env_config(n_envs=n, seed=seed, task=oracle.IMAGE_MATCHING), m)
    env = sg.VecTaskEnv(robots=(robot,), n_envs=n, seed=seed, task="image_matching")
    A, O = env.action_dim, env.obs_dim
    assert O == ref.obs_dim == 3 * A + 3 + 2 * 1024
    wh = 1024
    o_ref = ref.reset()
    obs = env.reset()
    torch.cuda.synchronize()
    _check_obs(obs.cpu().numpy(), o_ref, A, wh, "reset")
    sc = env.images()["scenes"].cpu().numpy()[:, :15].reshape(n, 3, 5)
    np.testing.assert_array_equal(sc, ref.images()["scenes"].astype(np.float32))
    ar = oracle.make_stream(seed, 0xAC7104)
    for s in range(steps):
        a32 = oracle.fill_uniform_actions(ar, n, A).astype(np.float32)
        res = env.step(torch.from_numpy(a32).cuda())
        ref.step(a32.astype(np.float64))
        torch.cuda.synchronize()
        r = ref.result()
        np.testing.assert_array_equal(res.timed_out.cpu().numpy(), r["timed_out"], err_msg=f"timed_out @{s}")
        np.testing.assert_array_equal(res.terminated.cpu().numpy(), r["terminated"])
        st, c = env.state(), ref.counters()
        for k in ("step_count", "episode_count"):
            np.testing.assert_array_equal(st[k].cpu().numpy(), c[k], err_msg=f"{k} @{s}")
        np.testing.assert_array_equal(st["rng_state"].cpu().numpy(), ref.rng()[0], err_msg=f"rng @{s}")
        sr = ref.state()
        for k in ("q", "qdot", "q_target"):
            err = np.abs(st[k].cpu().numpy().T - sr[k]).max()
            assert err <= TOL[k], f"{k} err {err:.3e} @{s}"
        assert np.abs(st["tips"].cpu().numpy().T - sr["tips"]).max() <= TOL["pos"]
        o_ref, t_ref = ref.obs()
        o_dev = res.observations.cpu().numpy()
        _check_obs(o_dev, o_ref, A, wh, f"obs @{s}")
        ended = r["timed_out"].astype(bool)
        t_dev = res.terminal_observations.cpu().numpy()
        if ended.any():
            _check_obs(t_dev[ended], t_ref[ended], A, wh, f"terminal obs @{s}")
            np.testing.assert_array_equal(env.images()["scenes"].cpu().numpy()[:, :15].reshape(n, 3, 5),
                                          ref.images()["scenes"].astype(np.float32))
        # reward = -mean |current - target| of the pre-reset row (envs.cpp:513-523):
        # within the rows' image differences of the oracle's, and internally
        # consistent on the device
        pre_dev = np.where(ended[:, None], t_dev, o_dev)
        pre_ref = np.where(ended[:, None], t_ref, o_ref)
        h0 = 3 * A + 3
        bound = np.abs(pre_dev[:, h0:] - pre_ref[:, h0:]).sum(1) / wh
        rew = res.rewards.cpu().numpy()
        assert (np.abs(rew - r["rewards"]) <= bound + TOL["reward"]).all(), f"reward @{s}"
        np.testing.assert_allclose(rew, -np.abs(pre_dev[:, h0 + wh:] - pre_dev[:, h0:h0 + wh]).mean(1), atol=1e-6)
        np.testing.assert_allclose(res.task_error.cpu().numpy(), -rew, atol=0)
    return env, ref


def test_image_matching_psm(sg, oracle):
    """PSM camera ImageMatching, 64 envs, 310 steps: one synchronized reset
    burst (new scene, target view and stream state per env)."""
    env, ref = _run(sg, oracle, "psm", 64, 310, seed=0)
    assert (ref.counters()["episode_count"] == 1).all()


def test_image_matching_ecm(sg, oracle):
    """ECM (the endoscope: camera looks down its tip -z axis), 48 envs, 305 steps."""
    _run(sg, oracle, "ecm", 48, 305, seed=2)


def test_image_matching_fused_steps_bench_stream_and_host_step(sg, oracle):
    """K fused steps == K single steps bit for bit (episode_len 7, ragged CTA),
    the bench stream bit-exact, and sg_env_step_host == sg_env_step."""
    _cuda()
    n = 300
    kw = dict(robots=("star",), n_envs=n, seed=5, episode_len=7, task="image_matching")
    a, b = sg.VecTaskEnv(**kw), sg.VecTaskEnv(**kw)
    a.reset(); b.reset()
    a.bench_begin(5); b.bench_begin(5)
    ar = oracle.make_stream(5, 0xAC7104)
    for _ in range(2):
        a.bench_step(1)
        np.testing.assert_array_equal(a.bench_actions().cpu().numpy(),
                                      oracle.fill_uniform_actions(ar, n, 8).astype(np.float32))
    b.bench_step(2)
    for launch in (9, 5):
        for _ in range(launch):
            a.bench_step(1)
        b.bench_step(launch)
        torch.cuda.synchronize()
        sa, sb = a.state(), b.state()
        for k in ("q", "qdot", "q_target", "tips", "step_count", "episode_count", "rng_state"):
            assert torch.equal(sa[k], sb[k]), k
        assert torch.equal(a.images()["target"], b.images()["target"])
        ra, rb = a._result(), b._result()
        assert torch.equal(ra.observations, rb.observations)
        ended = ra.timed_out.bool()
        assert torch.equal(ra.terminal_observations[ended], rb.terminal_observations[ended])
    d, h = sg.VecTaskEnv(**kw), sg.VecTaskEnv(**kw)
    d.reset(); h.reset()
    rng = np.random.default_rng(1)
    for s in range(8):
        act = rng.uniform(-1.2, 1.2, (n, 8)).astype(np.float32)
        res = d.step(torch.from_numpy(act).cuda())
        out = h.step_host(act)
        np.testing.assert_array_equal(out["observations"], res.observations.cpu().numpy())
        np.testing.assert_array_equal(out["rewards"], res.rewards.cpu().numpy())
        assert out["action_saturations"] == int(((act < -1) | (act > 1)).sum())
        if out["timed_out"].any():
            e = out["timed_out"].astype(bool)
            np.testing.assert_array_equal(out["terminal_observations"][e], res.terminal_observations.cpu().numpy()[e])
    with pytest.raises(sg.ConfigError, match="width and height"):
        sg.VecTaskEnv(robots=("psm",), n_envs=4, task="image_matching", render_width=4)
    with pytest.raises(sg.ConfigError, match="exactly 1 robot"):
        sg.VecTaskEnv(robots=("psm", "ecm"), n_envs=4, task="image_matching")


def test_image_matching_sharded_rows(sg, oracle):
    """row_offset shards are bit-identical to the rows of one env (streams by
    global row, bench stream by global index) across a reset burst."""
    _cuda()
    kw = dict(robots=("psm",), seed=3, task="image_matching", episode_len=40)
    full = sg.VecTaskEnv(n_envs=96, **kw)
    part = sg.VecTaskEnv(n_envs=40, row_offset=56, **kw)
    full.reset(); part.reset()
    full.bench_begin(3); part.bench_begin(3, global_n_envs=96)
    full.bench_step(45); part.bench_step(45)
    torch.cuda.synchronize()
    assert torch.equal(full._result().observations[56:], part._result().observations)
    assert torch.equal(full.images()["target"][56:], part.images()["target"])
    assert torch.equal(full.state()["rng_state"][56:], part.state()["rng_state"])


@pytest.mark.parametrize("w,h,fov", [(48, 40, 0.9), (64, 64, 1.2)])
def test_image_matching_render_configs(sg, oracle, w, h, fov):
    """Non-default RenderConfig (render.hpp:31-38): 48 x 40 runs the
    lane-per-column path (128 % w != 0), 64 x 64 the 4-pixels-per-lane path;
    images within the pixel tolerance of the oracle over a reset burst."""
    _cuda()
    m = oracle.resolve_robot("ecm")
    n = 24
    rc = dict(render_w=w, render_h=h, render_fov=fov, render_near=0.01, render_far=1.5)
    ref = oracle.Env(oracle.env_config(n_envs=n, seed=4, task=oracle.IMAGE_MATCHING, episode_len=30, **rc), m)
    env = sg.VecTaskEnv(robots=("ecm",), n_envs=n, seed=4, task="image_matching", episode_len=30,
                        render_width=w, render_height=h, render_fov=fov, render_near=0.01, render_far=1.5)
    A = env.action_dim
    assert env.obs_dim == ref.obs_dim == 3 * A + 3 + 2 * w * h
    o_ref = ref.reset()
    _check_obs(env.reset().cpu().numpy(), o_ref, A, w * h, "reset")
    ar = oracle.make_stream(4, 0xAC7104)
    for s in range(35):
        a32 = oracle.fill_uniform_actions(ar, n, A).astype(np.float32)
        res = env.step(torch.from_numpy(a32).cuda())
        ref.step(a32.astype(np.float64))
        r = ref.result()
        np.testing.assert_array_equal(res.timed_out.cpu().numpy(), r["timed_out"])
        _check_obs(res.observations.cpu().numpy(), ref.obs()[0], A, w * h, f"obs @{s}")
        assert np.abs(res.rewards.cpu().numpy() - r["rewards"]).max() < 5e-3
