"""GPU parity for MultiToolReaching (envs.cpp:101-116, 304-360, 540-593; SURVEY
§8f rank 3): the sm_100a multi-tool kernels behind the C-ABI vs the fp64
oracle (tests/test_oracle_multitool.py pins the oracle against an independent
restatement).

Bit-exact: terminated / timed_out, step / hold / episode counters, every
tool's PCG32 stream. Tolerance (per step): joint state as in
tests/test_gpu_parity.py, tips / goals / observation positions 2e-5 m,
reward / task_error 2e-5 — except that a collision penalty may flip when the
oracle's minimum tip separation lies within 1e-5 m of the threshold (fp32 vs
fp64 distance), which the test checks explicitly.
"""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

TOL = dict(q=1e-5, qdot=1e-4, q_target=1e-5, pos=2e-5, reward=2e-5)


def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")


def _min_sep(obs, A, T):
    tips = obs[:, 2 * A:2 * A + 3 * T].reshape(-1, T, 3)
    sep = np.full(len(obs), np.inf)
    for t in range(T):
        for u in range(t + 1, T):
            sep = np.minimum(sep, np.linalg.norm(tips[:, t] - tips[:, u], axis=1))
    return sep


def _obs_tol(A, T):
    return np.concatenate([np.full(A, TOL["q"]), np.full(A, TOL["qdot"]), np.full(3 * T, TOL["pos"]),
                           np.full(A, TOL["q_target"]), np.full(3 * T, TOL["pos"])])


def _run(sg, oracle, robots, n, steps, seed, **kw):
    _cuda()
    ms = [oracle.resolve_robot(r) for r in robots]
    T = len(ms)
    ref = oracle.MultiToolEnv(oracle.env_config(n_envs=n, seed=seed, task=oracle.MULTI_TOOL, **kw), ms)
    env = sg.VecTaskEnv(robots=robots, n_envs=n, seed=seed, task="multi_tool_reaching", **kw)
    A, O = env.action_dim, env.obs_dim
    assert (A, O) == (ref.action_dim, ref.obs_dim)
    o_ref = ref.reset()
    obs = env.reset()
    torch.cuda.synchronize()
    otol = _obs_tol(A, T)
    assert (np.abs(obs.cpu().numpy() - o_ref) <= otol).all()
    ar = oracle.make_stream(seed, 0xAC7104)
    thr, pen = kw.get("collision_threshold", 0.01), kw.get("collision_penalty", 1.0)
    flips = collisions = 0
    for s in range(steps):
        a32 = oracle.fill_uniform_actions(ar, n, A).astype(np.float32)
        res = env.step(torch.from_numpy(a32).cuda())
        ref.step(a32.astype(np.float64))
        torch.cuda.synchronize()
        r = ref.result()
        np.testing.assert_array_equal(res.terminated.cpu().numpy(), r["terminated"], err_msg=f"terminated @{s}")
        np.testing.assert_array_equal(res.timed_out.cpu().numpy(), r["timed_out"], err_msg=f"timed_out @{s}")
        st, c = env.state(), ref.counters()
        for k in ("step_count", "hold_count", "episode_count"):
            np.testing.assert_array_equal(st[k].cpu().numpy(), c[k], err_msg=f"{k} @{s}")
        rs, ri = ref.rng()
        np.testing.assert_array_equal(st["rng_state"].cpu().numpy(), rs, err_msg=f"rng @{s}")
        np.testing.assert_array_equal(st["rng_inc"].cpu().numpy(), ri)
        sr = ref.state()
        for k in ("q", "qdot", "q_target"):
            err = np.abs(st[k].cpu().numpy().T - sr[k]).max()
            assert err <= TOL[k], f"{k} err {err:.3e} @{s}"
        for k in ("tips", "goals"):
            err = np.abs(st[k].cpu().numpy().T - sr[k]).max()
            assert err <= TOL["pos"], f"{k} err {err:.3e} @{s}"
        o_ref, t_ref = ref.obs()
        o_dev = res.observations.cpu().numpy()
        bad = np.abs(o_dev - o_ref) > otol
        assert not bad.any(), f"obs @{s}: {np.argwhere(bad)[:4]}"
        ended = (r["terminated"] | r["timed_out"]).astype(bool)
        if ended.any():
            bad = np.abs(res.terminal_observations.cpu().numpy()[ended] - t_ref[ended]) > otol
            assert not bad.any(), f"terminal obs @{s}"
        pre = np.where(ended[:, None], t_ref, o_ref)  # pre-reset observation rows
        sep = _min_sep(pre, A, T)
        collisions += int((sep < thr).sum())
        d = res.rewards.cpu().numpy() - r["rewards"]
        off = np.abs(d) > TOL["reward"]
        if off.any():  # only collision-threshold ties may differ, by exactly the penalty
            assert (np.abs(np.abs(d[off]) - pen) <= TOL["reward"]).all(), f"reward @{s}: {d[off]}"
            assert (np.abs(sep[off] - thr) < 1e-5).all(), f"reward flip away from the threshold @{s}"
            flips += int(off.sum())
        err = np.abs(res.task_error.cpu().numpy() - r["task_error"]).max()
        assert err <= TOL["reward"], f"task_error {err:.3e} @{s}"
    return env, ref, collisions, flips


def test_bimanual_psm_reach(sg, oracle):
    """Two PSMs on the default bases (+-0.7 r along x), 64 envs, 320 steps:
    one reset burst; both tools' streams bit-exact."""
    env, ref, _, _ = _run(sg, oracle, ("psm", "psm"), 64, 320, seed=1)
    assert (ref.counters()["episode_count"] == 1).all()


def test_trimanual_psm_psm_ecm_camera(sg, oracle):
    """PSM + PSM + ECM camera (third base behind the scene, pitched 0.9 rad):
    the camera goal is the other tips' midpoint, its reward the view penalty
    (angle between the camera's -z axis and the midpoint); collision penalty
    threshold raised to 0.2 m so it fires."""
    env, ref, collisions, flips = _run(sg, oracle, ("psm", "psm", "ecm"), 64, 310, seed=3,
                                       collision_threshold=0.2)
    assert collisions > 0
    assert flips <= 2


def test_mixed_chains_custom_bases(sg, oracle):
    """STAR (8 DoF) + PSM + ECM on caller-supplied bases (one rotated about z):
    workspace centres through the bases and parity over an episode boundary."""
    _cuda()
    c, s = math.cos(0.2), math.sin(0.2)
    bases = np.array([[-0.3, 0.0, -0.8, 1, 0, 0, 0], [0.1, 0.05, 0.0, c, 0, 0, s], [0.0, -0.3, 0.075, 1, 0, 0, 0]])
    ms = [oracle.resolve_robot(r) for r in ("star", "psm", "ecm")]
    ref = oracle.MultiToolEnv(oracle.env_config(n_envs=40, seed=8, task=oracle.MULTI_TOOL, episode_len=50), ms,
                              bases=bases)
    env = sg.VecTaskEnv(robots=("star", "psm", "ecm"), n_envs=40, seed=8, task="multi_tool_reaching",
                        episode_len=50, tool_bases=bases)
    centers, b, dofs = env.tools()
    rc, _, rb = ref.workspace()
    np.testing.assert_allclose(centers, rc, atol=1e-15)
    np.testing.assert_array_equal(b, rb)
    assert dofs == [8, 7, 6]
    o_ref = ref.reset()
    obs = env.reset()
    A, T = env.action_dim, 3
    assert (np.abs(obs.cpu().numpy() - o_ref) <= _obs_tol(A, T)).all()
    ar = oracle.make_stream(8, 0xAC7104)
    for s in range(120):
        a32 = oracle.fill_uniform_actions(ar, 40, A).astype(np.float32)
        res = env.step(torch.from_numpy(a32).cuda())
        ref.step(a32.astype(np.float64))
        r = ref.result()
        np.testing.assert_array_equal(res.timed_out.cpu().numpy(), r["timed_out"])
        np.testing.assert_array_equal(env.state()["rng_state"].cpu().numpy(), ref.rng()[0])
        assert (np.abs(res.observations.cpu().numpy() - ref.obs()[0]) <= _obs_tol(A, T)).all(), s
        np.testing.assert_allclose(res.rewards.cpu().numpy(), r["rewards"], atol=TOL["reward"])
    assert (ref.counters()["episode_count"] == 2).all()


def test_multitool_fused_steps_and_bench_stream(sg, oracle):
    """Bench stream rows of A = 20 draws (bench.cpp:31-35) bit-exact, and K
    fused steps == K single-step launches bit for bit (episode_len 7: resets
    inside and across launches; 1000 envs: ragged last warp)."""
    _cuda()
    n = 1000
    kw = dict(robots=("psm", "psm", "ecm"), n_envs=n, seed=2, episode_len=7, task="multi_tool_reaching")
    a, b = sg.VecTaskEnv(**kw), sg.VecTaskEnv(**kw)
    a.reset(); b.reset()
    a.bench_begin(2); b.bench_begin(2)
    ar = oracle.make_stream(2, 0xAC7104)
    for s in range(3):
        a.bench_step(1)
        np.testing.assert_array_equal(a.bench_actions().cpu().numpy(),
                                      oracle.fill_uniform_actions(ar, n, 20).astype(np.float32))
    b.bench_step(3)
    for launch in (9, 4):
        for _ in range(launch):
            a.bench_step(1)
        b.bench_step(launch)
        torch.cuda.synchronize()
        sa, sb = a.state(), b.state()
        for k in ("q", "qdot", "q_target", "goals", "tips", "step_count", "episode_count", "rng_state"):
            assert torch.equal(sa[k], sb[k]), k
        ra, rb = a._result(), b._result()
        assert torch.equal(ra.observations, rb.observations)
        ended = (ra.terminated | ra.timed_out).bool()
        assert torch.equal(ra.terminal_observations[ended], rb.terminal_observations[ended])


def test_multitool_host_step_and_errors(sg, oracle):
    """sg_env_step_host == sg_env_step for the multi-tool env (terminal rows on
    ended steps, saturation count); non-finite actions raise SimError; config
    errors of the reference (robot count, tool_bases count)."""
    _cuda()
    n = 96
    kw = dict(robots=("psm", "psm"), n_envs=n, seed=6, episode_len=3, task="multi_tool_reaching")
    d, h = sg.VecTaskEnv(**kw), sg.VecTaskEnv(**kw)
    d.reset(); h.reset()
    rng = np.random.default_rng(0)
    for s in range(7):
        a = rng.uniform(-1.3, 1.3, (n, 14)).astype(np.float32)
        res = d.step(torch.from_numpy(a).cuda())
        out = h.step_host(a)
        np.testing.assert_array_equal(out["observations"], res.observations.cpu().numpy())
        np.testing.assert_array_equal(out["rewards"], res.rewards.cpu().numpy())
        np.testing.assert_array_equal(out["timed_out"], res.timed_out.cpu().numpy())
        assert out["action_saturations"] == int(((a < -1) | (a > 1)).sum())
        if out["timed_out"].any():
            ended = out["timed_out"].astype(bool)
            np.testing.assert_array_equal(out["terminal_observations"][ended],
                                          res.terminal_observations.cpu().numpy()[ended])
    assert h.host_counters()[0] == 2 * n
    bad = np.zeros((n, 14), np.float32)
    bad[5, 9] = np.nan
    with pytest.raises(sg.SimError, match="non-finite action"):
        h.step_host(bad)
    with pytest.raises(sg.ConfigError, match="requires >= 2 robots"):
        sg.VecTaskEnv(robots=("psm",), n_envs=4, task="multi_tool_reaching")
    with pytest.raises(sg.ConfigError, match="one entry per robot"):
        sg.VecTaskEnv(robots=("psm", "psm"), n_envs=4, task="multi_tool_reaching", tool_bases=np.zeros((3, 7)))
    with pytest.raises(sg.ConfigError, match="at most 4"):
        sg.VecTaskEnv(robots=("psm",) * 5, n_envs=4, task="multi_tool_reaching")


def test_multitool_sharded_rows_and_cpp_example(sg, oracle, tmp_path):
    """row_offset shards (per-tool streams seeded by global row) are
    bit-identical to the rows of one env; the C++ drop-in example runs."""
    _cuda()
    kw = dict(robots=("psm", "psm", "ecm"), seed=4, task="multi_tool_reaching")
    full = sg.VecTaskEnv(n_envs=256, **kw)
    part = sg.VecTaskEnv(n_envs=128, row_offset=128, **kw)
    full.reset(); part.reset()
    full.bench_begin(4); part.bench_begin(4, global_n_envs=256)
    full.bench_step(310); part.bench_step(310)
    torch.cuda.synchronize()
    assert torch.equal(full._result().observations[128:], part._result().observations)
    assert torch.equal(full.state()["rng_state"][:, 128:], part.state()["rng_state"])
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    libdir = os.path.dirname(sg.lib_path())
    exe = str(tmp_path / "multitool_cpp")
    r = subprocess.run(["g++", "-std=c++17", "-O2", "-I", os.path.join(root, "include"),
                        os.path.join(root, "examples", "multitool_cpp.cpp"), f"-L{libdir}", "-lsg_env",
                        f"-Wl,-rpath,{libdir}", "-o", exe], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    run = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert run.returncode == 0, run.stdout + run.stderr
    assert "tools 3  action_dim 20  obs_dim 78" in run.stdout and run.stdout.count("mean reward") == 10


@pytest.mark.parametrize("mode", ["velocity", "torque"])
def test_multitool_control_modes(sg, oracle, mode):
    """Velocity / torque control (dynamics.cpp:141-150) on every tool with
    adversarial actions in [-2, 2]: saturation counts exact, limits hold,
    joint state within 10x the step tolerance of the oracle over 120 steps."""
    _cuda()
    robots = ("psm", "psm", "ecm")
    ms = [oracle.resolve_robot(r) for r in robots]
    dyns = []
    for m in ms:
        d = oracle.default_dynamics(m)
        d.control_mode = {"velocity": 1, "torque": 2}[mode]
        dyns.append(d)
    n = 48
    ref = oracle.MultiToolEnv(oracle.env_config(n_envs=n, seed=12, task=oracle.MULTI_TOOL), ms, dyns=dyns)
    env = sg.VecTaskEnv(robots=robots, n_envs=n, seed=12, task="multi_tool_reaching",
                        dynamics=dict(control_mode=mode))
    ref.reset(); env.reset()
    rng = oracle.make_stream(3, 0)
    f32 = lambda v: np.float64(np.float32(v))
    lo = np.concatenate([[f32(m.dof_joint(d).limit_lo) for d in range(m.dof)] for m in ms])
    hi = np.concatenate([[f32(m.dof_joint(d).limit_hi) for d in range(m.dof)] for m in ms])
    for s in range(120):
        a = (2.0 * oracle.fill_uniform_actions(rng, n, 20)).astype(np.float32)
        hr = env.step_host(a)
        ref.step(a.astype(np.float64))
        assert hr["action_saturations"] == ref.result()["saturations"]
        q = env.state()["q"].cpu().numpy().T.astype(np.float64)
        assert (q >= lo).all() and (q <= hi).all()
        assert np.abs(q - ref.state()["q"]).max() <= 1e-4, s
        np.testing.assert_array_equal(hr["timed_out"], ref.result()["timed_out"])
