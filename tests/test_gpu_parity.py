"""GPU parity: the sm_100a step behind the C-ABI vs the fp64 CPU oracle.

Contract (north_star): reset masks, termination/timeout
flags, step/hold/episode counters, waypoint indices and per-env RNG states are
BIT-EXACT; joint state, tips, observations and rewards agree within the fp32
tolerances below on every step of a fixed horizon. The tolerances are set from
the intrinsic fp32-vs-fp64 drift the oracle measures on the same inputs
(tests/test_oracle_env.py::test_fp32_drift_bounds).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

TOL = dict(q=1e-5, qdot=1e-4, q_target=1e-5, tips=2e-5, goals=1e-6, obs_pos=2e-5, reward=2e-5)


def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")


def _soa(t):  # device SoA (dof x n) -> host (n x dof)
    return t.detach().cpu().numpy().T.astype(np.float64)


def _run_pair(sg, oracle, robot, task, n, steps, seed=0, sigma=0.05, check_every=1, actions_fn=None, tol=None,
              mode="position", per_step=None):
    """Step the device env and the fp64 oracle with the same actions; compare.
    mode: control mode (dynamics.cpp:133-185); per_step(s, env, ref, res, a32):
    extra checks after every step."""
    _cuda()
    TOL = dict(globals()["TOL"], **(tol or {}))
    m = oracle.resolve_robot(robot)
    ocfg = oracle.env_config(n_envs=n, seed=seed, task=task, goal_sigma=sigma)
    dyn = oracle.default_dynamics(m)
    dyn.control_mode = {"position": 0, "velocity": 1, "torque": 2}[mode]
    ref = oracle.Env(ocfg, m, dyn)
    ref.reset()
    env = sg.VecTaskEnv(robots=(robot,), n_envs=n, seed=seed, task=task, goal_sigma=sigma,
                        dynamics=dict(control_mode=mode))
    obs = env.reset()
    torch.cuda.synchronize()
    A, O = env.action_dim, env.obs_dim
    o_ref = ref.obs()[0]
    _compare_obs(obs.cpu().numpy(), o_ref, A)
    ar = oracle.make_stream(seed, 0xAC7104)
    worst = {}
    for s in range(steps):
        a = actions_fn(s) if actions_fn else oracle.fill_uniform_actions(ar, n, A)
        a32 = a.astype(np.float32)
        res = env.step(torch.from_numpy(a32).cuda())
        ref.step(a32.astype(np.float64))
        if per_step is not None:
            per_step(s, env, ref, res, a32)
        if s % check_every and s != steps - 1:
            continue
        torch.cuda.synchronize()
        r = ref.result()
        # ---- bit-exact --------------------------------------------------------
        np.testing.assert_array_equal(res.terminated.cpu().numpy(), r["terminated"], err_msg=f"terminated @{s}")
        np.testing.assert_array_equal(res.timed_out.cpu().numpy(), r["timed_out"], err_msg=f"timed_out @{s}")
        st = env.state()
        c = ref.counters()
        np.testing.assert_array_equal(st["step_count"].cpu().numpy(), c["step_count"], err_msg=f"step_count @{s}")
        np.testing.assert_array_equal(st["hold_count"].cpu().numpy(), c["hold_count"], err_msg=f"hold @{s}")
        np.testing.assert_array_equal(st["episode_count"].cpu().numpy(), c["episode_count"], err_msg=f"episodes @{s}")
        if task == oracle.PATH_FOLLOWING:
            np.testing.assert_array_equal(st["waypoint_idx"].cpu().numpy(), c["waypoint_idx"], err_msg=f"wp idx @{s}")
            np.testing.assert_array_equal(st["waypoint_len"].cpu().numpy(), c["waypoint_len"], err_msg=f"wp len @{s}")
        rs, ri = ref.rng()
        np.testing.assert_array_equal(st["rng_state"].cpu().numpy(), rs, err_msg=f"rng @{s}")
        np.testing.assert_array_equal(st["rng_inc"].cpu().numpy(), ri)
        # ---- tolerance ---------------------------------------------------------
        sr = ref.state()
        for k in ("q", "qdot", "q_target"):
            err = np.abs(_soa(st[k]) - sr[k]).max()
            worst[k] = max(worst.get(k, 0.0), err)
            assert err <= TOL[k], f"{robot} {k} err {err:.3e} @ step {s}"
        for k in ("tips", "goals"):
            err = np.abs(_soa(st[k]) - sr[k]).max()
            worst[k] = max(worst.get(k, 0.0), err)
            assert err <= TOL[k], f"{robot} {k} err {err:.3e} @ step {s}"
        err = np.abs(res.rewards.cpu().numpy() - r["rewards"]).max()
        worst["reward"] = max(worst.get("reward", 0.0), err)
        assert err <= TOL["reward"]
        err = np.abs(res.task_error.cpu().numpy() - r["task_error"]).max()
        assert err <= TOL["reward"]
        o_dev = res.observations.cpu().numpy()
        o_ref, t_ref = ref.obs()
        _compare_obs(o_dev, o_ref, A, TOL)
        ended = (r["terminated"] | r["timed_out"]).astype(bool)
        if ended.any():
            _compare_obs(res.terminal_observations.cpu().numpy()[ended], t_ref[ended], A, TOL)
    return env, ref, worst


def _compare_obs(o_dev, o_ref, A, TOL=TOL):
    # layout [q | qdot | tip | q_target | goal] (envs.cpp:166-192)
    tol = np.concatenate([np.full(A, TOL["q"]), np.full(A, TOL["qdot"]), np.full(3, TOL["obs_pos"]),
                          np.full(A, TOL["q_target"]), np.full(3, TOL["obs_pos"])])
    err = np.abs(o_dev.astype(np.float64) - o_ref)
    bad = err > tol
    assert not bad.any(), f"obs mismatch at {np.argwhere(bad)[:5]} max err {err.max():.3e}"


def test_config1_psm_reach_1000_steps(sg, oracle):
    """BASELINE config 1: PSM reach, 64 envs, 1000 steps (+ warm-up), seed 0,
    random actions from make_stream(0, 0xac7104) — three synchronized reset
    bursts at steps 300/600/900."""
    env, ref, worst = _run_pair(sg, oracle, "psm", oracle.TARGET_REACHING, 64, 1001)
    c = ref.counters()
    assert (c["episode_count"] == 3).all()
    assert ref.goal_draws() == 264  # 256 resets + 8 rejections (survey probe, Appendix E)


def test_active_tracking_drifting_goals(sg, oracle):
    """ActiveTracking (envs.cpp:493-512): the goal drifts after
    scoring with velocity noise from the env stream (6 u32 per env-step) and
    both clamps active; streams, flags and counters bit-exact, goals within
    2e-5 m (fp32 random walk vs the oracle's fp64) over two reset bursts."""
    env, ref, worst = _run_pair(sg, oracle, "psm", oracle.ACTIVE_TRACKING, 64, 650, seed=5,
                                tol=dict(goals=2e-5))
    c = ref.counters()
    assert (c["episode_count"] == 2).all() and (c["hold_count"] == 0).all()  # bursts at 300, 600
    assert worst["goals"] > 0.0


@pytest.mark.parametrize("robot,task,sigma", [("psm", 0, 0.05), ("ecm", 0, 0.05), ("star", 3, 0.15)])
@pytest.mark.parametrize("n", [1, 31, 33])
def test_tiny_and_ragged_env_counts(sg, oracle, robot, task, sigma, n):
    """One env, one short team, and one full team + a 1-env team (the ragged
    last team computes on padding lanes and masks only its stores): every
    chain, across the step-300 reset burst, against the fp64 oracle."""
    _run_pair(sg, oracle, robot, task, n, 305, seed=9, sigma=sigma, check_every=4)


def test_ecm_reach(sg, oracle):
    _run_pair(sg, oracle, "ecm", oracle.TARGET_REACHING, 96, 650, seed=3)


def test_star_path_following(sg, oracle):
    env, ref, worst = _run_pair(sg, oracle, "star", oracle.PATH_FOLLOWING, 48, 620, seed=1, sigma=0.15)
    # waypoint tables: fp64 arithmetic on both sides, rounded to fp32 on the device
    st = env.state()
    wl = st["waypoint_len"].cpu().numpy()
    wps = st["waypoints"].cpu().numpy()
    for row in range(env.n_envs):
        ref_w = ref.waypoints(row)
        assert len(ref_w) == wl[row]
        np.testing.assert_array_equal(wps[row, : wl[row]], ref_w.astype(np.float32))


def test_path_following_waypoint_advance(sg, oracle):
    """Drive the tip onto its path with a large success radius so waypoint
    indices advance and episodes terminate by goal; indices stay bit-exact."""
    _cuda()
    m = oracle.resolve_robot("star")
    n = 32
    kw = dict(n_envs=n, seed=5, task=oracle.PATH_FOLLOWING, goal_sigma=0.15, success_radius=0.25)
    ref = oracle.Env(oracle.env_config(**kw), m)
    ref.reset()
    env = sg.VecTaskEnv(robots=("star",), **kw)
    env.reset()
    ar = oracle.make_stream(5, 0xAC7104)
    advanced = 0
    for s in range(400):
        a = (0.05 * oracle.fill_uniform_actions(ar, n, m.dof)).astype(np.float32)
        res = env.step(torch.from_numpy(a).cuda())
        ref.step(a.astype(np.float64))
        c = ref.counters()
        st = env.state()
        np.testing.assert_array_equal(st["waypoint_idx"].cpu().numpy(), c["waypoint_idx"], err_msg=f"@{s}")
        np.testing.assert_array_equal(res.terminated.cpu().numpy(), ref.result()["terminated"], err_msg=f"@{s}")
        advanced += int((c["waypoint_idx"] > 0).sum())
    assert advanced > 0


def test_target_reaching_terminations(sg, oracle):
    """Large success radius: hold counters run up to success_hold and episodes
    terminate by goal; terminated flags, holds and resets stay bit-exact."""
    _cuda()
    m = oracle.resolve_robot("psm")
    n = 64
    kw = dict(n_envs=n, seed=9, success_radius=0.06, success_hold=3)
    ref = oracle.Env(oracle.env_config(**kw), m)
    ref.reset()
    env = sg.VecTaskEnv(robots=("psm",), **kw)
    env.reset()
    zeros = np.zeros((n, m.dof), np.float32)
    terms = 0
    for s in range(200):
        res = env.step(torch.from_numpy(zeros).cuda())
        ref.step(zeros.astype(np.float64))
        r = ref.result()
        np.testing.assert_array_equal(res.terminated.cpu().numpy(), r["terminated"], err_msg=f"@{s}")
        np.testing.assert_array_equal(env.state()["hold_count"].cpu().numpy(), ref.counters()["hold_count"])
        np.testing.assert_array_equal(env.state()["rng_state"].cpu().numpy(), ref.rng()[0])
        terms += int(r["terminated"].sum())
    assert terms > 0


def test_bench_action_stream_bit_exact(sg, oracle):
    """Device jump-ahead generator == the reference's serial fill
    (bench.cpp:31-35) rounded to fp32, across steps and with sharding."""
    _cuda()
    n, A = 300, 7
    ar = oracle.make_stream(11, 0xAC7104)
    expected = [oracle.fill_uniform_actions(ar, n, A).astype(np.float32) for _ in range(4)]
    env = sg.VecTaskEnv(robots=("psm",), n_envs=n, seed=11)
    env.reset()
    env.bench_begin(11, first_step=0)
    for s in range(4):
        env.bench_step(1)
        np.testing.assert_array_equal(env.bench_actions().cpu().numpy(), expected[s])
    # shard: rows [100, 300) of the same global stream, starting at step 2
    shard = sg.VecTaskEnv(robots=("psm",), n_envs=200, seed=11, row_offset=100)
    shard.reset()
    shard.bench_begin(11, first_step=2, global_n_envs=n)
    shard.bench_step(1)
    np.testing.assert_array_equal(shard.bench_actions().cpu().numpy(), expected[2][100:])


@pytest.mark.parametrize("layout", ["legacy", "packed"])
def test_config1_through_the_drivers_k20_fused_launches(sg, oracle, layout):
    """BASELINE config 1 on the exact path the driver's headline times:
    bench.py --steps 20 runs sg_env_bench_step launches of K = 20 fused steps
    with in-kernel actions. 64 PSM envs, seed 0: the warm-up step, then 50
    launches of 20 steps (1001 steps, three synchronized reset bursts at
    300 / 600 / 900) against the fp64 oracle fed the reference's serial
    action stream. After every launch: flags, counters and streams bit-exact,
    state / observations / rewards within the standard tolerances."""
    import os
    _cuda()
    n, seed = 64, 0
    m = oracle.resolve_robot("psm")
    ref = oracle.Env(oracle.env_config(n_envs=n, seed=seed), m)
    ref.reset()
    os.environ["SG_TEAM_LAYOUT"] = layout
    try:
        env = sg.VecTaskEnv(robots=("psm",), n_envs=n, seed=seed)
    finally:
        del os.environ["SG_TEAM_LAYOUT"]
    env.reset()
    env.bench_begin(seed)
    ar = oracle.make_stream(seed, 0xAC7104)
    A = m.dof

    def ref_steps(k):
        for _ in range(k):
            ref.step(oracle.fill_uniform_actions(ar, n, A).astype(np.float32).astype(np.float64))

    env.bench_step(1)
    ref_steps(1)
    for launch in range(50):
        env.bench_step(20)
        ref_steps(20)
        torch.cuda.synchronize()
        r, st, c = ref.result(), env.state(), ref.counters()
        res = env._result()
        np.testing.assert_array_equal(res.terminated.cpu().numpy(), r["terminated"])
        np.testing.assert_array_equal(res.timed_out.cpu().numpy(), r["timed_out"])
        for k in ("step_count", "hold_count", "episode_count"):
            np.testing.assert_array_equal(st[k].cpu().numpy(), c[k], err_msg=f"{k} @ launch {launch}")
        np.testing.assert_array_equal(st["rng_state"].cpu().numpy(), ref.rng()[0])
        sr = ref.state()
        for k in ("q", "qdot", "q_target", "tips", "goals"):
            assert np.abs(_soa(st[k]) - sr[k]).max() <= TOL[k], (k, launch)
        assert np.abs(res.rewards.cpu().numpy() - r["rewards"]).max() <= TOL["reward"]
        o_ref, t_ref = ref.obs()
        _compare_obs(res.observations.cpu().numpy(), o_ref, A)
        ended = (r["terminated"] | r["timed_out"]).astype(bool)
        if ended.any():
            _compare_obs(res.terminal_observations.cpu().numpy()[ended], t_ref[ended], A)
    assert (ref.counters()["episode_count"] == 3).all()


@pytest.mark.parametrize("robot,task", [("psm", "target_reaching"), ("star", "path_following")])
def test_fused_k_steps_equal_single_steps(sg, oracle, robot, task):
    """K fused steps == K single-step launches, bit for bit. For PathFollowing
    the fused launches install precomputed reset records (path_record_kernel)
    while single steps reset inline: both must give identical state,
    waypoint tables and RNG streams (episode_len 7 -> resets inside and
    across launches, ragged team count)."""
    _cuda()
    n = 1000
    kw = dict(robots=(robot,), n_envs=n, seed=2, episode_len=7, task=task,
              goal_sigma=0.15 if robot == "star" else 0.05)
    a, b = sg.VecTaskEnv(**kw), sg.VecTaskEnv(**kw)
    a.reset(); b.reset()
    a.bench_begin(2); b.bench_begin(2)
    for launch in (20, 3, 11):
        for _ in range(launch):
            a.bench_step(1)
        b.bench_step(launch)
        torch.cuda.synchronize()
        sa, sb = a.state(), b.state()
        keys = ["q", "qdot", "q_target", "goals", "tips", "step_count", "episode_count", "rng_state"]
        if task == "path_following":
            keys += ["waypoint_idx", "waypoint_len"]
            wl = sa["waypoint_len"].cpu().numpy()
            wa, wb = sa["waypoints"].cpu().numpy(), sb["waypoints"].cpu().numpy()
            for row in range(n):
                np.testing.assert_array_equal(wa[row, : wl[row]], wb[row, : wl[row]])
        for k in keys:
            assert torch.equal(sa[k], sb[k]), k
        ra, rb = a._result(), b._result()
        assert torch.equal(ra.observations, rb.observations)
        ended = (ra.terminated | ra.timed_out).bool()
        assert torch.equal(ra.terminal_observations[ended], rb.terminal_observations[ended])


def test_sharded_rows_match_single_device(sg, oracle):
    """Rank r of a sharded job (row_offset) is bit-identical to rows of one env."""
    _cuda()
    full = sg.VecTaskEnv(robots=("psm",), n_envs=256, seed=4)
    part = sg.VecTaskEnv(robots=("psm",), n_envs=128, seed=4, row_offset=128)
    full.reset(); part.reset()
    full.bench_begin(4); part.bench_begin(4, global_n_envs=256)
    full.bench_step(350); part.bench_step(350)
    torch.cuda.synchronize()
    assert torch.equal(full._result().observations[128:], part._result().observations)
    assert torch.equal(full.state()["rng_state"][128:], part.state()["rng_state"])


@pytest.mark.parametrize("world", [2, 4])
def test_star_path_following_shards_match_single_device(sg, oracle, world):
    """BASELINE config 4 sharding: STAR PathFollowing ranks with row_offset
    (global rows [r*N, (r+1)*N), dynamics.cpp:238 streams seeded by global row)
    are bit-identical to the same rows of one device stepping world*N envs,
    through fused bench launches (reset-record kernel, two synchronized reset
    bursts: envs.cpp:241-267 paths + spline waypoint tables) and through
    caller-action steps (each rank applies its slice of the global rows)."""
    _cuda()
    N = 96
    kw = dict(robots=("star",), seed=11, task="path_following", goal_sigma=0.15)
    full = sg.VecTaskEnv(n_envs=world * N, **kw)
    parts = [sg.VecTaskEnv(n_envs=N, row_offset=r * N, **kw) for r in range(world)]
    full.reset()
    for p in parts:
        p.reset()
    full.bench_begin(11)
    for p in parts:
        p.bench_begin(11, global_n_envs=world * N)
    for k in (1, 349, 300):
        full.bench_step(k)
        for p in parts:
            p.bench_step(k)
    rng = np.random.default_rng(2)
    for _ in range(3):  # caller actions: every rank steps its rows of the global batch
        act = torch.from_numpy(rng.uniform(-1.1, 1.1, size=(world * N, 8)).astype(np.float32)).cuda()
        full.step(act)
        for r, p in enumerate(parts):
            p.step(act[r * N:(r + 1) * N].contiguous())
    torch.cuda.synchronize()
    sf, rf = full.state(), full._result()
    for r, p in enumerate(parts):
        rows = slice(r * N, (r + 1) * N)
        sp, rp = p.state(), p._result()
        for k in ("step_count", "hold_count", "episode_count", "rng_state", "waypoint_idx", "waypoint_len"):
            assert torch.equal(sf[k][rows], sp[k]), (r, k)
        for k in ("q", "qdot", "q_target", "goals", "tips"):
            assert torch.equal(sf[k][:, rows], sp[k]), (r, k)
        wl = sp["waypoint_len"].cpu().numpy()
        wf, wp = sf["waypoints"][rows].cpu().numpy(), sp["waypoints"].cpu().numpy()
        for e in range(N):
            np.testing.assert_array_equal(wf[e, : wl[e]], wp[e, : wl[e]])
        for k in ("observations", "rewards", "task_error", "terminated", "timed_out"):
            assert torch.equal(getattr(rf, k)[rows], getattr(rp, k)), (r, k)
    assert int(sf["episode_count"].min()) >= 2  # two synchronized reset bursts (steps 300 and 600)


def test_host_step_matches_device_step(sg, oracle):
    """sg_env_step_host == sg_env_step; terminal observations reach the host on
    every step where rows ended (episode_len 3 -> ends every third step)."""
    _cuda()
    n = 200
    a = sg.VecTaskEnv(robots=("ecm",), n_envs=n, seed=8, episode_len=3)
    b = sg.VecTaskEnv(robots=("ecm",), n_envs=n, seed=8, episode_len=3)
    a.reset(); b.reset()
    rng = np.random.default_rng(0)
    ends = 0
    for _ in range(7):
        act = rng.uniform(-1.5, 1.5, size=(n, 6)).astype(np.float32)
        hr = a.step_host(act)
        dr = b.step(torch.from_numpy(act).cuda())
        torch.cuda.synchronize()
        np.testing.assert_array_equal(hr["observations"], dr.observations.cpu().numpy())
        np.testing.assert_array_equal(hr["rewards"], dr.rewards.cpu().numpy())
        ended = (hr["terminated"] | hr["timed_out"]).astype(bool)
        np.testing.assert_array_equal(ended, (dr.terminated | dr.timed_out).cpu().numpy().astype(bool))
        if ended.any():
            ends += 1
            np.testing.assert_array_equal(hr["terminal_observations"][ended],
                                          dr.terminal_observations.cpu().numpy()[ended])
        assert hr["action_saturations"] == int(((act < -1) | (act > 1)).sum())
    assert ends == 2 and a.host_counters()[0] == 2 * n


def _pinned_out(n, o, offset_bytes=0):
    """StepResult host buffers in pinned memory (zero-copy path); offset_bytes
    shifts the observation buffer off 16-byte alignment (staged-copy path)."""
    def pin(shape, dt, extra=0):
        count = int(np.prod(shape))
        t = torch.empty(count * np.dtype(dt).itemsize + extra, dtype=torch.uint8).pin_memory()
        return t[extra:].numpy().view(dt).reshape(shape)
    return dict(observations=pin((n, o), np.float32, offset_bytes),
                terminal_observations=pin((n, o), np.float32), rewards=pin((n,), np.float32),
                task_error=pin((n,), np.float32), terminated=pin((n,), np.uint8), timed_out=pin((n,), np.uint8))


@pytest.mark.parametrize("robot,n", [("psm", 16384), ("ecm", 1000), ("star", 77)])
def test_host_step_zero_copy_matches_staged_and_device(sg, oracle, robot, n):
    """Pinned host buffers (kernel reads actions / writes the StepResult over
    PCIe) == pageable host buffers (staged copies) == the device step, bit for
    bit, on every field and on every step of a reset burst (episode_len 4);
    ragged team counts (n % 32 != 0) and a misaligned observation buffer."""
    _cuda()
    kw = dict(robots=(robot,), n_envs=n, seed=3, episode_len=4)
    if robot == "star":
        kw.update(task="path_following", goal_sigma=0.15)
    envs = [sg.VecTaskEnv(**kw) for _ in range(4)]
    for e in envs:
        e.reset()
    A, O = envs[0].action_dim, envs[0].obs_dim
    rng = np.random.default_rng(1)
    pinned_act = torch.empty((n, A), dtype=torch.float32).pin_memory()
    outs = [_pinned_out(n, O), None, _pinned_out(n, O, offset_bytes=4)]
    for s in range(9):
        act = rng.uniform(-1.2, 1.2, size=(n, A)).astype(np.float32)
        pinned_act.numpy()[:] = act
        res = [envs[0].step_host(pinned_act.numpy(), outs[0]), envs[1].step_host(act),
               envs[2].step_host(pinned_act.numpy(), outs[2])]
        dr = envs[3].step(torch.from_numpy(act).cuda())
        torch.cuda.synchronize()
        ended = (dr.terminated | dr.timed_out).cpu().numpy().astype(bool)
        dev = dict(observations=dr.observations, rewards=dr.rewards, task_error=dr.task_error,
                   terminated=dr.terminated, timed_out=dr.timed_out)
        for r in res:
            for k, v in dev.items():
                np.testing.assert_array_equal(r[k], v.cpu().numpy(), err_msg=f"{k} @{s}")
            if ended.any():
                np.testing.assert_array_equal(r["terminal_observations"][ended],
                                              dr.terminal_observations.cpu().numpy()[ended])
            assert r["action_saturations"] == int(((act < -1) | (act > 1)).sum())
    assert envs[0].host_counters() == envs[1].host_counters() == envs[2].host_counters()
    assert envs[0].host_counters()[0] == 2 * n


@pytest.mark.parametrize("robots,task", [(("psm",), "target_reaching"), (("psm", "psm", "ecm"), "multi_tool_reaching")])
def test_host_step_counts_only_its_own_rows(sg, oracle, robots, task):
    """A host step after device steps reports the rows that ended and the
    saturated entries of THAT step only (StepResult.action_saturations is per
    step, envs.hpp:82-89): ended rows / saturations of earlier sg_env_step calls
    must not leak into it, and a host step without result buffers still
    advances the totals."""
    _cuda()
    n = 96
    env = sg.VecTaskEnv(robots=robots, n_envs=n, seed=5, episode_len=3, task=task)
    env.reset()
    A = env.action_dim
    sat_act = np.full((n, A), 1.5, dtype=np.float32)  # every entry saturates
    for _ in range(3):  # device steps: every row times out at the third
        env.step(torch.from_numpy(sat_act).cuda())
    torch.cuda.synchronize()
    act = np.zeros((n, A), dtype=np.float32)
    act[:5, 0] = 2.0  # 5 saturated entries
    r = env.step_host(act)
    assert r["action_saturations"] == 5
    assert not (r["terminated"] | r["timed_out"]).any()
    assert env.host_counters() == (0, 5)
    sg._check(sg.lib().sg_env_step_host(env._h, torch.from_numpy(act).pin_memory().data_ptr(), None))  # no result
    r = env.step_host(act)  # third step of the episode: every row times out
    assert r["action_saturations"] == 5 and r["timed_out"].all()
    assert env.host_counters() == (n, 15)


def test_nonfinite_action_is_sim_error(sg, oracle):
    _cuda()
    env = sg.VecTaskEnv(robots=("psm",), n_envs=8)
    env.reset()
    act = np.zeros((8, 7), np.float32)
    act[3, 2] = np.nan
    with pytest.raises(sg.SimError, match="non-finite action"):
        env.step_host(act)
    with pytest.raises(sg.SimError, match="shape"):
        env.step_host(np.zeros((8, 6), np.float32))


@pytest.mark.parametrize("mode", ["position", "velocity", "torque"])
def test_control_modes_limits_and_parity(sg, oracle, mode):
    """Adversarial actions in [-2, 2] (test_dynamics.cpp:134-163) in every
    control mode (these run on the generic-chain kernel): every field --
    q, qdot, q_target, tips, goals, observations, terminal observations,
    rewards, task_error -- at the standard per-step tolerances, flags /
    counters / streams bit-exact, saturation counts exact per step, and the
    joint and velocity limits hold on every step."""
    m = oracle.resolve_robot("psm")
    # the device stores limits in fp32: the bounds hold against the fp32-rounded limits
    f32 = lambda v: np.float64(np.float32(v))
    lo = np.array([f32(m.dof_joint(d).limit_lo) for d in range(m.dof)])
    hi = np.array([f32(m.dof_joint(d).limit_hi) for d in range(m.dof)])
    vl = np.array([f32(m.dof_joint(d).velocity_limit) for d in range(m.dof)])
    rng = oracle.make_stream(42, 0)
    n = 64
    seen = dict(sat=0)

    def actions(s):
        return 2.0 * oracle.fill_uniform_actions(rng, n, m.dof)

    def check(s, env, ref, res, a32):
        st = env.state()
        q, qd = _soa(st["q"]), _soa(st["qdot"])
        assert (q >= lo).all() and (q <= hi).all()
        assert (np.abs(qd) <= vl).all()
        assert int(((a32 < -1) | (a32 > 1)).sum()) == ref.result()["saturations"]
        seen["sat"] += ref.result()["saturations"]
        assert int(res.saturations_total.item()) == seen["sat"]  # device running total, exact

    _run_pair(sg, oracle, "psm", oracle.TARGET_REACHING, n, 250, seed=99, actions_fn=actions, mode=mode,
              per_step=check)
    assert seen["sat"] > 0


def test_fk_batch_matches_matrix_oracle(sg, oracle):
    """FK vs the 4x4 homogeneous-matrix oracle (test_robot_model.cpp:139-151):
    1000 random in-limit q per robot; fp32 device vs fp64 oracle."""
    _cuda()
    rng = oracle.make_stream(2024, 11)
    for name in ("psm", "ecm", "star"):
        m = oracle.resolve_robot(name)
        qs = np.array([[oracle.uniform(rng, m.dof_joint(d).limit_lo, m.dof_joint(d).limit_hi)
                        for d in range(m.dof)] for _ in range(1000)])
        ref = np.array([oracle.fk_matrix(m, q)[:3, 3] for q in qs])
        rob = sg.Robot.resolve(name)
        pos = rob.fk(torch.from_numpy(qs.astype(np.float32)).cuda()).cpu().numpy()
        assert np.abs(pos - ref).max() < 2e-6, name
    with pytest.raises(sg.SimError, match="outside"):
        bad = np.zeros((1, 7), np.float32)
        bad[0, 0] = 5.0
        sg.Robot.resolve("psm").fk(torch.from_numpy(bad).cuda())


def test_custom_descriptor_generic_axes_and_fixed_joints(sg, oracle):
    """Generic (non axis-aligned) joint axes, rotated origins and fixed joints
    take the generic FK path; parity vs the oracle FK."""
    _cuda()
    s3 = float(1 / np.sqrt(3.0))
    text = f"""[robot]
name = weird
[joint]
name = a
kind = revolute
axis = {s3!r} {s3!r} {s3!r}
origin_xyz = 0.1 0 0.2
origin_rpy = 0.3 -0.2 0.5
limits = -2 2
velocity_limit = 3
effort_limit = 10
[joint]
name = f
kind = fixed
origin_xyz = 0 0.05 0
origin_rpy = 0.1 0.2 0.3
[joint]
name = b
kind = prismatic
axis = 0 0.6 0.8
origin_xyz = 0 0 0.1
origin_rpy = 0 0 0
limits = -0.1 0.3
velocity_limit = 1
effort_limit = 10
[joint]
name = c
kind = revolute
axis = 0 -1 0
origin_xyz = 0.02 0 0
origin_rpy = 0 0 0
limits = -1 1
velocity_limit = 3
effort_limit = 10
[joint]
name = g
kind = fixed
origin_xyz = 0 0 0.07
origin_rpy = 0 0.4 0
[tool_tip]
xyz = 0.01 0.02 0.03
rpy = 0 0 0
"""
    m = oracle.parse_robot(text)
    rng = oracle.make_stream(3, 3)
    qs = np.array([[oracle.uniform(rng, m.dof_joint(d).limit_lo, m.dof_joint(d).limit_hi)
                    for d in range(m.dof)] for _ in range(500)])
    ref = np.array([oracle.fk_matrix(m, q)[:3, 3] for q in qs])
    rob = sg.Robot.parse(text)
    pos = rob.fk(torch.from_numpy(qs.astype(np.float32)).cuda()).cpu().numpy()
    assert np.abs(pos - ref).max() < 2e-6


def test_cpp_dropin_runs_on_the_device(sg, tmp_path):
    """examples/bench_sim_cpp.cpp (scalpel_b200::VecTaskEnv, include/sg/env.hpp)
    runs the reference's bench_sim loop on the device from C++."""
    _cuda()
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    libdir = os.path.dirname(sg.lib_path())
    exe = str(tmp_path / "bench_sim_cpp")
    r = subprocess.run(["g++", "-std=c++17", "-O2", "-I", os.path.join(root, "include"),
                        os.path.join(root, "examples", "bench_sim_cpp.cpp"), f"-L{libdir}", "-lsg_env",
                        f"-Wl,-rpath,{libdir}", "-o", exe], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    run = subprocess.run([exe, "1024", "50"], capture_output=True, text=True, timeout=120)
    assert run.returncode == 0, run.stdout + run.stderr
    assert "1024 envs x 50 steps" in run.stdout


@pytest.mark.parametrize("robot", ["ecm", "star"])
def test_active_tracking_specialised_chains(sg, oracle, robot):
    """ActiveTracking on the ECM / STAR specialised-chain kernels (point-form
    FK in the last team warp): streams and flags bit-exact, goals within
    2e-5 m over a reset burst."""
    sigma = 0.15 if robot == "star" else 0.05
    env, ref, worst = _run_pair(sg, oracle, robot, oracle.ACTIVE_TRACKING, 64, 310, seed=7, sigma=sigma,
                                tol=dict(goals=2e-5))
    assert (ref.counters()["episode_count"] == 1).all()


@pytest.mark.parametrize("robots,task", [(("psm",), "target_reaching"), (("star",), "path_following"),
                                         (("psm", "psm", "ecm"), "multi_tool_reaching")])
def test_step_into_caller_buffers_equals_step(sg, oracle, robots, task):
    """sg_env_step_into writes the step's observations / rewards / task_error
    / flags into caller device buffers (the trainer's rollout slots) and is
    otherwise the same step: bit-identical results and state across a reset
    burst (episode_len 5); terminal observations stay env-owned."""
    _cuda()
    n = 256
    kw = dict(robots=robots, n_envs=n, seed=6, episode_len=5, task=task,
              goal_sigma=0.15 if task == "path_following" else 0.05)
    a, b = sg.VecTaskEnv(**kw), sg.VecTaskEnv(**kw)
    a.reset(); b.reset()
    A, O = a.action_dim, a.obs_dim
    rng = np.random.default_rng(3)
    for s in range(7):
        act = torch.from_numpy(rng.uniform(-1, 1, size=(n, A)).astype(np.float32)).cuda()
        dst = dict(observations=torch.full((n, O), 7.0, device="cuda"), rewards=torch.zeros(n, device="cuda"),
                   task_error=torch.zeros(n, device="cuda"),
                   terminated=torch.full((n,), 9, dtype=torch.uint8, device="cuda"),
                   timed_out=torch.full((n,), 9, dtype=torch.uint8, device="cuda"))
        ra = a.step_into(act, **dst)
        rb = b.step(act)
        torch.cuda.synchronize()
        for k, v in dst.items():
            assert torch.equal(v, getattr(rb, k)), (k, s)
        ended = (rb.terminated | rb.timed_out).bool()
        assert torch.equal(ra.terminal_observations[ended], rb.terminal_observations[ended])
        sa, sb = a.state(), b.state()
        for k in ("q", "qdot", "rng_state", "step_count"):
            assert torch.equal(sa[k], sb[k]), (k, s)
