"""Oracle VecTaskEnv (envs.cpp) properties, fp32 drift bounds (which set the
GPU parity tolerances) and the committed golden digests."""
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_config1_episode_structure(oracle):
    """BASELINE config 1: PSM reach, 64 envs, seed 0, warm-up + 1000 steps of the
    bench stream: every env times out at steps 300/600/900, nothing terminates
    by goal; 256 resets draw 264 goal candidates (survey probe, Appendix E)."""
    m = oracle.resolve_robot("psm")
    e = oracle.Env(oracle.env_config(n_envs=64, seed=0), m)
    e.reset()
    ar = oracle.make_stream(0, 0xAC7104)
    timeouts = terms = 0
    for s in range(1001):
        e.step(oracle.fill_uniform_actions(ar, 64, 7))
        r = e.result()
        timeouts += int(r["timed_out"].sum())
        terms += int(r["terminated"].sum())
        if r["timed_out"].any():
            assert (s + 1) % 300 == 0 and r["timed_out"].all()
    assert timeouts == 192 and terms == 0
    assert e.goal_draws() == 264
    assert (e.counters()["episode_count"] == 3).all()


def test_fp32_drift_bounds(oracle):
    """Intrinsic fp32 drift (fp32 oracle vs fp64 oracle, same inputs): the GPU
    parity tolerances in tests/test_gpu_parity.py must cover it."""
    from tests.test_gpu_parity import TOL
    for robot, task, sigma, n, steps in (("psm", 0, 0.05, 64, 400), ("star", 3, 0.15, 32, 350)):
        m = oracle.resolve_robot(robot)
        cfg = oracle.env_config(n_envs=n, seed=0, task=task, goal_sigma=sigma)
        a64, a32 = oracle.Env(cfg, m), oracle.Env(cfg, m, precision="f32")
        a64.reset(); a32.reset()
        ar = oracle.make_stream(0, 0xAC7104)
        for _ in range(steps):
            a = oracle.fill_uniform_actions(ar, n, m.dof).astype(np.float32).astype(np.float64)
            a64.step(a); a32.step(a)
            s64, s32 = a64.state(), a32.state()
            for k in ("q", "qdot", "q_target"):
                assert np.abs(s64[k] - s32[k]).max() <= TOL[k] / 2, (robot, k)
            assert np.abs(s64["tips"] - s32["tips"]).max() <= TOL["tips"] / 2
            r64, r32 = a64.result(), a32.result()
            assert np.array_equal(r64["timed_out"], r32["timed_out"])
            assert np.array_equal(r64["terminated"], r32["terminated"])
            for k in ("step_count", "hold_count", "episode_count", "waypoint_idx", "waypoint_len"):
                assert np.array_equal(a64.counters()[k], a32.counters()[k])


def test_path_following_reset_properties(oracle):
    """sample_path (envs.cpp:241-267): waypoints start at wps[0] = goal, stay
    inside the workspace ball, and never exceed the device table capacity
    floor(1.3*sqrt(3)/spacing) + 4 (|a|+|b|+|c| arc-length bound)."""
    m = oracle.resolve_robot("star")
    n = 400
    e = oracle.Env(oracle.env_config(n_envs=n, seed=3, task=oracle.PATH_FOLLOWING, goal_sigma=0.15), m)
    e.reset()
    center, radius = e.workspace()
    cap = int(np.floor(1.3 * np.sqrt(3.0) / 0.02)) + 4
    lens = e.counters()["waypoint_len"]
    assert lens.max() <= cap and lens.min() >= 1
    goals = e.state()["goals"]
    for row in range(0, n, 7):
        w = e.waypoints(row)
        assert np.array_equal(w[0], goals[row])
        assert (np.linalg.norm(w - center, axis=1) <= radius + 1e-9).all()
        if len(w) > 2:
            gaps = np.linalg.norm(np.diff(w, axis=0), axis=1)[:-1]
            assert np.all(gaps <= 0.02 * 1.0001)  # chord <= arc-length spacing


def test_sharded_rows_equal_global_rows(oracle):
    """row_offset seeding: rows [64, 128) of a 128-env oracle equal a 64-env
    shard with row_offset 64 fed the same actions (multi-GPU sharding rule)."""
    m = oracle.resolve_robot("psm")
    full = oracle.Env(oracle.env_config(n_envs=128, seed=5), m)
    part = oracle.Env(oracle.env_config(n_envs=64, seed=5, row_offset=64), m)
    full.reset(); part.reset()
    ar = oracle.make_stream(5, 0xAC7104)
    for _ in range(310):
        a = oracle.fill_uniform_actions(ar, 128, 7)
        full.step(a); part.step(a[64:])
    assert np.array_equal(full.obs()[0][64:], part.obs()[0])
    assert np.array_equal(full.rng()[0][64:], part.rng()[0])


def _digest(oracle, robot, task, sigma, n, steps, seed):
    m = oracle.resolve_robot(robot)
    e = oracle.Env(oracle.env_config(n_envs=n, seed=seed, task=task, goal_sigma=sigma), m)
    e.reset()
    ar = oracle.make_stream(seed, 0xAC7104)
    rows = []
    for s in range(steps):
        e.step(oracle.fill_uniform_actions(ar, n, m.dof))
        if s % 50 == 49 or s == steps - 1:
            o, t = e.obs()
            r = e.result()
            c = e.counters()
            rows.append(dict(step=s, obs_sum=float(o.sum()), obs_abs=float(np.abs(o).sum()),
                             reward_sum=float(r["rewards"].sum()), timed_out=int(r["timed_out"].sum()),
                             terminated=int(r["terminated"].sum()), episodes=int(c["episode_count"].sum()),
                             wp=int(c["waypoint_idx"].sum()), rng_xor=int(np.bitwise_xor.reduce(e.rng()[0]))))
    return rows


def test_golden_digests(oracle):
    """Regression pin: the oracle reproduces the committed digests (generated
    by tests/golden/make_golden.py) bit for bit."""
    with open(os.path.join(GOLDEN, "oracle_digests.json")) as f:
        golden = json.load(f)
    for case in golden["cases"]:
        got = _digest(oracle, case["robot"], case["task"], case["sigma"], case["n"], case["steps"], case["seed"])
        assert got == case["rows"], case["name"]


def test_active_tracking_stream_consumption(oracle):
    """ActiveTracking (envs.cpp:493-512): after the reset draws, every step
    takes exactly 3 normals (6 u32) from each env's stream for the goal
    velocity noise, and goals stay inside spawn +- goal_offset_clip."""
    m = oracle.resolve_robot("psm")
    n = 8
    env = oracle.Env(oracle.env_config(n_envs=n, seed=11, task=oracle.ACTIVE_TRACKING), m)
    env.reset()
    s0, inc = env.rng()
    spawn = env.state()["goals"].copy()
    rng = oracle.make_stream(0, 0xAC7104)
    for _ in range(20):
        env.step(oracle.fill_uniform_actions(rng, n, m.dof))
    s1, _ = env.rng()
    for i in range(n):
        r = oracle.Pcg32(int(s0[i]), int(inc[i]))
        for _ in range(6 * 20):
            oracle.next_u32(r)
        assert r.state == s1[i]
    g = env.state()["goals"]
    assert (np.abs(g - spawn) <= 0.2 + 1e-12).all()
    assert np.abs(g - spawn).max() > 0.0
