"""Oracle MultiToolReaching (envs.cpp:90-116, 304-360, 540-593) pinned against an
independent pure-Python restatement: 4x4 homogeneous-matrix FK (the
reference's own FK test oracle, test_robot_model.cpp:27-56), per-DoF dynamics
loops (dynamics.cpp:127-185), per-tool PCG32 streams (dynamics.cpp:238) and the
task's reward / camera-goal / collision / hold rules written out from envs.cpp.
The reference has no MultiToolReaching test, so this cross-check (and the
structural properties below) is what pins the C restatement."""
import math

import numpy as np
import pytest


class PyMultiTool:
    """Pure-Python MultiToolReaching, row by row like envs.cpp."""

    def __init__(self, O, cfg, robots, seed):
        self.O, self.cfg, self.m = O, cfg, robots
        self.T = len(robots)
        self.n = cfg.n_envs
        self.radius = cfg.workspace_radius if cfg.workspace_radius > 0 else 3.0 * cfg.goal_sigma
        # default_tool_bases (envs.cpp:101-116)
        dx = 0.7 * self.radius
        self.base = [(np.zeros(3), np.eye(3)) for _ in range(self.T)]
        self.base[0] = (np.array([-dx, 0.0, 0.0]), np.eye(3))
        self.base[1] = (np.array([dx, 0.0, 0.0]), np.eye(3))
        if self.T >= 3:
            c, s = math.cos(0.9), math.sin(0.9)  # quat_from_rpy(0.9, 0, 0) = Rx(0.9)
            self.base[2] = (np.array([0.0, -2.0 * self.radius, 0.5 * self.radius]),
                            np.array([[1, 0, 0], [0, c, -s], [0, s, c]]))
        for t in range(3, self.T):
            self.base[t] = (np.array([0.0, (t - 1.0) * 2.0 * dx, 0.0]), np.eye(3))
        self.dyn = [O.default_dynamics(m) for m in robots]
        self.ecm = [m.name.decode() == "ecm" for m in robots]
        self.centers = []
        self.q, self.qd, self.qt, self.rng = [], [], [], []
        for t, m in enumerate(robots):
            mid = np.array([0.5 * (m.dof_joint(d).limit_lo + m.dof_joint(d).limit_hi) for d in range(m.dof)])
            self.centers.append(self._world(t, mid)[0])
            self.q.append(np.tile(mid, (self.n, 1)))
            self.qd.append(np.zeros((self.n, m.dof)))
            self.qt.append(np.tile(mid, (self.n, 1)))
            self.rng.append([O.make_stream(seed, (t << 32) + i) for i in range(self.n)])
        self.goals = np.zeros((self.n, 3 * self.T))
        self.tips = np.zeros((self.n, 3 * self.T))
        self.axes = np.zeros((self.n, 3 * self.T))
        self.step_count = np.zeros(self.n, np.int64)
        self.hold = np.zeros(self.n, np.int64)
        self.episodes = np.zeros(self.n, np.int64)
        self.collisions = 0

    def _world(self, t, q):
        M = self.O.fk_matrix(self.m[t], q)
        bp, bR = self.base[t]
        return bp + bR @ M[:3, 3], bR @ M[:3, :3]

    def _refresh(self, i):
        for t in range(self.T):
            p, R = self._world(t, self.q[t][i])
            self.tips[i, 3 * t:3 * t + 3] = p
            self.axes[i, 3 * t:3 * t + 3] = R @ np.array([0.0, 0.0, -1.0])

    def _mid(self, i, t):
        return np.mean([self.tips[i, 3 * u:3 * u + 3] for u in range(self.T) if u != t], axis=0)

    def _goal(self, r, c):
        s = self.cfg.goal_sigma
        for _ in range(1000):
            nz, ny, nx = (s * self.O.normal(r) for _ in range(3))  # g++ right-to-left
            g = c + np.array([nx, ny, nz])
            if np.linalg.norm(g - c) <= self.radius:
                return g
        raise AssertionError("goal sampling")

    def reset_row(self, i):
        for t, m in enumerate(self.m):
            for d in range(m.dof):
                j = m.dof_joint(d)
                quarter = 0.25 * (j.limit_hi - j.limit_lo)
                self.q[t][i, d] = self.O.uniform(self.rng[t][i], j.limit_lo + quarter, j.limit_hi - quarter)
                self.qd[t][i, d] = 0.0
                self.qt[t][i, d] = self.q[t][i, d]
        self._refresh(i)
        for t in range(self.T):
            self.goals[i, 3 * t:3 * t + 3] = (self._mid(i, t) if self.ecm[t]
                                              else self._goal(self.rng[t][i], self.centers[t]))
        self.step_count[i] = 0
        self.hold[i] = 0
        self.episodes[i] += 1

    def reset(self):
        for i in range(self.n):
            self.reset_row(i)
            self.episodes[i] = 0
        return self.observe()

    def observe(self):
        return np.concatenate([np.hstack(self.q), np.hstack(self.qd), self.tips, np.hstack(self.qt),
                               self.goals], axis=1)

    def step(self, actions):
        col = 0
        for t, m in enumerate(self.m):
            cfg = self.dyn[t]
            dt = cfg.control_dt / cfg.substeps
            jaw = self.O.lib().sgo_jaw_dof(m)
            for i in range(self.n):
                for d in range(m.dof):
                    j = m.dof_joint(d)
                    a = min(max(actions[i, col + d], -1.0), 1.0)
                    lo, hi = j.limit_lo, j.limit_hi
                    if d == jaw:
                        self.qt[t][i, d] = hi if a > 0 else lo
                    else:
                        self.qt[t][i, d] = hi if a >= 1 else (lo if a <= -1 else lo + 0.5 * (a + 1) * (hi - lo))
                    q, qd = self.q[t][i, d], self.qd[t][i, d]
                    for _ in range(cfg.substeps):
                        tau = cfg.kp[d] * (self.qt[t][i, d] - q) - cfg.kd[d] * qd
                        tau = min(max(tau, -j.effort_limit), j.effort_limit)
                        qd += (tau - cfg.damping[d] * qd) / cfg.inertia[d] * dt
                        qd = min(max(qd, -j.velocity_limit), j.velocity_limit)
                        q += qd * dt
                        if q < lo:
                            q, qd = lo, 0.0
                        elif q > hi:
                            q, qd = hi, 0.0
                    self.q[t][i, d], self.qd[t][i, d] = q, qd
            col += m.dof
        rew = np.zeros(self.n); err = np.zeros(self.n)
        term = np.zeros(self.n, np.uint8); tout = np.zeros(self.n, np.uint8)
        for i in range(self.n):
            self._refresh(i)
            self.step_count[i] += 1
            reward, es, ec, all_in = 0.0, 0.0, 0, True
            for t in range(self.T):
                tip = self.tips[i, 3 * t:3 * t + 3]
                if self.ecm[t]:
                    mid = self._mid(i, t)
                    self.goals[i, 3 * t:3 * t + 3] = mid
                    to_mid = mid - tip
                    if np.linalg.norm(to_mid) > 1e-12:
                        c = float(np.dot(self.axes[i, 3 * t:3 * t + 3], to_mid / np.linalg.norm(to_mid)))
                        reward += -self.cfg.view_penalty * math.acos(min(max(c, -1.0), 1.0))
                else:
                    dist = float(np.linalg.norm(tip - self.goals[i, 3 * t:3 * t + 3]))
                    reward += self.cfg.reward_scale * dist
                    es += dist
                    ec += 1
                    all_in &= dist < self.cfg.success_radius
            sep = min(np.linalg.norm(self.tips[i, 3 * t:3 * t + 3] - self.tips[i, 3 * u:3 * u + 3])
                      for t in range(self.T) for u in range(t + 1, self.T))
            if sep < self.cfg.collision_threshold:
                reward -= self.cfg.collision_penalty
                self.collisions += 1
            err[i] = es / ec if ec else 0.0
            self.hold[i] = self.hold[i] + 1 if all_in else 0
            term[i] = self.hold[i] >= self.cfg.success_hold
            tout[i] = self.step_count[i] >= self.cfg.episode_len
            rew[i] = reward
        obs = self.observe()
        tobs = obs.copy()
        for i in range(self.n):
            if term[i] or tout[i]:
                self.reset_row(i)
        return self.observe(), tobs, rew, err, term, tout


@pytest.mark.parametrize("robots,threshold", [(("psm", "psm"), 0.01), (("psm", "psm", "ecm"), 0.2)])
def test_multitool_matches_python_restatement(oracle, robots, threshold):
    """C oracle == independent Python restatement over a reset burst (episode
    length 40), including the ECM camera goal / view penalty, the collision
    penalty (threshold 0.2 m so it fires) and per-tool streams."""
    n, seed = 4, 7
    ms = [oracle.resolve_robot(r) for r in robots]
    cfg = oracle.env_config(n_envs=n, seed=seed, task=oracle.MULTI_TOOL, episode_len=40,
                            collision_threshold=threshold)
    c_env = oracle.MultiToolEnv(cfg, ms)
    py = PyMultiTool(oracle, cfg, ms, seed)
    np.testing.assert_allclose(c_env.reset(), py.reset(), atol=1e-12)
    ar = oracle.make_stream(seed, 0xAC7104)
    for s in range(85):
        a = oracle.fill_uniform_actions(ar, n, c_env.action_dim)
        c_env.step(a)
        obs, tobs, rew, err, term, tout = py.step(a)
        r = c_env.result()
        o, to = c_env.obs()
        assert np.array_equal(r["timed_out"], tout) and np.array_equal(r["terminated"], term), s
        np.testing.assert_allclose(o, obs, atol=1e-10, err_msg=f"obs @{s}")
        ended = (tout | term).astype(bool)
        np.testing.assert_allclose(to[ended], tobs[ended], atol=1e-10)
        np.testing.assert_allclose(r["rewards"], rew, atol=1e-9, err_msg=f"reward @{s}")
        np.testing.assert_allclose(r["task_error"], err, atol=1e-10)
        st = c_env.state()
        np.testing.assert_allclose(st["axes"], py.axes, atol=1e-10)
    s_c, _ = c_env.rng()
    for t in range(len(ms)):
        assert [int(x) for x in s_c[t]] == [py.rng[t][i].state for i in range(n)]
    assert (c_env.counters()["episode_count"] == 2).all()
    assert (py.collisions > 0) == (threshold > 0.1)


def test_default_tool_bases(oracle):
    """default_tool_bases (envs.cpp:101-116)."""
    r = 0.15
    b2 = oracle.default_tool_bases(2, r)
    np.testing.assert_array_equal(b2[:, :3], [[-0.7 * r, 0, 0], [0.7 * r, 0, 0]])
    np.testing.assert_array_equal(b2[:, 3:], [[1, 0, 0, 0]] * 2)
    b4 = oracle.default_tool_bases(4, r)
    np.testing.assert_allclose(b4[2], [0, -2 * r, 0.5 * r, math.cos(0.45), math.sin(0.45), 0, 0], atol=1e-15)
    np.testing.assert_array_equal(b4[3, :3], [0, 2.0 * 2.0 * 0.7 * r, 0])
    np.testing.assert_array_equal(oracle.default_tool_bases(1, r), [[0, 0, 0, 1, 0, 0, 0]])


def test_min_separation(oracle):
    """multi_tool_min_separation (envs.cpp:90-99): +inf for < 2 tips."""
    assert math.isinf(oracle.multi_tool_min_separation(np.zeros((1, 3))))
    tips = np.array([[0, 0, 0], [0.3, 0, 0], [0.3, 0.04, 0]])
    assert oracle.multi_tool_min_separation(tips) == pytest.approx(0.04)


def test_multitool_stream_consumption(oracle):
    """reset(): tool t's stream supplies its dof q draws then 6 u32 per goal
    attempt; the ECM camera arm draws no goal (its goal is the tips' midpoint)."""
    ms = [oracle.resolve_robot(r) for r in ("psm", "psm", "ecm")]
    cfg = oracle.env_config(n_envs=3, seed=11, task=oracle.MULTI_TOOL)
    e = oracle.MultiToolEnv(cfg, ms)
    e.reset()
    st, _ = e.rng()
    for i in range(3):
        r = oracle.make_stream(11, (2 << 32) + i)
        for _ in range(6):
            oracle.next_u32(r)
        assert r.state == int(st[2, i])
        for t in (0, 1):
            r = oracle.make_stream(11, (t << 32) + i)
            for _ in range(7):
                oracle.next_u32(r)
            k = 0
            while r.state != int(st[t, i]):
                oracle.next_u32(r)
                k += 1
                assert k <= 6000
            assert k % 6 == 0 and k >= 6
    g = e.state()["goals"]
    tips = e.state()["tips"]
    np.testing.assert_allclose(g[:, 6:9], 0.5 * (tips[:, 0:3] + tips[:, 3:6]), atol=1e-15)


def test_multitool_config_errors(oracle):
    m = oracle.resolve_robot("psm")
    with pytest.raises(oracle.OracleError, match="requires >= 2 robots"):
        oracle.MultiToolEnv(oracle.env_config(n_envs=2, task=oracle.MULTI_TOOL), [m])
    with pytest.raises(oracle.OracleError, match="collision_threshold"):
        oracle.MultiToolEnv(oracle.env_config(n_envs=2, task=oracle.MULTI_TOOL, collision_threshold=-1.0), [m, m])


def test_multitool_row_offset_shards(oracle):
    """Sharding: tool t of global row g draws from
    make_stream(seed, t * 2^32 + g), so a shard with row_offset equals the
    same rows of one env (bench stream indexed by global row)."""
    ms = [oracle.resolve_robot(r) for r in ("psm", "psm", "ecm")]
    cfg = dict(seed=9, task=oracle.MULTI_TOOL, episode_len=30)
    full = oracle.MultiToolEnv(oracle.env_config(n_envs=12, **cfg), ms)
    part = oracle.MultiToolEnv(oracle.env_config(n_envs=5, row_offset=7, **cfg), ms)
    full.reset(); part.reset()
    ar = oracle.make_stream(9, 0xAC7104)
    for _ in range(40):
        a = oracle.fill_uniform_actions(ar, 12, 20)
        full.step(a)
        part.step(a[7:])
        np.testing.assert_array_equal(full.obs()[0][7:], part.obs()[0])
    np.testing.assert_array_equal(full.rng()[0][:, 7:], part.rng()[0])
