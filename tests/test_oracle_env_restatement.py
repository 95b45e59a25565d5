"""Oracle VecTaskEnv (single robot: TargetReaching, ActiveTracking,
PathFollowing) pinned against an independent pure-Python restatement written
from the reference's envs.cpp / dynamics.cpp / spline.cpp, row by row:

* reset_row (envs.cpp:304-360): quarter-range q draws, sample_goal
  (envs.cpp:230-239, g++ right-to-left argument order: z drawn first),
  sample_path (envs.cpp:241-267) with the spline waypoints of
  spline.cpp:40-72 re-implemented here (cumulative chord table, arc-length
  emission loop, degenerate-length cut), tracking spawn / velocity state;
* step (envs.cpp:437-617): position-control dynamics (dynamics.cpp:130-186),
  tips by the 4x4 homogeneous-matrix FK (the reference's own FK test oracle,
  test_robot_model.cpp:27-56), per-task reward / hold / waypoint advance /
  goal drift (envs.cpp:480-528), flags, terminal observations, resets of the
  ended rows and their re-observation (envs.cpp:600-616);
* observe_rows (envs.cpp:362-410): q, qdot, tip, q_target, goal / current
  waypoint.

The reference's own tests never touch envs.cpp, so the C oracle's env level
was pinned only by the survey probe's statistics and by digests the oracle
itself generated; this restatement shares no code with it (only the PCG32
primitives and the 4x4 FK, both pinned by the reference's KATs) and checks it
step by step, across reset bursts, terminations and waypoint advances."""
import math

import numpy as np
import pytest


def _norm(v):  # Eigen .norm(): sqrt of the in-order sum of squares
    return math.sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2])


class PySpline:
    """CubicSpline3 (spline.hpp:23-35), t0 = 0, t1 = 1."""

    def __init__(self, a, b, c, d):
        self.a, self.b, self.c, self.d = list(a), list(b), list(c), list(d)

    def eval(self, t):
        u = t - 0.0
        return [((self.a[k] * u + self.b[k]) * u + self.c[k]) * u + self.d[k] for k in range(3)]


def py_waypoints(sp: PySpline, spacing: float):
    """sample_spline_waypoints (spline.cpp:40-72) with 1000 subdivisions."""
    n, span = 1000, 1.0
    pts = [sp.eval(0.0)]
    cum = [0.0]
    for k in range(1, n + 1):
        pts.append(sp.eval(0.0 + span * k / n))
        cum.append(cum[-1] + _norm([pts[k][j] - pts[k - 1][j] for j in range(3)]))
    total = cum[n]
    wps = [pts[0]]
    if total <= 1e-12:
        return wps
    seg, s = 0, spacing
    while s < total - 1e-12:
        while seg + 1 < n and cum[seg + 1] < s:
            seg += 1
        seg_len = cum[seg + 1] - cum[seg]
        frac = (s - cum[seg]) / seg_len if seg_len > 0.0 else 0.0
        wps.append(sp.eval(0.0 + span * (seg + frac) / n))
        s += spacing
    wps.append(pts[n])
    return wps


class PyVecTaskEnv:
    TARGET, TRACK, PATH = 0, 1, 3

    def __init__(self, O, cfg, m):
        self.O, self.cfg, self.m = O, cfg, m
        self.n, self.A = cfg.n_envs, m.dof
        self.dyn = O.default_dynamics(m)
        self.jaw = O.lib().sgo_jaw_dof(m)
        self.radius = cfg.workspace_radius if cfg.workspace_radius > 0.0 else 3.0 * cfg.goal_sigma
        mid = [0.5 * (m.dof_joint(d).limit_lo + m.dof_joint(d).limit_hi) for d in range(self.A)]
        self.center = list(O.fk_matrix(m, np.array(mid))[:3, 3])
        self.rng = [O.make_stream(cfg.seed, cfg.row_offset + i) for i in range(self.n)]
        z = lambda: [[0.0] * self.A for _ in range(self.n)]
        self.q, self.qd, self.qt = z(), z(), z()
        self.tips = [[0.0] * 3 for _ in range(self.n)]
        self.goals = [[0.0] * 3 for _ in range(self.n)]
        self.spawn = [[0.0] * 3 for _ in range(self.n)]
        self.vel = [[0.0] * 3 for _ in range(self.n)]
        self.wps = [None] * self.n
        self.widx = [0] * self.n
        self.step_count = [0] * self.n
        self.hold = [0] * self.n
        self.episodes = [0] * self.n

    # -- envs.cpp:230-267 --------------------------------------------------
    def _goal(self, r, c):
        s = self.cfg.goal_sigma
        for _ in range(1000):
            nz = 0.0 + s * self.O.normal(r)  # Vector3d(n(), n(), n()): g++ evaluates right to left
            ny = 0.0 + s * self.O.normal(r)
            nx = 0.0 + s * self.O.normal(r)
            g = [c[0] + nx, c[1] + ny, c[2] + nz]
            if _norm([g[k] - c[k] for k in range(3)]) <= self.radius:
                return g
        raise AssertionError("goal sampling")

    def _path(self, i):
        r = self.rng[i]
        a = [self.O.uniform(r, -0.5, 0.5) for _ in range(3)]
        b = [self.O.uniform(r, -0.5, 0.5) for _ in range(3)]
        c = [self.O.uniform(r, -0.3, 0.3) for _ in range(3)]
        d = self._goal(r, self.center)
        sp = PySpline(a, b, c, d)
        max_off = 0.0
        for k in range(101):
            p = sp.eval(0.01 * k)
            max_off = max(max_off, _norm([p[j] - d[j] for j in range(3)]))
        allowed = self.radius - _norm([d[j] - self.center[j] for j in range(3)])
        if max_off > 0.0 and max_off > allowed:
            scale = 0.95 * max(allowed, 0.0) / max_off
            sp = PySpline([x * scale for x in a], [x * scale for x in b], [x * scale for x in c], d)
        self.wps[i] = py_waypoints(sp, self.cfg.waypoint_spacing)
        self.widx[i] = 0

    def _tip(self, i):
        self.tips[i] = list(self.O.fk_matrix(self.m, np.array(self.q[i]))[:3, 3])

    # -- envs.cpp:304-360 --------------------------------------------------
    def reset_row(self, i):
        r = self.rng[i]
        for d in range(self.A):
            j = self.m.dof_joint(d)
            quarter = 0.25 * (j.limit_hi - j.limit_lo)
            self.q[i][d] = self.O.uniform(r, j.limit_lo + quarter, j.limit_hi - quarter)
            self.qd[i][d] = 0.0
            self.qt[i][d] = self.q[i][d]
        self._tip(i)
        task = self.cfg.task
        if task == self.TARGET:
            self.goals[i] = self._goal(r, self.center)
        elif task == self.TRACK:
            g = self._goal(r, self.center)
            self.goals[i], self.spawn[i], self.vel[i] = list(g), list(g), [0.0, 0.0, 0.0]
        else:
            self._path(i)
            self.goals[i] = list(self.wps[i][0])
        self.step_count[i] = 0
        self.hold[i] = 0
        self.episodes[i] += 1

    def observe(self, i):
        goal = self.wps[i][self.widx[i]] if self.cfg.task == self.PATH else self.goals[i]
        return self.q[i] + self.qd[i] + self.tips[i] + self.qt[i] + list(goal)

    def reset(self):
        for i in range(self.n):
            self.reset_row(i)
            self.episodes[i] = 0
        return np.array([self.observe(i) for i in range(self.n)])

    # -- dynamics.cpp:130-186 (position control) ---------------------------
    def _dynamics(self, i, a_row):
        cfg = self.dyn
        dt = cfg.control_dt / cfg.substeps
        for d in range(self.A):
            j = self.m.dof_joint(d)
            lo, hi, vl, ef = j.limit_lo, j.limit_hi, j.velocity_limit, j.effort_limit
            a = a_row[d]
            if a < -1.0 or a > 1.0:
                a = -1.0 if a < -1.0 else 1.0
            if d == self.jaw:
                self.qt[i][d] = hi if a > 0.0 else lo
            else:
                self.qt[i][d] = hi if a >= 1.0 else (lo if a <= -1.0 else lo + 0.5 * (a + 1.0) * (hi - lo))
            q, qd = self.q[i][d], self.qd[i][d]
            for _ in range(cfg.substeps):
                tau = cfg.kp[d] * (self.qt[i][d] - q) - cfg.kd[d] * qd
                tau = ef if tau > ef else tau
                tau = -ef if tau < -ef else tau
                qd += (tau - cfg.damping[d] * qd) / cfg.inertia[d] * dt
                qd = vl if qd > vl else qd
                qd = -vl if qd < -vl else qd
                q += qd * dt
                if q < lo:
                    q, qd = lo, 0.0
                elif q > hi:
                    q, qd = hi, 0.0
            self.q[i][d], self.qd[i][d] = q, qd

    # -- envs.cpp:437-617 --------------------------------------------------
    def step(self, actions):
        cfg, n = self.cfg, self.n
        for i in range(n):
            self._dynamics(i, actions[i])
        for i in range(n):
            self._tip(i)
        rew, err = np.zeros(n), np.zeros(n)
        term, tout = np.zeros(n, np.uint8), np.zeros(n, np.uint8)
        for i in range(n):
            self.step_count[i] += 1
            tip = self.tips[i]
            goal_met = False
            if cfg.task == self.TARGET:
                dist = _norm([tip[k] - self.goals[i][k] for k in range(3)])
                reward = cfg.reward_scale * dist
                self.hold[i] = self.hold[i] + 1 if dist < cfg.success_radius else 0
                goal_met = self.hold[i] >= cfg.success_hold
            elif cfg.task == self.TRACK:
                g = list(self.goals[i])
                dist = _norm([tip[k] - g[k] for k in range(3)])
                reward = cfg.reward_scale * dist
                vel = list(self.vel[i])
                g = [g[k] + vel[k] for k in range(3)]
                for k in range(3):  # the goal drifts after scoring
                    lo = self.spawn[i][k] - cfg.goal_offset_clip
                    hi = self.spawn[i][k] + cfg.goal_offset_clip
                    g[k] = min(max(g[k], lo), hi)
                    vel[k] += 0.0 + cfg.tracking_vel_noise_std * self.O.normal(self.rng[i])
                    vel[k] = min(max(vel[k], -cfg.tracking_vel_clamp), cfg.tracking_vel_clamp)
                self.goals[i], self.vel[i] = g, vel
            else:
                wps = self.wps[i]
                d_of = lambda k: _norm([tip[j] - wps[k][j] for j in range(3)])
                dist = d_of(self.widx[i])
                reward = -cfg.path_penalty * dist
                while self.widx[i] + 1 < len(wps) and d_of(self.widx[i]) < cfg.success_radius:
                    self.widx[i] += 1
                goal_met = self.widx[i] + 1 == len(wps) and d_of(self.widx[i]) < cfg.success_radius
                self.goals[i] = list(wps[self.widx[i]])
            rew[i], err[i] = reward, dist
            term[i] = 1 if goal_met else 0
            tout[i] = 1 if self.step_count[i] >= cfg.episode_len else 0
        obs = np.array([self.observe(i) for i in range(n)])
        tobs = obs.copy()
        for i in range(n):
            if term[i] or tout[i]:
                self.reset_row(i)
                obs[i] = self.observe(i)
        return obs, tobs, rew, err, term, tout


CASES = [
    # robot, task, overrides, steps: resets by timeout and by goal (hold), waypoint advances
    ("psm", PyVecTaskEnv.TARGET, dict(episode_len=50), 160),
    ("ecm", PyVecTaskEnv.TARGET, dict(episode_len=60, success_radius=0.12, success_hold=3), 200),
    ("psm", PyVecTaskEnv.TRACK, dict(episode_len=70, tracking_vel_noise_std=0.004, goal_offset_clip=0.02), 160),
    ("star", PyVecTaskEnv.PATH, dict(episode_len=80, goal_sigma=0.15), 180),
    ("star", PyVecTaskEnv.PATH, dict(episode_len=90, goal_sigma=0.15, success_radius=0.25, waypoint_spacing=0.05), 200),
]


@pytest.mark.parametrize("robot,task,over,steps", CASES)
def test_env_matches_python_restatement(oracle, robot, task, over, steps):
    n, seed = 4, 11
    m = oracle.resolve_robot(robot)
    cfg = oracle.env_config(n_envs=n, seed=seed, task=task, **over)
    c_env = oracle.Env(cfg, m)
    py = PyVecTaskEnv(oracle, cfg, m)
    np.testing.assert_allclose(c_env.reset(), py.reset(), atol=1e-12)
    if task == PyVecTaskEnv.PATH:
        for i in range(n):
            np.testing.assert_allclose(c_env.waypoints(i, 512), np.array(py.wps[i]), atol=1e-12)
    ar = oracle.make_stream(seed, 0xAC7104)
    ended = goal_ends = advances = 0
    for s in range(steps):
        a = oracle.fill_uniform_actions(ar, n, m.dof) * 1.2  # some saturate
        c_env.step(a)
        obs, tobs, rew, err, term, tout = py.step(a)
        r = c_env.result()
        o, to = c_env.obs()
        assert np.array_equal(r["timed_out"], tout) and np.array_equal(r["terminated"], term), s
        np.testing.assert_allclose(o, obs, atol=1e-10, err_msg=f"obs @{s}")
        e = (tout | term).astype(bool)
        np.testing.assert_allclose(to[e], tobs[e], atol=1e-10, err_msg=f"terminal obs @{s}")
        np.testing.assert_allclose(r["rewards"], rew, atol=1e-10, err_msg=f"reward @{s}")
        np.testing.assert_allclose(r["task_error"], err, atol=1e-10)
        st = c_env.state()
        np.testing.assert_allclose(st["goals"], np.array(py.goals), atol=1e-10, err_msg=f"goals @{s}")
        cn = c_env.counters()
        assert list(cn["step_count"]) == py.step_count and list(cn["hold_count"]) == py.hold, s
        assert list(cn["episode_count"]) == py.episodes
        if task == PyVecTaskEnv.PATH:
            assert list(cn["waypoint_idx"]) == py.widx and list(cn["waypoint_len"]) == [len(w) for w in py.wps]
            advances += sum(py.widx)
        ended += int(e.sum())
        goal_ends += int(term.sum())
    s_c, _ = c_env.rng()
    assert [int(x) for x in s_c] == [py.rng[i].state for i in range(n)]
    assert ended > 0
    if over.get("success_hold") or over.get("success_radius"):
        assert goal_ends > 0 or advances > 0  # the goal / waypoint logic fired
