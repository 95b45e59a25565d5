"""ORACLE — test infrastructure only.

ctypes binding of oracle/sg_oracle.c (a plain-C restatement of the reference
"scalpel" hot path). Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` leg may import this module, and only as
the checker or the timed CPU baseline. The product path (the CUDA library
behind include/sg_env.h) never loads it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_BUILD = os.path.join(_HERE, "_build")
ASSETS = os.path.join(os.path.dirname(_HERE), "assets", "robots")

MAX_JOINTS = 32
TARGET_REACHING, ACTIVE_TRACKING, IMAGE_MATCHING, PATH_FOLLOWING, MULTI_TOOL = range(5)
POSITION, VELOCITY, TORQUE = range(3)


class Pcg32(C.Structure):
    _fields_ = [("state", C.c_uint64), ("inc", C.c_uint64)]


class Joint(C.Structure):
    _fields_ = [
        ("name", C.c_char * 64),
        ("kind", C.c_int32),
        ("axis", C.c_double * 3),
        ("origin_xyz", C.c_double * 3),
        ("origin_quat", C.c_double * 4),
        ("limit_lo", C.c_double),
        ("limit_hi", C.c_double),
        ("velocity_limit", C.c_double),
        ("effort_limit", C.c_double),
    ]


class Robot(C.Structure):
    _fields_ = [
        ("name", C.c_char * 64),
        ("n_joints", C.c_int32),
        ("joints", Joint * MAX_JOINTS),
        ("tip_xyz", C.c_double * 3),
        ("tip_quat", C.c_double * 4),
        ("jaw_joint", C.c_int32),
        ("dof", C.c_int32),
        ("dof_to_joint", C.c_int32 * MAX_JOINTS),
    ]

    def dof_joint(self, d: int) -> Joint:
        return self.joints[self.dof_to_joint[d]]


class Dyn(C.Structure):
    _fields_ = [
        ("control_dt", C.c_double),
        ("substeps", C.c_int32),
        ("control_mode", C.c_int32),
        ("kp", C.c_double * MAX_JOINTS),
        ("kd", C.c_double * MAX_JOINTS),
        ("inertia", C.c_double * MAX_JOINTS),
        ("damping", C.c_double * MAX_JOINTS),
    ]


class EnvCfg(C.Structure):
    _fields_ = [
        ("task", C.c_int32),
        ("n_envs", C.c_int64),
        ("episode_len", C.c_int32),
        ("goal_sigma", C.c_double),
        ("goal_offset_clip", C.c_double),
        ("reward_scale", C.c_double),
        ("path_penalty", C.c_double),
        ("success_radius", C.c_double),
        ("success_hold", C.c_int32),
        ("workspace_radius", C.c_double),
        ("waypoint_spacing", C.c_double),
        ("tracking_vel_noise_std", C.c_double),
        ("tracking_vel_clamp", C.c_double),
        ("seed", C.c_uint64),
        ("row_offset", C.c_int64),
        ("collision_threshold", C.c_double),
        ("collision_penalty", C.c_double),
        ("view_penalty", C.c_double),
        ("render_w", C.c_int32),
        ("render_h", C.c_int32),
        ("render_fov", C.c_double),
        ("render_near", C.c_double),
        ("render_far", C.c_double),
    ]


class Pose(C.Structure):
    _fields_ = [("xyz", C.c_double * 3), ("quat", C.c_double * 4)]


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def build() -> None:
    """Compile both oracle variants (make in oracle/)."""
    subprocess.run(["make", "-s", "-C", _HERE, "all"], check=True)


_P = C.POINTER
_d = _P(C.c_double)


def _ptr(a: np.ndarray, t=C.c_double):
    return a.ctypes.data_as(_P(t))


def _load(precision: str) -> C.CDLL:
    path = os.path.join(_BUILD, f"libsg_oracle_{precision}.so")
    if not os.path.exists(path):
        build()
    lib = C.CDLL(path)
    sig = {
        "sgo_pcg32_seed": (None, [_P(Pcg32), C.c_uint64, C.c_uint64]),
        "sgo_pcg32_next": (C.c_uint32, [_P(Pcg32)]),
        "sgo_pcg32_uniform": (C.c_double, [_P(Pcg32), C.c_double, C.c_double]),
        "sgo_pcg32_normal": (C.c_double, [_P(Pcg32)]),
        "sgo_make_stream": (None, [C.c_uint64, C.c_uint64, _P(Pcg32)]),
        "sgo_fill_uniform_actions": (None, [_P(Pcg32), _d, C.c_int64]),
        "sgo_fill_normals": (None, [_P(Pcg32), _d, C.c_int64]),
        "sgo_parse_robot": (C.c_int, [C.c_char_p, C.c_char_p, _P(Robot), C.c_char_p, C.c_int]),
        "sgo_jaw_dof": (C.c_int, [_P(Robot)]),
        "sgo_fk": (None, [_P(Robot), _d, _d, _d]),
        "sgo_fk_matrix": (None, [_P(Robot), _d, _d]),
        "sgo_default_dynamics": (None, [_P(Robot), _P(Dyn)]),
        "sgo_sim_create": (C.c_void_p, [_P(Robot), C.c_int64, C.c_uint64, C.c_uint64]),
        "sgo_sim_destroy": (None, [C.c_void_p]),
        "sgo_sim_step": (C.c_int, [C.c_void_p, _d, _P(Dyn), _P(C.c_int64)]),
        "sgo_sim_reset_rows": (None, [C.c_void_p, _P(C.c_uint8)]),
        "sgo_sim_get": (None, [C.c_void_p, _d, _d, _d]),
        "sgo_sim_set": (None, [C.c_void_p, _d, _d, _d]),
        "sgo_spline_waypoints": (C.c_int, [_d, C.c_double, C.c_double, C.c_double, _d, C.c_int]),
        "sgo_spline_arc_length": (C.c_double, [_d, C.c_double, C.c_double, C.c_int]),
        "sgo_env_cfg_default": (None, [_P(EnvCfg)]),
        "sgo_env_create": (C.c_void_p, [_P(EnvCfg), _P(Robot), _P(Dyn), C.c_int, C.c_char_p, C.c_int]),
        "sgo_env_destroy": (None, [C.c_void_p]),
        "sgo_env_obs_dim": (C.c_int, [C.c_void_p]),
        "sgo_env_action_dim": (C.c_int, [C.c_void_p]),
        "sgo_env_lanes": (C.c_int, [C.c_void_p]),
        "sgo_env_reset": (C.c_int, [C.c_void_p]),
        "sgo_env_step": (C.c_int, [C.c_void_p, _d]),
        "sgo_env_error": (C.c_char_p, [C.c_void_p]),
        "sgo_env_get_obs": (None, [C.c_void_p, _d, _d]),
        "sgo_env_get_result": (None, [C.c_void_p, _d, _P(C.c_uint8), _P(C.c_uint8), _d, _P(C.c_int64)]),
        "sgo_env_get_state": (None, [C.c_void_p, _d, _d, _d, _d, _d]),
        "sgo_env_get_counters": (None, [C.c_void_p, _P(C.c_int32), _P(C.c_int32), _P(C.c_int64),
                                        _P(C.c_int32), _P(C.c_int32)]),
        "sgo_env_get_rng": (None, [C.c_void_p, _P(C.c_uint64), _P(C.c_uint64)]),
        "sgo_env_get_waypoints": (C.c_int, [C.c_void_p, C.c_int64, _d, C.c_int]),
        "sgo_env_workspace": (None, [C.c_void_p, _d, _d]),
        "sgo_env_goal_draws": (C.c_int64, [C.c_void_p]),
        "sgo_env_set_state": (None, [C.c_void_p, _d, _d, _d]),
        "sgo_render": (None, [_d, _d, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, _d, C.c_int, _d]),
        "sgo_env_get_images": (None, [C.c_void_p, _d, _d, _d, _d]),
        "sgo_default_tool_bases": (None, [C.c_int, C.c_double, _P(Pose)]),
        "sgo_multi_tool_min_separation": (C.c_double, [_d, C.c_int]),
        "sgo_mt_env_create": (C.c_void_p, [_P(EnvCfg), _P(Robot), C.c_int, _P(Pose), _P(Dyn), C.c_int,
                                           C.c_char_p, C.c_int]),
        "sgo_mt_env_destroy": (None, [C.c_void_p]),
        "sgo_mt_env_dims": (None, [C.c_void_p, _P(C.c_int), _P(C.c_int), _P(C.c_int)]),
        "sgo_mt_env_reset": (C.c_int, [C.c_void_p]),
        "sgo_mt_env_step": (C.c_int, [C.c_void_p, _d]),
        "sgo_mt_env_error": (C.c_char_p, [C.c_void_p]),
        "sgo_mt_env_get_obs": (None, [C.c_void_p, _d, _d]),
        "sgo_mt_env_get_result": (None, [C.c_void_p, _d, _P(C.c_uint8), _P(C.c_uint8), _d, _P(C.c_int64)]),
        "sgo_mt_env_get_state": (None, [C.c_void_p, _d, _d, _d, _d, _d, _d]),
        "sgo_mt_env_get_counters": (None, [C.c_void_p, _P(C.c_int32), _P(C.c_int32), _P(C.c_int64)]),
        "sgo_mt_env_get_rng": (None, [C.c_void_p, _P(C.c_uint64), _P(C.c_uint64)]),
        "sgo_mt_env_workspace": (None, [C.c_void_p, _d, _d, _d]),
        "sgo_bench_sim": (C.c_int, [_P(EnvCfg), _P(Robot), C.c_int64, C.c_int, C.c_int, _d,
                                    _P(C.c_int64)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


_LIBS: dict[str, C.CDLL] = {}


def lib(precision: str = "f64") -> C.CDLL:
    if precision not in _LIBS:
        _LIBS[precision] = _load(precision)
    return _LIBS[precision]


# ---------------------------------------------------------------- rng

def make_stream(seed: int, stream_id: int, precision: str = "f64") -> Pcg32:
    r = Pcg32()
    lib(precision).sgo_make_stream(seed, stream_id, C.byref(r))
    return r


def pcg32(initstate: int, initseq: int) -> Pcg32:
    r = Pcg32()
    lib().sgo_pcg32_seed(C.byref(r), initstate, initseq)
    return r


def next_u32(r: Pcg32) -> int:
    return lib().sgo_pcg32_next(C.byref(r))


def uniform(r: Pcg32, lo: float, hi: float) -> float:
    return lib().sgo_pcg32_uniform(C.byref(r), lo, hi)


def normal(r: Pcg32) -> float:
    return lib().sgo_pcg32_normal(C.byref(r))


def fill_normals(r: Pcg32, n: int, a: int) -> np.ndarray:
    """n x a standard normals from one serial stream, row-major (ppo.cpp:264-270)."""
    out = np.empty((n, a), dtype=np.float64)
    lib().sgo_fill_normals(C.byref(r), _ptr(out), out.size)
    return out


def fill_uniform_actions(r: Pcg32, n: int, a: int) -> np.ndarray:
    out = np.empty((n, a), dtype=np.float64)
    lib().sgo_fill_uniform_actions(C.byref(r), _ptr(out), out.size)
    return out


# ---------------------------------------------------------------- robot

def parse_robot(text: str, origin: str = "inline") -> Robot:
    m = Robot()
    err = C.create_string_buffer(512)
    rc = lib().sgo_parse_robot(text.encode(), origin.encode(), C.byref(m), err, 512)
    if rc:
        raise OracleError(rc, err.value.decode())
    return m


def resolve_robot(name: str) -> Robot:
    with open(os.path.join(ASSETS, f"{name}.robot")) as f:
        return parse_robot(f.read(), f"builtin:{name}")


def fk(m: Robot, q, precision: str = "f64"):
    q = np.ascontiguousarray(q, dtype=np.float64)
    pos = np.zeros(3)
    quat = np.zeros(4)
    lib(precision).sgo_fk(C.byref(m), _ptr(q), _ptr(pos), _ptr(quat))
    return pos, quat


def fk_matrix(m: Robot, q) -> np.ndarray:
    q = np.ascontiguousarray(q, dtype=np.float64)
    out = np.zeros(16)
    lib().sgo_fk_matrix(C.byref(m), _ptr(q), _ptr(out))
    return out.reshape(4, 4)


def default_dynamics(m: Robot) -> Dyn:
    d = Dyn()
    lib().sgo_default_dynamics(C.byref(m), C.byref(d))
    return d


def mid_configuration(m: Robot) -> np.ndarray:
    return np.array([0.5 * (m.dof_joint(d).limit_lo + m.dof_joint(d).limit_hi) for d in range(m.dof)])


# ---------------------------------------------------------------- sim batch

class SimBatch:
    """Standalone SimBatch for the dynamics KATs (sim_batch.hpp:28-41)."""

    def __init__(self, m: Robot, n: int, seed: int, salt: int = 0, precision: str = "f64"):
        self._lib = lib(precision)
        self.m, self.n, self.dof = m, n, m.dof
        self._h = self._lib.sgo_sim_create(C.byref(m), n, seed, salt)

    def __del__(self):
        if getattr(self, "_h", None):
            self._lib.sgo_sim_destroy(self._h)
            self._h = None

    def step(self, actions: np.ndarray, cfg: Dyn) -> int:
        a = np.ascontiguousarray(actions, dtype=np.float64)
        sat = C.c_int64(0)
        rc = self._lib.sgo_sim_step(self._h, _ptr(a), C.byref(cfg), C.byref(sat))
        if rc:
            raise OracleError(1, "dynamics.step: non-finite action entry")
        return sat.value

    def reset_rows(self, mask) -> None:
        m = np.ascontiguousarray(mask, dtype=np.uint8)
        self._lib.sgo_sim_reset_rows(self._h, _ptr(m, C.c_uint8))

    def get(self):
        q = np.zeros((self.n, self.dof)); qd = np.zeros_like(q); qt = np.zeros_like(q)
        self._lib.sgo_sim_get(self._h, _ptr(q), _ptr(qd), _ptr(qt))
        return q, qd, qt

    def set(self, q=None, qd=None, qt=None) -> None:
        cv = lambda x: None if x is None else np.ascontiguousarray(x, dtype=np.float64)
        q, qd, qt = cv(q), cv(qd), cv(qt)
        self._lib.sgo_sim_set(self._h, _ptr(q) if q is not None else None,
                              _ptr(qd) if qd is not None else None,
                              _ptr(qt) if qt is not None else None)


# ---------------------------------------------------------------- spline

def spline_waypoints(coeffs, spacing: float, t0: float = 0.0, t1: float = 1.0, cap: int = 4096):
    c = np.ascontiguousarray(coeffs, dtype=np.float64).reshape(12)
    out = np.zeros((cap, 3))
    n = lib().sgo_spline_waypoints(_ptr(c), t0, t1, spacing, _ptr(out), cap)
    if n < 0:
        raise OracleError(2, "invalid spline or spacing")
    return out[: min(n, cap)].copy()


def spline_arc_length(coeffs, subdivisions: int = 1000, t0: float = 0.0, t1: float = 1.0) -> float:
    c = np.ascontiguousarray(coeffs, dtype=np.float64).reshape(12)
    return lib().sgo_spline_arc_length(_ptr(c), t0, t1, subdivisions)


# ---------------------------------------------------------------- env

def env_config(**kw) -> EnvCfg:
    c = EnvCfg()
    lib().sgo_env_cfg_default(C.byref(c))
    for k, v in kw.items():
        setattr(c, k, v)
    return c


class Env:
    """Oracle VecTaskEnv (envs.cpp) for TargetReaching / PathFollowing."""

    def __init__(self, cfg: EnvCfg, robot: Robot, dyn: Dyn | None = None, threads: int = 1,
                 precision: str = "f64"):
        self._lib = lib(precision)
        err = C.create_string_buffer(512)
        self._h = self._lib.sgo_env_create(C.byref(cfg), C.byref(robot),
                                           C.byref(dyn) if dyn is not None else None,
                                           threads, err, 512)
        if not self._h:
            raise OracleError(2, err.value.decode())
        self.n = cfg.n_envs
        self.obs_dim = self._lib.sgo_env_obs_dim(self._h)
        self.action_dim = self._lib.sgo_env_action_dim(self._h)
        self.lanes = self._lib.sgo_env_lanes(self._h)
        self.task = cfg.task

    def __del__(self):
        if getattr(self, "_h", None):
            self._lib.sgo_env_destroy(self._h)
            self._h = None

    def _check(self, rc: int):
        if rc:
            raise OracleError(rc, self._lib.sgo_env_error(self._h).decode())

    def reset(self) -> np.ndarray:
        self._check(self._lib.sgo_env_reset(self._h))
        return self.obs()[0]

    def step(self, actions: np.ndarray) -> None:
        a = np.ascontiguousarray(actions, dtype=np.float64)
        assert a.shape == (self.n, self.action_dim)
        self._check(self._lib.sgo_env_step(self._h, _ptr(a)))

    def obs(self):
        o = np.zeros((self.n, self.obs_dim)); t = np.zeros_like(o)
        self._lib.sgo_env_get_obs(self._h, _ptr(o), _ptr(t))
        return o, t

    def result(self):
        r = np.zeros(self.n); te = np.zeros(self.n)
        term = np.zeros(self.n, np.uint8); tout = np.zeros(self.n, np.uint8)
        sat = C.c_int64(0)
        self._lib.sgo_env_get_result(self._h, _ptr(r), _ptr(term, C.c_uint8), _ptr(tout, C.c_uint8),
                                     _ptr(te), C.byref(sat))
        return dict(rewards=r, terminated=term, timed_out=tout, task_error=te, saturations=sat.value)

    def state(self):
        A = self.action_dim
        q = np.zeros((self.n, A)); qd = np.zeros_like(q); qt = np.zeros_like(q)
        tips = np.zeros((self.n, 3)); goals = np.zeros((self.n, 3))
        self._lib.sgo_env_get_state(self._h, _ptr(q), _ptr(qd), _ptr(qt), _ptr(tips), _ptr(goals))
        return dict(q=q, qdot=qd, q_target=qt, tips=tips, goals=goals)

    def counters(self):
        i32 = lambda: np.zeros(self.n, np.int32)
        sc, hc, wi, wl = i32(), i32(), i32(), i32()
        ec = np.zeros(self.n, np.int64)
        self._lib.sgo_env_get_counters(self._h, _ptr(sc, C.c_int32), _ptr(hc, C.c_int32),
                                       _ptr(ec, C.c_int64), _ptr(wi, C.c_int32), _ptr(wl, C.c_int32))
        return dict(step_count=sc, hold_count=hc, episode_count=ec, waypoint_idx=wi, waypoint_len=wl)

    def rng(self):
        s = np.zeros(self.n, np.uint64); i = np.zeros(self.n, np.uint64)
        self._lib.sgo_env_get_rng(self._h, _ptr(s, C.c_uint64), _ptr(i, C.c_uint64))
        return s, i

    def waypoints(self, row: int, cap: int = 256) -> np.ndarray:
        out = np.zeros((cap, 3))
        n = self._lib.sgo_env_get_waypoints(self._h, row, _ptr(out), cap)
        return out[:n].copy()

    def workspace(self):
        c = np.zeros(3); r = C.c_double(0)
        self._lib.sgo_env_workspace(self._h, _ptr(c), C.byref(r))
        return c, r.value

    def images(self):
        """ImageMatching state: target / current images (n, w*h), scenes (n, 3, 5)
        {cx, cy, cz, radius, albedo}, target cameras (n, 7) xyz + wxyz."""
        wh = (self.obs_dim - 3 * self.action_dim - 3) // 2
        t = np.zeros((self.n, wh)); c = np.zeros_like(t)
        sc = np.zeros((self.n, 3, 5)); cam = np.zeros((self.n, 7))
        self._lib.sgo_env_get_images(self._h, _ptr(t), _ptr(c), _ptr(sc), _ptr(cam))
        return dict(target=t, current=c, scenes=sc, target_cameras=cam)

    def goal_draws(self) -> int:
        return self._lib.sgo_env_goal_draws(self._h)

    def set_state(self, q=None, qdot=None, q_target=None):
        cv = lambda x: None if x is None else np.ascontiguousarray(x, dtype=np.float64)
        q, qdot, q_target = cv(q), cv(qdot), cv(q_target)
        self._lib.sgo_env_set_state(self._h, _ptr(q) if q is not None else None,
                                    _ptr(qdot) if qdot is not None else None,
                                    _ptr(q_target) if q_target is not None else None)


def render(cam_pos, cam_quat, spheres, width=32, height=32, fov=1.0471975511965976, near=0.005, far=2.0,
           precision: str = "f64") -> np.ndarray:
    """render.cpp:34-67: spheres (k, 5) {cx, cy, cz, radius, albedo} -> (h, w) image."""
    sp = np.ascontiguousarray(np.asarray(spheres, dtype=np.float64).reshape(-1, 5))
    p = np.ascontiguousarray(cam_pos, dtype=np.float64)
    q = np.ascontiguousarray(cam_quat, dtype=np.float64)
    out = np.zeros(width * height)
    lib(precision).sgo_render(_ptr(p), _ptr(q), width, height, fov, near, far, _ptr(sp), len(sp), _ptr(out))
    return out.reshape(height, width)


def default_tool_bases(n_tools: int, workspace_radius: float) -> np.ndarray:
    """default_tool_bases (envs.cpp:101-116) as an (n_tools, 7) array: xyz, quat (w, x, y, z)."""
    arr = (Pose * n_tools)()
    lib().sgo_default_tool_bases(n_tools, workspace_radius, arr)
    return np.array([list(p.xyz) + list(p.quat) for p in arr])


def multi_tool_min_separation(tips) -> float:
    t = np.ascontiguousarray(tips, dtype=np.float64).reshape(-1, 3)
    return lib().sgo_multi_tool_min_separation(_ptr(t), len(t))


class MultiToolEnv:
    """Oracle VecTaskEnv for MultiToolReaching (envs.cpp:101-116, 304-360, 540-593):
    one SimBatch per tool (stream id = tool * 2^32 + global row), tool-major
    action / observation columns, base poses applied to every tip."""

    def __init__(self, cfg: EnvCfg, robots, bases=None, dyns=None, threads: int = 1,
                 precision: str = "f64"):
        self._lib = lib(precision)
        T = len(robots)
        arr = (Robot * T)(*robots)
        pb = None
        if bases is not None:
            b = np.asarray(bases, dtype=np.float64).reshape(T, 7)
            pb = (Pose * T)()
            for t in range(T):
                pb[t].xyz[:] = list(b[t, :3])
                pb[t].quat[:] = list(b[t, 3:])
        pd = (Dyn * T)(*dyns) if dyns is not None else None
        err = C.create_string_buffer(512)
        self._h = self._lib.sgo_mt_env_create(C.byref(cfg), arr, T, pb, pd, threads, err, 512)
        if not self._h:
            raise OracleError(2, err.value.decode())
        a, o, dofs = C.c_int(0), C.c_int(0), (C.c_int * T)()
        self._lib.sgo_mt_env_dims(self._h, C.byref(a), C.byref(o), dofs)
        self.n, self.n_tools = cfg.n_envs, T
        self.action_dim, self.obs_dim, self.dofs = a.value, o.value, list(dofs)

    def __del__(self):
        if getattr(self, "_h", None):
            self._lib.sgo_mt_env_destroy(self._h)
            self._h = None

    def _check(self, rc: int):
        if rc:
            raise OracleError(rc, self._lib.sgo_mt_env_error(self._h).decode())

    def reset(self) -> np.ndarray:
        self._check(self._lib.sgo_mt_env_reset(self._h))
        return self.obs()[0]

    def step(self, actions: np.ndarray) -> None:
        a = np.ascontiguousarray(actions, dtype=np.float64)
        assert a.shape == (self.n, self.action_dim)
        self._check(self._lib.sgo_mt_env_step(self._h, _ptr(a)))

    def obs(self):
        o = np.zeros((self.n, self.obs_dim)); t = np.zeros_like(o)
        self._lib.sgo_mt_env_get_obs(self._h, _ptr(o), _ptr(t))
        return o, t

    def result(self):
        r = np.zeros(self.n); te = np.zeros(self.n)
        term = np.zeros(self.n, np.uint8); tout = np.zeros(self.n, np.uint8)
        sat = C.c_int64(0)
        self._lib.sgo_mt_env_get_result(self._h, _ptr(r), _ptr(term, C.c_uint8), _ptr(tout, C.c_uint8),
                                        _ptr(te), C.byref(sat))
        return dict(rewards=r, terminated=term, timed_out=tout, task_error=te, saturations=sat.value)

    def state(self):
        A, T = self.action_dim, self.n_tools
        q = np.zeros((self.n, A)); qd = np.zeros_like(q); qt = np.zeros_like(q)
        tips = np.zeros((self.n, 3 * T)); goals = np.zeros_like(tips); axes = np.zeros_like(tips)
        self._lib.sgo_mt_env_get_state(self._h, _ptr(q), _ptr(qd), _ptr(qt), _ptr(tips), _ptr(goals),
                                       _ptr(axes))
        return dict(q=q, qdot=qd, q_target=qt, tips=tips, goals=goals, axes=axes)

    def counters(self):
        sc = np.zeros(self.n, np.int32); hc = np.zeros(self.n, np.int32)
        ec = np.zeros(self.n, np.int64)
        self._lib.sgo_mt_env_get_counters(self._h, _ptr(sc, C.c_int32), _ptr(hc, C.c_int32),
                                          _ptr(ec, C.c_int64))
        return dict(step_count=sc, hold_count=hc, episode_count=ec)

    def rng(self):
        s = np.zeros((self.n_tools, self.n), np.uint64); i = np.zeros_like(s)
        self._lib.sgo_mt_env_get_rng(self._h, _ptr(s, C.c_uint64), _ptr(i, C.c_uint64))
        return s, i

    def workspace(self):
        T = self.n_tools
        c = np.zeros((T, 3)); b = np.zeros((T, 7)); r = C.c_double(0)
        self._lib.sgo_mt_env_workspace(self._h, _ptr(c), C.byref(r), _ptr(b))
        return c, r.value, b


def bench_sim(cfg: EnvCfg, robot: Robot, total_steps: int, runs: int, threads: int,
              precision: str = "f64"):
    """bench.cpp:97-135 on host cores; returns (run_seconds, run_steps)."""
    secs = np.zeros(runs)
    steps = np.zeros(runs, np.int64)
    rc = lib(precision).sgo_bench_sim(C.byref(cfg), C.byref(robot), total_steps, runs, threads,
                                      _ptr(secs), _ptr(steps, C.c_int64))
    if rc:
        raise OracleError(rc, "oracle bench_sim failed")
    return secs, steps
