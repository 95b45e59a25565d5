"""Python plumbing over the C-ABI of include/sg_env.h (ctypes).

The product is the CUDA library ``lib/libsg_env.so`` (host C++ + sm_100a
kernels). This module only binds it for tests, the smoke check and bench.py:
device buffers owned by an env handle are exposed as zero-copy torch views via
``__cuda_array_interface__``. There is no fallback: if the library is missing
the import of :func:`lib` raises.

Names follow the reference's BatchedEnv / VecTaskEnv surface
(proj/include/scalpel/envs.hpp:107-179): ``n_envs``, ``obs_dim``,
``action_dim``, ``reset()``, ``step(actions)``, ``task_error()``, ``layout()``.
"""
from __future__ import annotations

import ctypes as C
import os
import re
from dataclasses import dataclass

import numpy as np

from . import _build

SG_OK, SG_ERR_SIM, SG_ERR_CONFIG = 0, 1, 2
TASKS = {"target_reaching": 0, "active_tracking": 1, "image_matching": 2, "path_following": 3,
         "multi_tool_reaching": 4}
CONTROL_MODES = {"position": 0, "velocity": 1, "torque": 2}


class ConfigError(RuntimeError):
    """scalpel::ConfigError / ParseError (exit code 2)."""


class SimError(RuntimeError):
    """scalpel::SimError (exit code 1)."""


class EnvConfig(C.Structure):  # sg_env_config
    _fields_ = [
        ("task", C.c_int32), ("episode_len", C.c_int32), ("n_envs", C.c_int64),
        ("goal_sigma", C.c_double), ("goal_offset_clip", C.c_double), ("reward_scale", C.c_double),
        ("path_penalty", C.c_double), ("success_radius", C.c_double), ("success_hold", C.c_int32),
        ("reserved0", C.c_int32), ("workspace_radius", C.c_double), ("waypoint_spacing", C.c_double),
        ("tracking_vel_noise_std", C.c_double), ("tracking_vel_clamp", C.c_double),
        ("collision_threshold", C.c_double), ("collision_penalty", C.c_double),
        ("view_penalty", C.c_double), ("seed", C.c_uint64), ("row_offset", C.c_int64),
        ("tool_bases", C.POINTER(C.c_double)), ("n_tool_bases", C.c_int32), ("reserved1", C.c_int32),
        ("render_width", C.c_int32), ("render_height", C.c_int32), ("render_fov", C.c_double),
        ("render_near", C.c_double), ("render_far", C.c_double),
    ]


class DynConfig(C.Structure):  # sg_dynamics_config
    _fields_ = [
        ("control_dt", C.c_double), ("substeps", C.c_int32), ("control_mode", C.c_int32),
        ("kp", C.POINTER(C.c_double)), ("n_kp", C.c_int32), ("n_kd", C.c_int32),
        ("kd", C.POINTER(C.c_double)), ("inertia", C.POINTER(C.c_double)), ("n_inertia", C.c_int32),
        ("n_damping", C.c_int32), ("damping", C.POINTER(C.c_double)),
    ]


class StepViews(C.Structure):  # sg_step_views
    _fields_ = [
        ("observations", C.c_void_p), ("terminal_observations", C.c_void_p), ("rewards", C.c_void_p),
        ("task_error", C.c_void_p), ("terminated", C.c_void_p), ("timed_out", C.c_void_p),
        ("action_saturations_total", C.c_void_p), ("n_envs", C.c_int64), ("obs_dim", C.c_int32),
        ("action_dim", C.c_int32),
    ]


class StepOut(C.Structure):  # sg_step_out
    _fields_ = [("observations", C.c_void_p), ("rewards", C.c_void_p), ("task_error", C.c_void_p),
                ("terminated", C.c_void_p), ("timed_out", C.c_void_p)]


class HostResult(C.Structure):  # sg_host_result
    _fields_ = [
        ("observations", C.c_void_p), ("terminal_observations", C.c_void_p), ("rewards", C.c_void_p),
        ("task_error", C.c_void_p), ("terminated", C.c_void_p), ("timed_out", C.c_void_p),
        ("action_saturations", C.c_int64),
    ]


class StateViews(C.Structure):  # sg_state_views
    _fields_ = [
        ("q", C.c_void_p), ("qdot", C.c_void_p), ("q_target", C.c_void_p), ("goals", C.c_void_p),
        ("tips", C.c_void_p), ("step_count", C.c_void_p), ("hold_count", C.c_void_p),
        ("episode_count", C.c_void_p), ("waypoint_idx", C.c_void_p), ("waypoint_len", C.c_void_p),
        ("waypoints", C.c_void_p), ("rng_state", C.c_void_p), ("rng_inc", C.c_void_p),
        ("waypoint_cap", C.c_int32), ("dof", C.c_int32), ("n_envs", C.c_int64),
        ("n_tools", C.c_int32), ("reserved", C.c_int32),
    ]


_P = C.POINTER
_SIGS = {
    "sg_last_error": (C.c_char_p, []),
    "sg_version": (C.c_char_p, []),
    "sg_env_config_init": (None, [_P(EnvConfig)]),
    "sg_dynamics_config_init": (None, [_P(DynConfig)]),
    "sg_env_create": (C.c_int, [_P(EnvConfig), _P(DynConfig), _P(C.c_char_p), C.c_int32, C.c_int32,
                                _P(C.c_void_p)]),
    "sg_env_create_from_text": (C.c_int, [_P(EnvConfig), _P(DynConfig), _P(C.c_char_p), _P(C.c_char_p),
                                          C.c_int32, C.c_int32, _P(C.c_void_p)]),
    "sg_env_destroy": (None, [C.c_void_p]),
    "sg_env_set_stream": (C.c_int, [C.c_void_p, C.c_void_p]),
    "sg_env_dims": (C.c_int, [C.c_void_p, _P(C.c_int64), _P(C.c_int32), _P(C.c_int32)]),
    "sg_env_layout_count": (C.c_int32, [C.c_void_p]),
    "sg_env_layout_field": (C.c_int, [C.c_void_p, C.c_int32, _P(C.c_char_p), _P(C.c_int32), _P(C.c_int32)]),
    "sg_env_workspace": (C.c_int, [C.c_void_p, _P(C.c_double), _P(C.c_double)]),
    "sg_env_images": (C.c_int, [C.c_void_p, _P(C.c_void_p), _P(C.c_void_p), _P(C.c_void_p), _P(C.c_int32),
                                _P(C.c_int32)]),
    "sg_env_tools": (C.c_int, [C.c_void_p, _P(C.c_int32), _P(C.c_double), _P(C.c_double), _P(C.c_int32)]),
    "sg_env_reset": (C.c_int, [C.c_void_p, _P(StepViews)]),
    "sg_env_reset_host": (C.c_int, [C.c_void_p, C.c_void_p]),
    "sg_host_alloc": (C.c_int, [C.c_size_t, _P(C.c_void_p)]),
    "sg_host_free": (C.c_int, [C.c_void_p]),
    "sg_env_step": (C.c_int, [C.c_void_p, C.c_void_p, _P(StepViews)]),
    "sg_env_step_into": (C.c_int, [C.c_void_p, C.c_void_p, _P(StepOut), _P(StepViews)]),
    "sg_env_step_host": (C.c_int, [C.c_void_p, C.c_void_p, _P(HostResult)]),
    "sg_env_task_error": (C.c_int, [C.c_void_p, _P(C.c_void_p)]),
    "sg_env_host_counters": (C.c_int, [C.c_void_p, _P(C.c_uint64), _P(C.c_uint64)]),
    "sg_env_state": (C.c_int, [C.c_void_p, _P(StateViews)]),
    "sg_env_synchronize": (C.c_int, [C.c_void_p]),
    "sg_env_bench_begin": (C.c_int, [C.c_void_p, C.c_uint64, C.c_int64, C.c_int64]),
    "sg_env_bench_step": (C.c_int, [C.c_void_p, C.c_int32]),
    "sg_env_bench_actions": (C.c_int, [C.c_void_p, _P(C.c_void_p)]),
    "sg_robot_parse": (C.c_int, [C.c_char_p, C.c_char_p, _P(C.c_void_p)]),
    "sg_robot_resolve": (C.c_int, [C.c_char_p, _P(C.c_void_p)]),
    "sg_robot_destroy": (None, [C.c_void_p]),
    "sg_robot_dof": (C.c_int, [C.c_void_p, _P(C.c_int32), _P(C.c_int32)]),
    "sg_robot_fk": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]),
    "sg_policy_create": (C.c_int, [C.c_int32, C.c_int32, _P(C.c_int32), C.c_int32, C.c_int32, _P(C.c_void_p)]),
    "sg_policy_destroy": (None, [C.c_void_p]),
    "sg_policy_param_count": (C.c_int, [C.c_void_p, _P(C.c_int64), _P(C.c_int64)]),
    "sg_policy_load_params": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "sg_policy_init_params": (C.c_int, [C.c_void_p, C.c_uint64, C.c_double, C.c_void_p]),
    "sg_policy_forward": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_void_p,
                                    C.c_void_p]),
    "sg_policy_last_error": (C.c_char_p, []),
    "sg_policy_bootstrap": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_void_p,
                                      C.c_void_p, C.c_void_p]),
    "sg_policy_sample": (C.c_int, [C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_uint64, C.c_uint64,
                                   C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p]),
    "sg_policy_act": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_uint64, C.c_uint64,
                                C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "sg_policy_act_bootstrap": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_uint64,
                                          C.c_uint64, C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p,
                                          C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                          C.c_void_p]),
    "sg_policy_noise": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p, C.c_uint64,
                                  C.c_void_p, C.c_void_p, C.c_void_p]),
    "sg_policy_act_noise": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_void_p,
                                      C.c_void_p, C.c_void_p, C.c_void_p]),
    "sg_policy_train_forward": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_void_p,
                                          C.c_void_p, C.c_void_p, C.c_void_p]),
    "sg_policy_set_param_layout": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "sg_policy_pack_wt": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "sg_policy_dgrad_elu": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_int32, C.c_void_p,
                                      C.c_void_p, C.c_int64, C.c_void_p]),
    "sg_policy_layer_backward": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_int32, C.c_void_p,
                                           C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32,
                                           C.c_void_p, C.c_void_p]),
    "sg_policy_backward_tail": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                          C.c_void_p, C.c_void_p, C.c_int64] + [C.c_void_p] * 6),
    "sg_elu_backward_colsum": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_void_p,
                                         C.c_void_p]),
    "sg_policy_wgrad": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, C.c_int64, C.c_void_p, C.c_int32,
                                  C.c_void_p, C.c_void_p]),
    "sg_adam_step": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p,
                               C.c_void_p, C.c_double, C.c_double, C.c_double, C.c_double, C.c_double, C.c_int64,
                               C.c_int32, C.c_double, C.c_double, C.c_void_p]),
    "sg_checkpoint_save": (C.c_int, [C.c_char_p, C.c_int32, C.c_int32, C.c_void_p, C.c_int32, C.c_char_p,
                                     C.c_char_p, C.c_void_p, C.c_int64]),
    "sg_checkpoint_load": (C.c_int, [C.c_char_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_char_p,
                                     C.c_int32, C.c_char_p, C.c_int32, C.c_void_p, C.c_int64, C.c_void_p]),
    "sg_elu_forward": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_void_p]),
    "sg_elu_backward": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_void_p]),
    "sg_ppo_gather": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, C.c_int32,
                                C.c_void_p,
                                C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                C.c_void_p, C.c_void_p]),
    "sg_ppo_loss": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                              C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_double, C.c_double,
                              C.c_double, C.c_double, C.c_double, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                              C.c_void_p, C.c_void_p]),
    "sg_compute_gae": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                 C.c_void_p, C.c_int32, C.c_int64, C.c_double, C.c_double, C.c_void_p,
                                 C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
}

_LIB: C.CDLL | None = None


def lib_path() -> str:
    return _build.LIB


def lib() -> C.CDLL:
    """Load libsg_env.so (building it first when the sources are newer).
    Raises if it cannot be built or loaded — there is no fallback path."""
    global _LIB
    if _LIB is None:
        path = os.environ.get("SG_LIB_PATH") or _build.LIB  # override: A/B experiments only
        if path == _build.LIB and (not os.path.exists(path) or os.environ.get("SG_REBUILD")):
            _build.build()
        L = C.CDLL(path)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = L
    return _LIB


def header_symbols() -> list[str]:
    """Every function declared in include/sg_env.h."""
    with open(os.path.join(_build.INCLUDE, "sg_env.h")) as f:
        text = f.read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sg_[a-z0-9_]+)\s*\(", text)))


def _check(rc: int) -> None:
    if rc == SG_OK:
        return
    msg = lib().sg_last_error().decode()
    if rc == SG_ERR_CONFIG:
        raise ConfigError(msg)
    raise SimError(msg)


class _CudaArray:
    """Minimal __cuda_array_interface__ carrier for a raw device pointer."""

    def __init__(self, ptr: int, shape: tuple, typestr: str):
        self.__cuda_array_interface__ = {"shape": shape, "typestr": typestr, "data": (int(ptr), False),
                                         "version": 3, "strides": None}


def device_view(ptr: int, shape: tuple, dtype: str, device: int = 0):
    """Zero-copy torch view of env-owned device memory (valid while the env lives)."""
    import torch
    typestr = {"f32": "<f4", "u8": "|u1", "i32": "<i4", "i64": "<i8", "u64": "<u8"}[dtype]
    if ptr is None or ptr == 0:
        return None
    return torch.as_tensor(_CudaArray(ptr, shape, typestr), device=f"cuda:{device}")


# ----------------------------------------------------------------------------- robot

class Robot:
    """Parsed descriptor (parse_robot / resolve_robot, robot_model.cpp:191-349)."""

    def __init__(self, handle: int):
        self._h = handle
        dof, jaw = C.c_int32(), C.c_int32()
        _check(lib().sg_robot_dof(self._h, C.byref(dof), C.byref(jaw)))
        self.dof, self.jaw_dof = dof.value, jaw.value

    @classmethod
    def parse(cls, text: str, origin: str = "inline") -> "Robot":
        h = C.c_void_p()
        _check(lib().sg_robot_parse(text.encode(), origin.encode(), C.byref(h)))
        return cls(h.value)

    @classmethod
    def resolve(cls, name_or_path: str) -> "Robot":
        h = C.c_void_p()
        _check(lib().sg_robot_resolve(name_or_path.encode(), C.byref(h)))
        return cls(h.value)

    def fk(self, q):
        """Batched device FK: q (n x dof, cuda fp32) -> tip positions (n x 3)."""
        import torch
        q = q.contiguous().to(torch.float32)
        out = torch.empty((q.shape[0], 3), device=q.device, dtype=torch.float32)
        stream = torch.cuda.current_stream(q.device).cuda_stream
        _check(lib().sg_robot_fk(self._h, q.data_ptr(), q.shape[0], out.data_ptr(), stream))
        return out

    def __del__(self):
        if getattr(self, "_h", None) and _LIB is not None:
            _LIB.sg_robot_destroy(self._h)
            self._h = None


# ----------------------------------------------------------------------------- env

@dataclass
class StepResult:
    """scalpel::StepResult (envs.hpp:82-89) as device views."""
    observations: object
    rewards: object
    terminated: object
    timed_out: object
    terminal_observations: object
    task_error: object
    saturations_total: object


def env_config(**kw) -> EnvConfig:
    """sg_env_config with the reference defaults; tool_bases: (T, 7) array-like
    of xyz + quaternion (w, x, y, z) per robot (kept alive on the struct)."""
    c = EnvConfig()
    lib().sg_env_config_init(C.byref(c))
    for k, v in kw.items():
        if k == "task" and isinstance(v, str):
            v = TASKS[v]
        if k == "tool_bases":
            b = np.ascontiguousarray(np.asarray(v, dtype=np.float64).reshape(-1, 7))
            c._tool_bases = b
            c.tool_bases = b.ctypes.data_as(C.POINTER(C.c_double))
            c.n_tool_bases = b.shape[0]
            continue
        setattr(c, k, v)
    return c


def dyn_config(control_dt=0.01, substeps=4, control_mode="position", kp=(), kd=(), inertia=(),
               damping=()) -> tuple[DynConfig, list]:
    d = DynConfig()
    lib().sg_dynamics_config_init(C.byref(d))
    d.control_dt, d.substeps = control_dt, substeps
    d.control_mode = CONTROL_MODES[control_mode] if isinstance(control_mode, str) else control_mode
    keep = []
    for name in ("kp", "kd", "inertia", "damping"):
        vals = list(locals()[name])
        arr = (C.c_double * max(len(vals), 1))(*vals)
        keep.append(arr)
        setattr(d, name, C.cast(arr, C.POINTER(C.c_double)))
        setattr(d, "n_" + name, len(vals))
    return d, keep


class VecTaskEnv:
    """Device-resident VecTaskEnv behind the C-ABI (envs.hpp:123-179)."""

    def __init__(self, robots=("psm",), device: int = 0, dynamics: dict | None = None,
                 robot_texts: list[str] | None = None, **cfg):
        self.device = device
        self.cfg = env_config(**cfg)
        dyn, self._keep = dyn_config(**(dynamics or {}))
        h = C.c_void_p()
        if robot_texts is not None:
            arr = (C.c_char_p * len(robot_texts))(*[t.encode() for t in robot_texts])
            org = (C.c_char_p * len(robot_texts))(*[f"inline{i}".encode() for i in range(len(robot_texts))])
            _check(lib().sg_env_create_from_text(C.byref(self.cfg), C.byref(dyn), arr, org, len(robot_texts),
                                                 device, C.byref(h)))
        else:
            arr = (C.c_char_p * len(robots))(*[r.encode() for r in robots])
            _check(lib().sg_env_create(C.byref(self.cfg), C.byref(dyn), arr, len(robots), device, C.byref(h)))
        self._h = h.value
        n, o, a = C.c_int64(), C.c_int32(), C.c_int32()
        _check(lib().sg_env_dims(self._h, C.byref(n), C.byref(o), C.byref(a)))
        self.n_envs, self.obs_dim, self.action_dim = n.value, o.value, a.value
        self._views = StepViews()
        self._stream = None

    def __del__(self):
        if getattr(self, "_h", None) and _LIB is not None:
            _LIB.sg_env_destroy(self._h)
            self._h = None

    # -- plumbing ------------------------------------------------------------
    def set_stream(self, stream) -> None:
        """Bind a torch.cuda.Stream (or None for the legacy default stream)."""
        self._stream = stream
        _check(lib().sg_env_set_stream(self._h, None if stream is None else stream.cuda_stream))

    def layout(self) -> list[tuple[str, int, int]]:
        out = []
        for i in range(lib().sg_env_layout_count(self._h)):
            name, off, ln = C.c_char_p(), C.c_int32(), C.c_int32()
            _check(lib().sg_env_layout_field(self._h, i, C.byref(name), C.byref(off), C.byref(ln)))
            out.append((name.value.decode(), off.value, ln.value))
        return out

    def workspace(self):
        c = (C.c_double * 3)()
        r = C.c_double()
        _check(lib().sg_env_workspace(self._h, c, C.byref(r)))
        return np.array(list(c)), r.value

    def tools(self):
        """(centers (T, 3), bases (T, 7) xyz + wxyz, dofs) per tool (envs.hpp:144)."""
        T = C.c_int32()
        _check(lib().sg_env_tools(self._h, C.byref(T), None, None, None))
        c, b, d = (C.c_double * (3 * T.value))(), (C.c_double * (7 * T.value))(), (C.c_int32 * T.value)()
        _check(lib().sg_env_tools(self._h, C.byref(T), c, b, d))
        return np.array(list(c)).reshape(-1, 3), np.array(list(b)).reshape(-1, 7), list(d)

    def images(self) -> dict:
        """ImageMatching task state: target images (n, h*w), scenes (n, 16),
        target cameras (n, 12) as device views."""
        t, sc, cam = C.c_void_p(), C.c_void_p(), C.c_void_p()
        w, h = C.c_int32(), C.c_int32()
        _check(lib().sg_env_images(self._h, C.byref(t), C.byref(sc), C.byref(cam), C.byref(w), C.byref(h)))
        n, d = self.n_envs, self.device
        return dict(target=device_view(t.value, (n, w.value * h.value), "f32", d),
                    scenes=device_view(sc.value, (n, 16), "f32", d),
                    target_cameras=device_view(cam.value, (n, 12), "f32", d), width=w.value, height=h.value)

    def _result(self) -> StepResult:
        v, n, o, d = self._views, self.n_envs, self.obs_dim, self.device
        return StepResult(
            observations=device_view(v.observations, (n, o), "f32", d),
            rewards=device_view(v.rewards, (n,), "f32", d),
            terminated=device_view(v.terminated, (n,), "u8", d),
            timed_out=device_view(v.timed_out, (n,), "u8", d),
            terminal_observations=device_view(v.terminal_observations, (n, o), "f32", d),
            task_error=device_view(v.task_error, (n,), "f32", d),
            saturations_total=device_view(v.action_saturations_total, (1,), "u64", d),
        )

    # -- BatchedEnv surface -----------------------------------------------------
    def reset(self):
        _check(lib().sg_env_reset(self._h, C.byref(self._views)))
        return self._result().observations

    def step(self, actions) -> StepResult:
        """actions: cuda fp32 tensor (n_envs x action_dim), row-major."""
        if tuple(actions.shape) != (self.n_envs, self.action_dim):
            raise SimError("env.step: action shape mismatch")
        if not actions.is_contiguous() or str(actions.dtype) != "torch.float32":
            raise SimError("env.step: actions must be contiguous float32")
        _check(lib().sg_env_step(self._h, actions.data_ptr(), C.byref(self._views)))
        return self._result()

    def step_into(self, actions, observations=None, rewards=None, task_error=None, terminated=None,
                  timed_out=None) -> StepResult:
        """sg_env_step_into: the step's results written straight into the given
        device tensors (e.g. rollout-buffer slots); None -> the env's buffers."""
        if tuple(actions.shape) != (self.n_envs, self.action_dim):
            raise SimError("env.step: action shape mismatch")
        ptr = lambda t: None if t is None else t.data_ptr()
        out = StepOut(ptr(observations), ptr(rewards), ptr(task_error), ptr(terminated), ptr(timed_out))
        _check(lib().sg_env_step_into(self._h, actions.data_ptr(), C.byref(out), C.byref(self._views)))
        return self._result()

    def step_host(self, actions: np.ndarray, out: dict | None = None) -> dict:
        """Host actions in, host StepResult out (synchronous; e2e path)."""
        a = np.ascontiguousarray(actions, dtype=np.float32)
        if a.shape != (self.n_envs, self.action_dim):
            raise SimError("env.step: action shape mismatch")
        n, o = self.n_envs, self.obs_dim
        if out is None:
            out = dict(observations=np.empty((n, o), np.float32),
                       terminal_observations=np.empty((n, o), np.float32),
                       rewards=np.empty(n, np.float32), task_error=np.empty(n, np.float32),
                       terminated=np.empty(n, np.uint8), timed_out=np.empty(n, np.uint8))
        hr = HostResult()
        for k in ("observations", "terminal_observations", "rewards", "task_error", "terminated", "timed_out"):
            arr = out.get(k)
            setattr(hr, k, None if arr is None else arr.ctypes.data)
        _check(lib().sg_env_step_host(self._h, a.ctypes.data, C.byref(hr)))
        out["action_saturations"] = hr.action_saturations
        return out

    def step_host_ptr(self, actions_ptr: int, hr: HostResult) -> None:
        """Raw-pointer variant (pinned buffers) used by bench.py's e2e leg."""
        _check(lib().sg_env_step_host(self._h, actions_ptr, C.byref(hr)))

    def host_counters(self) -> tuple[int, int]:
        """(ended rows, saturated entries) seen by step_host so far."""
        e, s_ = C.c_uint64(), C.c_uint64()
        _check(lib().sg_env_host_counters(self._h, C.byref(e), C.byref(s_)))
        return e.value, s_.value

    def task_error(self):
        p = C.c_void_p()
        _check(lib().sg_env_task_error(self._h, C.byref(p)))
        return device_view(p.value, (self.n_envs,), "f32", self.device)

    def synchronize(self) -> None:
        _check(lib().sg_env_synchronize(self._h))

    def state(self) -> dict:
        s = StateViews()
        _check(lib().sg_env_state(self._h, C.byref(s)))
        n, A, d = self.n_envs, self.action_dim, self.device
        cap, T = s.waypoint_cap, s.n_tools
        rng_shape = (n,) if T == 1 else (T, n)
        return dict(
            q=device_view(s.q, (A, n), "f32", d), qdot=device_view(s.qdot, (A, n), "f32", d),
            q_target=device_view(s.q_target, (A, n), "f32", d), goals=device_view(s.goals, (3 * T, n), "f32", d),
            tips=device_view(s.tips, (3 * T, n), "f32", d), step_count=device_view(s.step_count, (n,), "i32", d),
            hold_count=device_view(s.hold_count, (n,), "i32", d),
            episode_count=device_view(s.episode_count, (n,), "i64", d),
            waypoint_idx=device_view(s.waypoint_idx, (n,), "i32", d),
            waypoint_len=device_view(s.waypoint_len, (n,), "i32", d),
            waypoints=device_view(s.waypoints, (n, cap, 3), "f32", d) if cap else None,
            rng_state=device_view(s.rng_state, rng_shape, "u64", d),
            rng_inc=device_view(s.rng_inc, rng_shape, "u64", d),
            waypoint_cap=cap, n_tools=T,
        )

    # -- bench workload (bench.cpp:31-35,97-135) --------------------------------
    def bench_begin(self, seed: int, first_step: int = 0, global_n_envs: int | None = None) -> None:
        g = self.n_envs + self.cfg.row_offset if global_n_envs is None else global_n_envs
        _check(lib().sg_env_bench_begin(self._h, seed, first_step, g))

    def bench_step(self, k_steps: int = 1) -> None:
        _check(lib().sg_env_bench_step(self._h, k_steps))

    def bench_actions(self):
        p = C.c_void_p()
        _check(lib().sg_env_bench_actions(self._h, C.byref(p)))
        return device_view(p.value, (self.n_envs, self.action_dim), "f32", self.device)


# ----------------------------------------------------------------------------- policy

TRAIN_STREAM = 0x7261696E  # ppo.cpp:233
_M64 = (1 << 64) - 1


def make_stream(seed: int, stream_id: int) -> tuple[int, int]:
    """rng.hpp:69-83 on the host: splitmix64 of seed ^ (0x2545f4914f6cdd1d *
    (id + 1)) -> pcg32_srandom(initstate, initseq); returns PCG32 (state, inc)."""
    x = (seed ^ ((0x2545F4914F6CDD1D * (stream_id + 1)) & _M64)) & _M64

    def splitmix(x):
        x = (x + 0x9E3779B97F4A7C15) & _M64
        z = x
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
        return x, z ^ (z >> 31)

    x, a = splitmix(x)
    x, b = splitmix(x)
    inc = ((b << 1) | 1) & _M64
    s = inc  # 0 * mult + inc
    s = (s + a) & _M64
    s = (s * 6364136223846793005 + inc) & _M64
    return s, inc


def _pcheck(rc: int) -> None:
    if rc == SG_OK:
        return
    msg = lib().sg_policy_last_error().decode()
    raise (ConfigError if rc == SG_ERR_CONFIG else SimError)(msg)


class HostBuffer:
    """Pinned, device-mapped host memory from sg_host_alloc (the library's
    allocator for host-step buffers: sg_env_step_host resolves them without a
    CUDA pointer query). .tensor is a CPU torch view; freed with the object."""

    def __init__(self, shape, dtype):
        import torch
        self.shape = tuple(shape)
        itemsize = torch.empty((), dtype=dtype).element_size()
        nbytes = max(1, int(np.prod(self.shape)) * itemsize)
        p = C.c_void_p()
        _check(lib().sg_host_alloc(nbytes, C.byref(p)))
        self.ptr = p.value
        raw = (C.c_uint8 * nbytes).from_address(self.ptr)
        self.tensor = torch.frombuffer(raw, dtype=torch.uint8).view(dtype).view(self.shape)

    def __del__(self):
        if getattr(self, "ptr", None) and _LIB is not None:
            self.tensor = None
            _LIB.sg_host_free(self.ptr)
            self.ptr = None


class Policy:
    """Actor-critic MLP (policy.hpp:63-72) with the tcgen05 forward kernel.
    Parameters live in one flat fp32 vector in the reference's layout."""

    def __init__(self, obs_dim: int, action_dim: int, hidden=(256, 128, 64), device: int = 0):
        self.obs_dim, self.action_dim, self.device = obs_dim, action_dim, device
        hid = (C.c_int32 * len(hidden))(*hidden)
        h = C.c_void_p()
        _pcheck(lib().sg_policy_create(obs_dim, action_dim, hid, len(hidden), device, C.byref(h)))
        self._h = h.value
        cnt, ls = C.c_int64(), C.c_int64()
        _pcheck(lib().sg_policy_param_count(self._h, C.byref(cnt), C.byref(ls)))
        self.param_count, self.log_std_offset = cnt.value, ls.value

    def __del__(self):
        if getattr(self, "_h", None) and _LIB is not None:
            _LIB.sg_policy_destroy(self._h)
            self._h = None

    def init_params(self, seed: int, init_log_std: float = -1.0) -> np.ndarray:
        out = np.zeros(self.param_count, np.float32)
        _pcheck(lib().sg_policy_init_params(self._h, seed, init_log_std, out.ctypes.data))
        return out

    def load_params(self, flat) -> None:
        """flat: cuda fp32 tensor (param_count) in the reference layout."""
        import torch
        need = getattr(self, "_layout_numel", None)
        assert flat.is_cuda and flat.dtype == torch.float32
        assert flat.numel() == self.param_count if need is None else flat.numel() >= need
        stream = torch.cuda.current_stream(flat.device).cuda_stream
        _pcheck(lib().sg_policy_load_params(self._h, flat.contiguous().data_ptr(), stream))

    def forward(self, obs, mean=None, value=None):
        import torch
        n = obs.shape[0]
        if mean is None:
            mean = torch.empty((n, self.action_dim), device=obs.device, dtype=torch.float32)
        if value is None:
            value = torch.empty((n,), device=obs.device, dtype=torch.float32)
        stream = torch.cuda.current_stream(obs.device).cuda_stream
        _pcheck(lib().sg_policy_forward(self._h, obs.data_ptr(), n, obs.stride(0), mean.data_ptr(),
                                        value.data_ptr(), stream))
        return mean, value

    def act(self, obs, seed: int = 0, log_std=None, draw_pos: int = 0, step_offset: int = 0, want_mean: bool = False):
        """Fused forward + sampling (sg_policy_act): (actions, log_probs, value[, mean])."""
        import torch
        n = obs.shape[0]
        dev = obs.device
        A = self.action_dim
        if log_std is None:
            log_std = torch.full((A,), -1.0, device=dev)
        s0, inc = make_stream(seed, TRAIN_STREAM)
        pos = torch.tensor([draw_pos], dtype=torch.int64, device=dev)
        acts = torch.empty((n, A), device=dev)
        logp = torch.empty((n,), device=dev)
        value = torch.empty((n,), device=dev)
        mean = torch.empty((n, A), device=dev) if want_mean else None
        stream = torch.cuda.current_stream(dev).cuda_stream
        _pcheck(lib().sg_policy_act(self._h, obs.data_ptr(), n, obs.stride(0), log_std.data_ptr(), s0, inc,
                                    pos.data_ptr(), step_offset, acts.data_ptr(), logp.data_ptr(),
                                    mean.data_ptr() if want_mean else None, value.data_ptr(), stream))
        return (acts, logp, value, mean) if want_mean else (acts, logp, value)

    def sample(self, mean, seed: int = 0, log_std=None, draw_pos: int = 0, step_offset: int = 0):
        """Trainer rollout sampling (ppo.cpp:262-277): a = mean + exp(log_std) z,
        z from make_stream(seed, 0x7261696e) at draw draw_pos + step_offset +
        2 A e for env e; log_std defaults to the init value -1. Returns
        (actions, log_probs)."""
        import torch
        n, A = mean.shape
        dev = mean.device
        if log_std is None:
            log_std = torch.full((A,), -1.0, device=dev)
        s0, inc = make_stream(seed, TRAIN_STREAM)
        pos = torch.tensor([draw_pos], dtype=torch.int64, device=dev)
        acts = torch.empty((n, A), device=dev)
        logp = torch.empty((n,), device=dev)
        stream = torch.cuda.current_stream(dev).cuda_stream
        _pcheck(lib().sg_policy_sample(mean.data_ptr(), n, A, log_std.data_ptr(), s0, inc, pos.data_ptr(), step_offset,
                                       acts.data_ptr(), logp.data_ptr(), stream))
        return acts, logp

    def set_param_layout(self, layout, in_dims) -> None:
        """sg_policy_set_param_layout: pack from a trainer's (padded) flat
        layout. layout[k] = ((w_off, out, in), (b_off, out)) for k = trunk*4 + l."""
        w = (C.c_int64 * 8)(*[L[0][0] for L in layout])
        b = (C.c_int64 * 8)(*[L[1][0] for L in layout])
        o = (C.c_int32 * 8)(*[L[0][1] for L in layout])
        i = (C.c_int32 * 4)(*in_dims)
        _pcheck(lib().sg_policy_set_param_layout(self._h, w, b, i, o))
        self._layout_numel = max(L[1][0] + L[1][1] for L in layout)

    def train_forward(self, obs_bf16, h1, h2, h3, out) -> None:
        """sg_policy_train_forward into caller buffers (bf16 CUDA tensors)."""
        import torch
        stream = torch.cuda.current_stream(obs_bf16.device).cuda_stream
        _pcheck(lib().sg_policy_train_forward(self._h, obs_bf16.data_ptr(), obs_bf16.shape[0], obs_bf16.stride(0),
                                              h1.data_ptr(), h2.data_ptr(), h3.data_ptr(), out.data_ptr(), stream))

    def noise(self, n: int, seed: int = 0, log_std=None, draw_pos: int = 0, step_offset: int = 0, device: int = 0):
        """sg_policy_noise: the sampling's stream part ahead of the forward.
        Returns (scaled noise n x A fp64, log_probs n)."""
        import torch
        A = self.action_dim
        dev = f"cuda:{device}"
        if log_std is None:
            log_std = torch.full((A,), -1.0, device=dev)
        s0, inc = make_stream(seed, TRAIN_STREAM)
        pos = torch.tensor([draw_pos], dtype=torch.int64, device=dev)
        sz = torch.empty((n, A), dtype=torch.float64, device=dev)
        logp = torch.empty((n,), device=dev)
        stream = torch.cuda.current_stream(dev).cuda_stream
        _pcheck(lib().sg_policy_noise(self._h, n, log_std.data_ptr(), s0, inc, pos.data_ptr(), step_offset,
                                      sz.data_ptr(), logp.data_ptr(), stream))
        return sz, logp

    def act_noise(self, obs, scaled_noise, want_mean: bool = False):
        """sg_policy_act_noise: forward + actions = mean + scaled_noise.
        Returns (actions, value[, mean])."""
        import torch
        n, dev, A = obs.shape[0], obs.device, self.action_dim
        acts = torch.empty((n, A), device=dev)
        value = torch.empty((n,), device=dev)
        mean = torch.empty((n, A), device=dev) if want_mean else None
        stream = torch.cuda.current_stream(dev).cuda_stream
        _pcheck(lib().sg_policy_act_noise(self._h, obs.data_ptr(), n, obs.stride(0), scaled_noise.data_ptr(),
                                          acts.data_ptr(), mean.data_ptr() if want_mean else None, value.data_ptr(),
                                          stream))
        return (acts, value, mean) if want_mean else (acts, value)


# -- PPO update kernels (train.cu) ---------------------------------------------
def _dtype_code(t) -> int:
    import torch
    if t.dtype == torch.bfloat16:
        return 1
    if t.dtype == torch.float32:
        return 0
    raise SimError(f"unsupported dtype {t.dtype}")


def elu_forward(z, out=None):
    """ELU (policy.cpp:33) on the device kernel; out may alias z."""
    import torch
    out = torch.empty_like(z) if out is None else out
    stream = torch.cuda.current_stream(z.device).cuda_stream
    _pcheck(lib().sg_elu_forward(z.data_ptr(), out.data_ptr(), z.numel(), _dtype_code(z), stream))
    return out


def elu_backward(h, dh, out=None):
    """d ELU from the output h: dz = dh * (h > 0 ? 1 : h + 1)."""
    import torch
    out = torch.empty_like(h) if out is None else out
    stream = torch.cuda.current_stream(h.device).cuda_stream
    _pcheck(lib().sg_elu_backward(h.data_ptr(), dh.data_ptr(), out.data_ptr(), h.numel(), _dtype_code(h), stream))
    return out


class WtImages:
    """sg_policy_pack_wt images of the six hidden-layer weights (trunk x layer
    1..3) of a flat parameter vector, for sg_policy_dgrad_elu."""

    def __init__(self, layout, device):
        import torch
        self.dims, self.offs = [], []
        w_off, out_d, in_d = [], [], []
        off = 0
        for t in (0, 1):
            for l in (1, 2, 3):
                (w0, o, i), _ = layout[4 * t + l]
                w_off.append(w0)
                out_d.append(o)
                in_d.append(i)
                self.dims.append((o, i))
                self.offs.append(off)
                off += i * ((o + 15) // 16 * 16) * 2
        self.buf = torch.zeros(off, dtype=torch.uint8, device=device)
        self._w = (C.c_int64 * 6)(*w_off)
        self._o = (C.c_int32 * 6)(*out_d)
        self._i = (C.c_int32 * 6)(*in_d)

    def pack(self, flat) -> None:
        import torch
        stream = torch.cuda.current_stream(flat.device).cuda_stream
        _pcheck(lib().sg_policy_pack_wt(flat.data_ptr(), self._w, self._o, self._i, self.buf.data_ptr(), stream))

    def image(self, trunk: int, layer: int) -> int:
        return self.buf.data_ptr() + self.offs[3 * trunk + layer - 1]


def dgrad_elu(dy, wt_ptr: int, n_in: int, h, out=None):
    """sg_policy_dgrad_elu: (dy W) * ELU'(h) for one hidden layer (bf16)."""
    import torch
    m, k = dy.shape
    out = torch.empty((m, n_in), dtype=torch.bfloat16, device=dy.device) if out is None else out
    stream = torch.cuda.current_stream(dy.device).cuda_stream
    _pcheck(lib().sg_policy_dgrad_elu(dy.data_ptr(), dy.stride(0), k, wt_ptr, n_in, h.data_ptr(), out.data_ptr(), m,
                                      stream))
    return out


def layer_backward(dy, wt_ptr: int, n_in: int, h, colsum=None, wgrad=None, out=None, x0=None, wgrad0=None):
    """sg_policy_layer_backward: returns dz = (dy W) * ELU'(h); colsum (fp32
    [n_in], or None) += the column sums of dz; wgrad (fp32 [k x n_in], or
    None) += dy^T h. With x0 (bf16 [m x 32], the 256-wide layer only):
    wgrad0 (fp32 [256 x 32]) += dz^T x0 too and dz is not written (returns
    None). One launch, h / dz / x0 moved by TMA."""
    import torch
    m, k = dy.shape
    if x0 is None:
        out = torch.empty((m, n_in), dtype=torch.bfloat16, device=dy.device) if out is None else out
    else:
        assert x0.is_contiguous() and x0.dtype == torch.bfloat16 and tuple(x0.shape) == (m, 32)
        assert wgrad0.is_contiguous() and wgrad0.dtype == torch.float32 and tuple(wgrad0.shape) == (256, 32)
        out = None
    if wgrad is not None:
        assert wgrad.is_contiguous() and wgrad.dtype == torch.float32 and wgrad.shape[1] == n_in
        assert wgrad.shape[0] >= k
    stream = torch.cuda.current_stream(dy.device).cuda_stream
    _pcheck(lib().sg_policy_layer_backward(dy.data_ptr(), dy.stride(0), k, wt_ptr, n_in, h.data_ptr(),
                                           out.data_ptr() if out is not None else None, m,
                                           colsum.data_ptr() if colsum is not None else None,
                                           wgrad.data_ptr() if wgrad is not None else None,
                                           x0.data_ptr() if x0 is not None else None, 32,
                                           wgrad0.data_ptr() if wgrad0 is not None else None, stream))
    return out


def backward_tail(dy3, wt3_ptr: int, wt2_ptr: int, h3, h2, db3, dw3, db2, dw2, db1, out=None):
    """sg_policy_backward_tail: the last two layers' backward in one launch;
    returns dZ_1 (bf16 [m x 128]) and accumulates db3 / dw3 / db2 / dw2 / db1."""
    import torch
    m, k3 = dy3.shape
    out = torch.empty((m, 128), dtype=torch.bfloat16, device=dy3.device) if out is None else out
    for t, shape in ((dw3, (k3, 64)), (dw2, (64, 128))):
        assert t.is_contiguous() and t.dtype == torch.float32 and tuple(t.shape) == shape
    stream = torch.cuda.current_stream(dy3.device).cuda_stream
    _pcheck(lib().sg_policy_backward_tail(dy3.data_ptr(), dy3.stride(0), k3, wt3_ptr, wt2_ptr, h3.data_ptr(),
                                          h2.data_ptr(), out.data_ptr(), m, db3.data_ptr(), dw3.data_ptr(),
                                          db2.data_ptr(), dw2.data_ptr(), db1.data_ptr(), stream))
    return out


def elu_backward_colsum(h, dh, colsum, out=True):
    """sg_elu_backward_colsum: dz = dh * ELU'(h) (h None: dz = dh) and
    colsum += column sums of dz (fp32). Returns dz (or None with out=False)."""
    import torch
    m, n = dh.shape
    dz = torch.empty_like(dh) if out else None
    stream = torch.cuda.current_stream(dh.device).cuda_stream
    _pcheck(lib().sg_elu_backward_colsum(h.data_ptr() if h is not None else None, dh.data_ptr(),
                                         dz.data_ptr() if dz is not None else None, m, n, colsum.data_ptr(), stream))
    return dz


def wgrad(dy, x, partial, out):
    """sg_policy_wgrad: out (fp32 [o x i]) = dy^T x, dy bf16 [m x o], x bf16 [m x i]."""
    import torch
    m, o = dy.shape
    i = x.shape[1]
    parts = partial.numel() // (o * i)
    parts = min(parts, 148)
    stream = torch.cuda.current_stream(dy.device).cuda_stream
    _pcheck(lib().sg_policy_wgrad(dy.data_ptr(), o, x.data_ptr(), i, m, partial.data_ptr(), parts, out.data_ptr(),
                                  stream))


def ppo_gather(idx, obs, act, logp, adv, ret, obs_out, act_out, logp_out, adv_out, ret_out):
    """Minibatch gather (ppo.cpp:173-190) of the rollout buffer in one launch."""
    import torch
    stream = torch.cuda.current_stream(obs.device).cuda_stream
    _pcheck(lib().sg_ppo_gather(idx.data_ptr(), idx.numel(), obs.data_ptr(), obs.shape[1], obs_out.data_ptr(),
                                obs_out.shape[1], 1 if obs_out.dtype == torch.bfloat16 else 0, act.data_ptr(),
                                act.shape[1],
                                act_out.data_ptr(), logp.data_ptr(), logp_out.data_ptr(), adv.data_ptr(),
                                adv_out.data_ptr(), ret.data_ptr(), ret_out.data_ptr(), stream))


def ppo_loss(mean_full, value_full, log_std_raw, act, old_logp, adv, ret, A, clip_eps, value_coef, entropy_coef,
             ls_min, ls_max, dmean, dvalue, dls, acc, out):
    """ppo_loss_and_grad's data part (ppo.cpp:90-154) on the fused kernel:
    out = {loss, policy_loss, value_loss, entropy, kl, clip_fraction};
    dmean / dvalue / dls the analytic gradients (train.cu sg_ppo_loss)."""
    import torch
    stream = torch.cuda.current_stream(mean_full.device).cuda_stream
    _pcheck(lib().sg_ppo_loss(mean_full.data_ptr(), mean_full.shape[1], value_full.data_ptr(), value_full.shape[1],
                              _dtype_code(mean_full), log_std_raw.data_ptr(), act.data_ptr(), old_logp.data_ptr(),
                              adv.data_ptr(), ret.data_ptr(), mean_full.shape[0], A, clip_eps, value_coef,
                              entropy_coef, ls_min, ls_max, dmean.data_ptr(), dvalue.data_ptr(), dls.data_ptr(),
                              acc.data_ptr(), out.data_ptr(), stream))


# -- checkpoints (save_checkpoint / load_checkpoint, policy.cpp:220-295) -------
def save_checkpoint(path: str, params, obs_dim: int, action_dim: int, robot: str, task: str,
                    hidden=(256, 128, 64)) -> None:
    """Write the reference's SCLPCKP1 checkpoint from a flat parameter vector
    in the reference layout (any array-like; stored as fp64)."""
    p = np.ascontiguousarray(np.asarray(params, dtype=np.float64).reshape(-1))
    hid = (C.c_int32 * len(hidden))(*hidden)
    _pcheck(lib().sg_checkpoint_save(path.encode(), obs_dim, action_dim, hid, len(hidden), robot.encode(),
                                     task.encode(), p.ctypes.data, p.size))


def load_checkpoint(path: str) -> tuple[dict, np.ndarray]:
    """Read a SCLPCKP1 checkpoint: (meta {obs_dim, action_dim, hidden, robot,
    task}, fp64 flat parameters in the reference layout)."""
    od, ad, nh, cnt = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int64()
    hid = (C.c_int32 * 64)()
    robot, task = C.create_string_buffer(1 << 12), C.create_string_buffer(1 << 12)
    _pcheck(lib().sg_checkpoint_load(path.encode(), C.byref(od), C.byref(ad), hid, C.byref(nh), robot, 1 << 12,
                                     task, 1 << 12, None, 0, C.byref(cnt)))
    params = np.empty(cnt.value, np.float64)
    _pcheck(lib().sg_checkpoint_load(path.encode(), None, None, None, None, None, 0, None, 0, params.ctypes.data,
                                     params.size, None))
    meta = dict(obs_dim=od.value, action_dim=ad.value, hidden=tuple(hid[: nh.value]), robot=robot.value.decode(),
                task=task.value.decode())
    return meta, params
