"""C-ABI boundary checks that need no GPU: the library loads, exports every
symbol include/sg_env.h declares, and its host logic (descriptor parsing,
error mapping, config defaults) behaves like the reference."""
import ctypes

import pytest


def test_library_exports_every_header_symbol(sg):
    lib = sg.lib()
    syms = sg.header_symbols()
    assert len(syms) >= 25
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_library_is_the_in_tree_sm100a_build(sg):
    import os
    import subprocess
    path = sg.lib_path()
    assert os.path.dirname(path).endswith(os.path.join("paper_2310_04676_b200", "lib"))
    out = subprocess.run(["cuobjdump", "-lelf", path], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_config_defaults_match_reference(sg):
    # envs.hpp:42-63, dynamics.hpp:34-44
    c = sg.env_config()
    assert (c.task, c.n_envs, c.episode_len, c.success_hold) == (0, 1024, 300, 10)
    assert (c.goal_sigma, c.reward_scale, c.path_penalty, c.success_radius) == (0.05, -1.0, 1.0, 0.005)
    assert (c.workspace_radius, c.waypoint_spacing, c.seed) == (0.0, 0.02, 0)
    d, _ = sg.dyn_config()
    assert (d.control_dt, d.substeps, d.control_mode) == (0.01, 4, 0)


def test_builtin_robots_via_abi(sg):
    for name, dof, jaw in (("psm", 7, 6), ("ecm", 6, -1), ("star", 8, -1)):
        r = sg.Robot.resolve(name)
        assert (r.dof, r.jaw_dof) == (dof, jaw)


def test_descriptor_errors_map_to_config_error(sg):
    # robot_model.cpp:191-283 messages, errors.hpp exit-code classes
    with pytest.raises(sg.ConfigError, match="somefile:3: unknown \\[robot\\] field 'bogus_key'"):
        sg.Robot.parse("[robot]\nname = x\nbogus_key = 1\n", "somefile")
    bad = ("[robot]\nname = x\n[joint]\nname = bad\nkind = revolute\naxis = 0 0 1\norigin_xyz = 0 0 0\n"
           "origin_rpy = 0 0 0\nlimits = 2 1\nvelocity_limit = 1\neffort_limit = 1\n[tool_tip]\nxyz = 0 0 0\n")
    with pytest.raises(sg.ConfigError, match="joint 'bad': limit_lo must be < limit_hi"):
        sg.Robot.parse(bad, "mem")
    with pytest.raises(sg.ConfigError, match="unknown robot 'not_a_robot'"):
        sg.Robot.resolve("not_a_robot")
    with pytest.raises(sg.ConfigError, match="cannot open robot description"):
        sg.Robot.resolve("/no/such/robot.robot")
    with pytest.raises(sg.ConfigError, match="missing \\[tool_tip\\]"):
        sg.Robot.parse("[robot]\nname = x\n[joint]\nname = j\nkind = revolute\naxis = 0 0 1\n"
                       "origin_xyz = 0 0 0\norigin_rpy = 0 0 0\nlimits = -1 1\nvelocity_limit = 1\n"
                       "effort_limit = 1\n", "mem")


def test_abi_and_oracle_parsers_agree(sg, oracle):
    """Two independent parsers (product C++ / oracle C) accept and reject the
    same inputs."""
    cases = ["[robot]\nname = x\n[joint]\nname = j\nkind = fixed\norigin_xyz = 0 0 1\norigin_rpy = 0 0 0\n"
             "[tool_tip]\nxyz = 0 0 0\n",
             "[robot]\nname = x\n[joint]\nname = j\nkind = revolute\naxis = 1 0 0\norigin_xyz = 0 0 0\n"
             "origin_rpy = 0 0 0\nlimits = -1 1\nvelocity_limit = 1\neffort_limit = 1\nbogus = 2\n[tool_tip]\n"
             "xyz = 0 0 0\n",
             "[robot]\nname = x\nformat_version = 2\n",
             "[robot]\nname = x\n[joint]\nname = j\nkind = revolute\naxis = 1 0 0\norigin_xyz = 0 0\n",
             open(oracle.ASSETS + "/psm.robot").read()]
    for text in cases:
        ok_abi = ok_or = True
        try:
            sg.Robot.parse(text, "t")
        except sg.ConfigError:
            ok_abi = False
        try:
            oracle.parse_robot(text, "t")
        except oracle.OracleError:
            ok_or = False
        assert ok_abi == ok_or, text


def test_env_creation_fails_loudly_without_a_gpu(sg):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(sg.SimError, match="CUDA"):
        sg.VecTaskEnv(robots=("psm",), n_envs=16)


def test_env_config_validation_is_config_error(sg):
    # envs.cpp:65-81 validation happens before any device work
    with pytest.raises(sg.ConfigError, match="n_envs must be >= 1"):
        sg.VecTaskEnv(robots=("psm",), n_envs=0)
    with pytest.raises(sg.ConfigError, match="reward_scale"):
        sg.VecTaskEnv(robots=("psm",), n_envs=4, reward_scale=1.0)
    with pytest.raises(sg.ConfigError, match="requires exactly 1 robot"):
        sg.VecTaskEnv(robots=("psm", "ecm"), n_envs=4)


def test_cpp_dropin_compiles_and_links(sg, tmp_path):
    """include/sg/env.hpp (the scalpel_b200 BatchedEnv / VecTaskEnv surface)
    compiles with g++ and links against libsg_env.so."""
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    libdir = os.path.dirname(sg.lib_path())
    exe = str(tmp_path / "bench_sim_cpp")
    r = subprocess.run(["g++", "-std=c++17", "-O2", "-I", os.path.join(root, "include"),
                        os.path.join(root, "examples", "bench_sim_cpp.cpp"), f"-L{libdir}", "-lsg_env",
                        f"-Wl,-rpath,{libdir}", "-o", exe], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    import torch
    if not torch.cuda.is_available():  # no device: the binary must fail loudly, not fall back
        run = subprocess.run([exe, "64", "2"], capture_output=True, text=True)
        assert run.returncode == 1 and "CUDA" in run.stderr


def test_every_header_symbol_has_a_ctypes_signature(sg):
    """Guards against calling an entry point with ctypes' default int
    conversion (pointer truncation)."""
    missing = [s for s in sg.header_symbols() if s not in sg._SIGS]
    assert not missing, missing


def test_cpp_multitool_example_and_pose_conversion(sg, oracle, tmp_path):
    """examples/multitool_cpp.cpp (tool bases through scalpel_b200::EnvConfig)
    compiles and links; pose_from_xyz_rpy reproduces quat_from_rpy
    (geometry.hpp:45-49) as the oracle's default_tool_bases uses it."""
    import os
    import subprocess
    import numpy as np
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    libdir = os.path.dirname(sg.lib_path())
    inc = os.path.join(root, "include")
    exe = str(tmp_path / "multitool_cpp")
    r = subprocess.run(["g++", "-std=c++17", "-O2", "-I", inc, os.path.join(root, "examples", "multitool_cpp.cpp"),
                        f"-L{libdir}", "-lsg_env", f"-Wl,-rpath,{libdir}", "-o", exe], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    src = tmp_path / "pose.cpp"
    src.write_text('#include <cstdio>\n#include "sg/env.hpp"\nint main(){ auto p = scalpel_b200::pose_from_xyz_rpy('
                   '0, -0.3, 0.075, 0.9, 0, 0); auto q = scalpel_b200::pose_from_xyz_rpy(0, 0, 0, 0.1, -0.2, 0.3);\n'
                   'std::printf("%.17g %.17g %.17g %.17g %.17g %.17g %.17g %.17g\\n", p.orientation[0], p.orientation[1],'
                   ' p.orientation[2], p.orientation[3], q.orientation[0], q.orientation[1], q.orientation[2],'
                   ' q.orientation[3]); }\n')
    pe = str(tmp_path / "pose")
    r = subprocess.run(["g++", "-std=c++17", "-I", inc, str(src), f"-L{libdir}", "-lsg_env", f"-Wl,-rpath,{libdir}",
                        "-o", pe], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    vals = [float(x) for x in subprocess.run([pe], capture_output=True, text=True).stdout.split()]
    np.testing.assert_allclose(vals[:4], oracle.default_tool_bases(3, 0.15)[2, 3:], atol=1e-16)
    from tests.test_oracle_image import _quat_rpy
    np.testing.assert_allclose(vals[4:], _quat_rpy(0.1, -0.2, 0.3), atol=1e-15)
    import torch
    if not torch.cuda.is_available():
        run = subprocess.run([exe], capture_output=True, text=True)
        assert run.returncode == 1 and "CUDA" in run.stdout
