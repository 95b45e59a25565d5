"""Oracle descriptor parser + FK vs the reference's robot-model tests
(proj/tests/test_robot_model.cpp)."""
import math
import os

import numpy as np
import pytest


def test_bundled_robots_joint_sequences(oracle):
    # test_robot_model.cpp:80-104
    psm = oracle.resolve_robot("psm")
    assert psm.dof == 7 and psm.jaw_joint == 6
    kinds = lambda m: "".join("P" if m.dof_joint(d).kind == 1 else "R" for d in range(m.dof))
    assert kinds(psm)[:6] == "RRPRRR" and kinds(psm)[6] == "R"
    import ctypes
    assert oracle.lib().sgo_jaw_dof(ctypes.byref(psm)) == 6
    ecm = oracle.resolve_robot("ecm")
    assert ecm.dof == 6 and ecm.jaw_joint == -1 and kinds(ecm) == "RRPRRR"
    star = oracle.resolve_robot("star")
    assert star.dof == 8 and kinds(star) == "R" * 8


def test_zero_configuration_composes_origins(oracle):
    # test_robot_model.cpp:119-127
    star = oracle.resolve_robot("star")
    pos, quat = oracle.fk(star, np.zeros(8))
    expected = sum(np.array(star.joints[i].origin_xyz[:]) for i in range(star.n_joints)) + np.array(star.tip_xyz[:])
    assert np.linalg.norm(pos - expected) < 1e-12
    assert abs(np.linalg.norm(quat) - 1.0) < 1e-9


def _one_link(length):
    return (f"[robot]\nname = onelink\n[joint]\nname = j0\nkind = revolute\naxis = 0 0 1\norigin_xyz = 0 0 0\n"
            f"origin_rpy = 0 0 0\nlimits = -3.14 3.14\nvelocity_limit = 1\neffort_limit = 1\n"
            f"[tool_tip]\nxyz = {length} 0 0\nrpy = 0 0 0\n")


def test_planar_quarter_turn(oracle):
    # test_robot_model.cpp:129-137
    m = oracle.parse_robot(_one_link(0.37))
    pos, _ = oracle.fk(m, [math.pi / 2])
    assert abs(pos[0]) < 1e-12 and abs(pos[1] - 0.37) < 1e-12 and abs(pos[2]) < 1e-12


def test_fk_matches_homogeneous_matrix_oracle(oracle):
    # test_robot_model.cpp:139-151: 1000 random in-limit q per robot, 1e-9
    rng = oracle.make_stream(2024, 11)
    for name in ("ecm", "psm", "star"):  # builtin_robot_names() order is embedding order; any order works
        m = oracle.resolve_robot(name)
        for _ in range(1000):
            q = [oracle.uniform(rng, m.dof_joint(d).limit_lo, m.dof_joint(d).limit_hi) for d in range(m.dof)]
            pos, quat = oracle.fk(m, q)
            M = oracle.fk_matrix(m, q)
            assert np.linalg.norm(pos - M[:3, 3]) < 1e-9
            w, x, y, z = quat
            R = np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                          [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                          [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])
            assert np.linalg.norm(R - M[:3, :3]) < 1e-9


def test_fk_position_continuity(oracle):
    # test_robot_model.cpp:241-255 (finite-difference Jacobian bound)
    rng = oracle.make_stream(31, 4)
    m = oracle.resolve_robot("star")
    h = 1e-6
    for _ in range(100):
        q = np.array([oracle.uniform(rng, m.dof_joint(d).limit_lo + 1e-5, m.dof_joint(d).limit_hi - 1e-5)
                      for d in range(m.dof)])
        J = np.stack([(oracle.fk(m, q + h * e)[0] - oracle.fk(m, q - h * e)[0]) / (2 * h) for e in np.eye(m.dof)], 1)
        dq = np.array([oracle.uniform(rng, -1, 1) for _ in range(m.dof)])
        dq *= 1e-6 / np.linalg.norm(dq)
        dp = oracle.fk(m, q + dq)[0] - oracle.fk(m, q)[0]
        assert np.linalg.norm(dp) <= 1.01 * np.linalg.norm(J) * np.linalg.norm(dq) + 1e-15


def test_descriptor_errors_carry_locations_and_names(oracle):
    # test_robot_model.cpp:285-319
    bad_limits = ("[robot]\nname = x\n[joint]\nname = bad\nkind = revolute\naxis = 0 0 1\norigin_xyz = 0 0 0\n"
                  "origin_rpy = 0 0 0\nlimits = 2 1\nvelocity_limit = 1\neffort_limit = 1\n"
                  "[tool_tip]\nxyz = 0 0 0\nrpy = 0 0 0\n")
    with pytest.raises(oracle.OracleError, match="bad"):
        oracle.parse_robot(bad_limits, "mem")
    with pytest.raises(oracle.OracleError, match="unit"):
        oracle.parse_robot(bad_limits.replace("axis = 0 0 1", "axis = 0 0 2").replace("limits = 2 1",
                                                                                       "limits = -1 1"), "mem")
    with pytest.raises(oracle.OracleError, match="somefile:3"):
        oracle.parse_robot("[robot]\nname = x\nbogus_key = 1\n", "somefile")


def test_mid_configuration_and_workspace_centres(oracle):
    # test_robot_model.cpp:321-329; SURVEY Appendix E centres
    star = oracle.resolve_robot("star")
    mid = oracle.mid_configuration(star)
    for d in range(star.dof):
        j = star.dof_joint(d)
        assert mid[d] == pytest.approx(0.5 * (j.limit_lo + j.limit_hi))
    expect = {"psm": (0, 0, -0.296), "ecm": (0, 0, -0.315), "star": (0.23192, 0, 1.03534)}
    for name, c in expect.items():
        m = oracle.resolve_robot(name)
        pos, _ = oracle.fk(m, oracle.mid_configuration(m))
        assert np.allclose(pos, c, atol=1e-5)


def test_assets_are_the_reference_descriptors(oracle):
    """assets/robots/*.robot are kept verbatim (north_star); the product embeds
    the same text. Joint limits parsed from disk equal the oracle's."""
    root = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "assets", "robots")
    for name in ("psm", "ecm", "star"):
        with open(os.path.join(root, f"{name}.robot")) as f:
            a = oracle.parse_robot(f.read(), name)
        b = oracle.resolve_robot(name)
        assert a.n_joints == b.n_joints
        for i in range(a.n_joints):
            assert a.joints[i].limit_lo == b.joints[i].limit_lo
            assert a.joints[i].limit_hi == b.joints[i].limit_hi
