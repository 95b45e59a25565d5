"""Oracle PD dynamics vs the reference's dynamics tests
(proj/tests/test_dynamics.cpp)."""
import numpy as np
import pytest

CHAIN = ("[robot]\nname = chain\n"
         "[joint]\nname = r0\nkind = revolute\naxis = 0 0 1\norigin_xyz = 0 0 0\n"
         "origin_rpy = 0 0 0\nlimits = -1.5 1.5\nvelocity_limit = 4\neffort_limit = 40\n"
         "[joint]\nname = p1\nkind = prismatic\naxis = 0 0 -1\norigin_xyz = 0 0 -0.05\n"
         "origin_rpy = 0 0 0\nlimits = 0.1 0.5\nvelocity_limit = 0.6\neffort_limit = 100\n"
         "[tool_tip]\nxyz = 0 0 0\nrpy = 0 0 0\n")  # test_dynamics.cpp:45-54


@pytest.fixture
def chain(oracle):
    return oracle.parse_robot(CHAIN)


def test_default_gains_overdamped_stable_poles(oracle):
    # test_dynamics.cpp:27-43, 58-77
    for name in ("psm", "ecm", "star"):
        m = oracle.resolve_robot(name)
        cfg = oracle.default_dynamics(m)
        dt = cfg.control_dt / cfg.substeps
        for d in range(m.dof):
            kp, kd, c, mass = cfg.kp[d], cfg.kd[d], cfg.damping[d], cfg.inertia[d]
            a = 1.0 - dt * (kd + c) / mass
            b = -dt * kp / mass
            ev = np.linalg.eigvals(np.array([[1.0 + dt * b, dt * a], [b, a]]))
            assert np.all(np.abs(ev) < 0.999)
            assert np.all(np.abs(ev.imag) < 1e-9) and np.all(ev.real > 0)


def test_torque_equilibrium_exact(oracle, chain):
    # test_dynamics.cpp:79-90
    cfg = oracle.default_dynamics(chain)
    cfg.control_mode = oracle.TORQUE
    for d in range(chain.dof):
        cfg.damping[d] = 0.0
    sim = oracle.SimBatch(chain, 4, 1)
    q0 = sim.get()[0]
    for _ in range(10):
        sim.step(np.zeros((4, 2)), cfg)
    q, qd, _ = sim.get()
    assert np.array_equal(q, q0) and not qd.any()


def test_position_mode_converges(oracle):
    # test_dynamics.cpp:92-106
    for name in ("psm", "ecm", "star"):
        m = oracle.resolve_robot(name)
        cfg = oracle.default_dynamics(m)
        sim = oracle.SimBatch(m, 8, 3)
        sim.reset_rows(np.ones(8, np.uint8))
        for _ in range(500):
            sim.step(np.zeros((8, m.dof)), cfg)
        q, _, qt = sim.get()
        assert np.abs(q - qt).max() < 1e-3


def test_action_endpoints_exact(oracle, chain):
    # test_dynamics.cpp:108-118
    cfg = oracle.default_dynamics(chain)
    sim = oracle.SimBatch(chain, 1, 0)
    sim.step(np.ones((1, 2)), cfg)
    assert sim.get()[2][0, 1] == chain.dof_joint(1).limit_hi
    sim.step(-np.ones((1, 2)), cfg)
    assert sim.get()[2][0, 1] == chain.dof_joint(1).limit_lo


def test_jaw_snaps(oracle):
    # test_dynamics.cpp:120-132
    psm = oracle.resolve_robot("psm")
    cfg = oracle.default_dynamics(psm)
    sim = oracle.SimBatch(psm, 1, 0)
    a = np.zeros((1, 7))
    a[0, 6] = 0.37
    sim.step(a, cfg)
    assert sim.get()[2][0, 6] == psm.dof_joint(6).limit_hi
    a[0, 6] = -0.002
    sim.step(a, cfg)
    assert sim.get()[2][0, 6] == psm.dof_joint(6).limit_lo


def test_limits_hold_under_adversarial_actions(oracle):
    # test_dynamics.cpp:134-163: 3 control modes x 600 steps, actions U(-2, 2)
    m = oracle.resolve_robot("psm")
    cfg = oracle.default_dynamics(m)
    sim = oracle.SimBatch(m, 64, 99)
    sim.reset_rows(np.ones(64, np.uint8))
    rng = oracle.make_stream(42, 0)
    lo = np.array([m.dof_joint(d).limit_lo for d in range(7)])
    hi = np.array([m.dof_joint(d).limit_hi for d in range(7)])
    vl = np.array([m.dof_joint(d).velocity_limit for d in range(7)])
    for mode in (oracle.POSITION, oracle.VELOCITY, oracle.TORQUE):
        cfg.control_mode = mode
        for _ in range(600):
            a = 2.0 * oracle.fill_uniform_actions(rng, 64, 7)
            sim.step(a, cfg)
            q, qd, _ = sim.get()
            assert (q >= lo).all() and (q <= hi).all() and (np.abs(qd) <= vl).all()


def test_saturation_count(oracle, chain):
    # test_dynamics.cpp:165-173
    cfg = oracle.default_dynamics(chain)
    sim = oracle.SimBatch(chain, 3, 0)
    assert sim.step(np.array([[0.5, 1.5], [-2.0, 0.0], [1.0, -1.0]]), cfg) == 2


def test_nonfinite_action_is_error(oracle, chain):
    # test_dynamics.cpp:175-184
    cfg = oracle.default_dynamics(chain)
    sim = oracle.SimBatch(chain, 2, 0)
    a = np.zeros((2, 2))
    a[1, 1] = np.nan
    with pytest.raises(oracle.OracleError):
        sim.step(a, cfg)


def test_energy_dissipates_in_torque_mode(oracle, chain):
    # test_dynamics.cpp:186-208
    cfg = oracle.default_dynamics(chain)
    cfg.control_mode = oracle.TORQUE
    sim = oracle.SimBatch(chain, 16, 5)
    sim.reset_rows(np.ones(16, np.uint8))
    rng = oracle.make_stream(6, 6)
    q, qd, qt = sim.get()
    for i in range(16):
        for d in range(2):
            v = chain.dof_joint(d).velocity_limit
            qd[i, d] = oracle.uniform(rng, -v, v)
    sim.set(qd=qd)
    prev = (qd * qd).sum()
    for _ in range(200):
        sim.step(np.zeros((16, 2)), cfg)
        now = (sim.get()[1] ** 2).sum()
        assert now <= prev + 1e-15
        prev = now


def test_substep_ratio(oracle, chain):
    # test_dynamics.cpp:210-243: halving the substep roughly halves the error
    rng = oracle.make_stream(13, 13)
    ratios = []
    for _ in range(60):
        q0 = np.zeros((1, 2)); qd0 = np.zeros((1, 2))
        for d in range(2):
            j = chain.dof_joint(d)
            mid, span = 0.5 * (j.limit_lo + j.limit_hi), 0.2 * (j.limit_hi - j.limit_lo)
            q0[0, d] = oracle.uniform(rng, mid - span, mid + span)
            qd0[0, d] = oracle.uniform(rng, -0.2 * j.velocity_limit, 0.2 * j.velocity_limit)
        a = np.array([[oracle.uniform(rng, -0.2, 0.2) for _ in range(2)]])

        def run(sub):
            sim = oracle.SimBatch(chain, 1, 7)
            sim.set(q=q0, qd=qd0)
            cfg = oracle.default_dynamics(chain)
            cfg.substeps = sub
            sim.step(a, cfg)
            return sim.get()[0][0]

        coarse, fine, ref = run(4), run(8), run(512)
        ratios.append(np.linalg.norm(coarse - ref) / np.linalg.norm(fine - ref))
    assert 1.5 < np.mean(ratios) < 2.5


def test_reset_rows_masked_reproducible_middle_half(oracle):
    # test_dynamics.cpp:245-283
    m = oracle.resolve_robot("star")
    a = oracle.SimBatch(m, 8, 4242)
    q_before = a.get()[0]
    a.reset_rows(np.zeros(8, np.uint8))
    assert np.array_equal(a.get()[0], q_before)
    odd = np.array([i % 2 for i in range(8)], np.uint8)
    a.reset_rows(odd)
    assert np.array_equal(a.get()[0][::2], q_before[::2])
    b = oracle.SimBatch(m, 8, 4242)
    b.reset_rows(odd)
    assert np.array_equal(a.get()[0], b.get()[0])
    lo = np.array([m.dof_joint(d).limit_lo for d in range(8)])
    hi = np.array([m.dof_joint(d).limit_hi for d in range(8)])
    for _ in range(200):
        b.reset_rows(np.ones(8, np.uint8))
        q, qd, qt = b.get()
        assert (q >= lo + 0.25 * (hi - lo)).all() and (q <= hi - 0.25 * (hi - lo)).all()
        assert np.array_equal(qt, q) and not qd.any()


def test_env_step_bitwise_independent_of_lane_count(oracle):
    # test_dynamics.cpp:285-304 / thread_pool.hpp:28-31 — worker-count invariance
    m = oracle.resolve_robot("psm")
    outs = []
    for lanes in (1, 2, 5):
        e = oracle.Env(oracle.env_config(n_envs=600, seed=11), m, threads=lanes)
        e.reset()
        r = oracle.make_stream(0, 0)
        for _ in range(50):
            e.step(oracle.fill_uniform_actions(r, 600, 7))
        outs.append(e.obs()[0])
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])
