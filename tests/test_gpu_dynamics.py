"""The reference's dynamics property tests (proj/tests/test_dynamics.cpp) run on
the DEVICE step through the C-ABI, in every control mode and on both kernel
families (the test chain runs on the generic-chain kernel with runtime joint
tables; PSM / ECM / STAR on their compile-time chains):

  torque-mode equilibrium exactly preserved        test_dynamics.cpp:79-90
  position mode converges to the mid-range target  :92-107
  full action hits the limit exactly, jaw snaps    :109-134
  energy dissipates in torque mode (zero input)    :186-207
  halving the substep ~halves the one-step error   :209-243
  stepping is bitwise reproducible                 :287-304 (here: across
                                                   launches and team layouts)

Joint state is written straight into the env's device state views; the
episode length is raised so no reset interferes."""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

TEST_CHAIN = (
    "[robot]\nname = chain\n"
    "[joint]\nname = r0\nkind = revolute\naxis = 0 0 1\norigin_xyz = 0 0 0\n"
    "origin_rpy = 0 0 0\nlimits = -1.5 1.5\nvelocity_limit = 4\neffort_limit = 40\n"
    "[joint]\nname = p1\nkind = prismatic\naxis = 0 0 -1\norigin_xyz = 0 0 -0.05\n"
    "origin_rpy = 0 0 0\nlimits = 0.1 0.5\nvelocity_limit = 0.6\neffort_limit = 100\n"
    "[tool_tip]\nxyz = 0 0 0\nrpy = 0 0 0\n")


def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")


def _env(sg, n, robot=None, text=None, seed=0, **dyn):
    kw = dict(n_envs=n, seed=seed, episode_len=100000, dynamics=dyn or None)
    if text is not None:
        return sg.VecTaskEnv(robot_texts=[text], **kw)
    return sg.VecTaskEnv(robots=(robot,), **kw)


def _step(env, actions):
    return env.step(torch.as_tensor(np.asarray(actions, dtype=np.float32)).cuda())


def test_torque_mode_equilibrium_exact(sg):
    _cuda()
    env = _env(sg, 4, text=TEST_CHAIN, control_mode="torque", damping=(0.0,))
    env.reset()
    st = env.state()
    q0 = st["q"].clone()
    st["qdot"].zero_()
    for _ in range(10):
        _step(env, np.zeros((4, 2)))
    torch.cuda.synchronize()
    st = env.state()
    assert torch.equal(st["q"], q0)
    assert not st["qdot"].any()


@pytest.mark.parametrize("robot", ["psm", "ecm", "star"])
def test_position_mode_converges_to_mid_range(sg, robot):
    _cuda()
    env = _env(sg, 8, robot=robot, seed=3)
    env.reset()
    A = env.action_dim
    for _ in range(500):  # zero action = the range midpoint (the jaw: closed)
        _step(env, np.zeros((8, A)))
    torch.cuda.synchronize()
    st = env.state()
    assert (st["q"] - st["q_target"]).abs().max().item() < 1e-3


def test_full_action_hits_the_limit_and_jaw_snaps(sg, oracle):
    _cuda()
    m = oracle.resolve_robot("psm")
    env = _env(sg, 1, robot="psm")
    env.reset()
    f32 = lambda v: float(np.float32(v))
    _step(env, np.ones((1, 7)))
    qt = env.state()["q_target"][:, 0].cpu().numpy()
    assert qt[2] == f32(m.dof_joint(2).limit_hi)  # prismatic insertion
    _step(env, -np.ones((1, 7)))
    qt = env.state()["q_target"][:, 0].cpu().numpy()
    assert qt[2] == f32(m.dof_joint(2).limit_lo)
    jaw = 6
    a = np.zeros((1, 7))
    a[0, jaw] = 0.37
    _step(env, a)
    assert env.state()["q_target"][jaw, 0].item() == f32(m.dof_joint(jaw).limit_hi)
    a[0, jaw] = -0.002
    _step(env, a)
    assert env.state()["q_target"][jaw, 0].item() == f32(m.dof_joint(jaw).limit_lo)


@pytest.mark.parametrize("text,robot", [(TEST_CHAIN, None), (None, "psm")])
def test_energy_dissipates_in_torque_mode(sg, oracle, text, robot):
    _cuda()
    n = 16
    env = _env(sg, n, robot=robot, text=text, seed=5, control_mode="torque")
    env.reset()
    A = env.action_dim
    m = oracle.parse_robot(text, "t") if text else oracle.resolve_robot(robot)
    rng = oracle.make_stream(6, 6)
    qd = np.array([[oracle.uniform(rng, -m.dof_joint(d).velocity_limit, m.dof_joint(d).velocity_limit)
                    for d in range(A)] for _ in range(n)], dtype=np.float32)
    env.state()["qdot"].copy_(torch.from_numpy(qd.T.copy()).cuda())
    prev = float((env.state()["qdot"].double() ** 2).sum())
    for _ in range(200):
        _step(env, np.zeros((n, A)))
        now = float((env.state()["qdot"].double() ** 2).sum())
        assert now <= prev + 1e-15
        prev = now
    assert prev < 0.5 * float((torch.from_numpy(qd).double() ** 2).sum())


def test_halving_the_substep_halves_the_one_step_error(sg, oracle):
    """One control step from the same state with 4, 8 and 512 substeps: the
    semi-implicit Euler error vs the 512-substep solution halves with the
    substep (mean ratio in (1.5, 2.5) over 60 trials, test_dynamics.cpp:209-243)."""
    _cuda()
    m = oracle.parse_robot(TEST_CHAIN, "t")
    rng = oracle.make_stream(13, 13)
    trials = 60
    q = np.zeros((trials, 2), dtype=np.float32)
    qd = np.zeros((trials, 2), dtype=np.float32)
    act = np.zeros((trials, 2), dtype=np.float32)
    for t in range(trials):
        for d in range(2):
            j = m.dof_joint(d)
            mid, span = 0.5 * (j.limit_lo + j.limit_hi), 0.2 * (j.limit_hi - j.limit_lo)
            q[t, d] = oracle.uniform(rng, mid - span, mid + span)
            qd[t, d] = oracle.uniform(rng, -0.2 * j.velocity_limit, 0.2 * j.velocity_limit)
        for d in range(2):
            act[t, d] = oracle.uniform(rng, -0.2, 0.2)
    out = {}
    for sub in (4, 8, 512):
        env = _env(sg, trials, text=TEST_CHAIN, substeps=sub)
        env.reset()
        st = env.state()
        st["q"].copy_(torch.from_numpy(q.T.copy()).cuda())
        st["qdot"].copy_(torch.from_numpy(qd.T.copy()).cuda())
        _step(env, act)
        out[sub] = env.state()["q"].double().cpu().numpy().T
    e_coarse = np.linalg.norm(out[4] - out[512], axis=1)
    e_fine = np.linalg.norm(out[8] - out[512], axis=1)
    assert (e_fine > 0).all()
    ratio = float(np.mean(e_coarse / e_fine))
    assert 1.5 < ratio < 2.5, ratio


@pytest.mark.parametrize("robot", ["psm", "star"])
def test_stepping_is_bitwise_reproducible_across_layouts(sg, robot):
    """Same seed and actions: identical state bit for bit, whether the steps run
    one launch per step or fused, and in the one-team-per-CTA or the packed
    four-teams-per-CTA layout (the per-env arithmetic does not depend on the
    thread mapping)."""
    _cuda()
    n = 300
    kw = dict(task="path_following", goal_sigma=0.15) if robot == "star" else {}
    res = []
    for layout in ("legacy", "packed"):
        os.environ["SG_TEAM_LAYOUT"] = layout
        try:
            env = sg.VecTaskEnv(robots=(robot,), n_envs=n, seed=11, **kw)
        finally:
            del os.environ["SG_TEAM_LAYOUT"]
        env.reset()
        env.bench_begin(11)
        for k in (1, 60, 1, 1, 250):
            env.bench_step(k)
        torch.cuda.synchronize()
        st = env.state()
        res.append({k: st[k].clone() for k in ("q", "qdot", "q_target", "tips", "goals", "rng_state", "step_count")}
                   | {"obs": env._result().observations.clone()})
    for k in res[0]:
        assert torch.equal(res[0][k], res[1][k]), k
