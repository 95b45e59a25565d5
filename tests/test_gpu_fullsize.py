"""Parity at the BASELINE sizes (configs 2-4: PSM 16,384 envs, ECM 65,536,
STAR path following 16,384) across a synchronized reset burst, with the
device's fused bench launches (the benchmarked path) against the fp64 oracle
stepping the same bench_sim action stream on all host cores.

Checked at launch boundaries: flags, step / hold / episode counters, waypoint
indices and every PCG32 stream bit-exact; joint state, tips, goals and
observations within the tolerances of tests/test_gpu_parity.py.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from tests.test_gpu_parity import TOL, _compare_obs, _soa  # noqa: E402


@pytest.mark.parametrize("robot,task,n,sigma", [
    ("psm", "target_reaching", 16384, 0.05),   # BASELINE configs[1]
    ("ecm", "target_reaching", 65536, 0.05),   # configs[2]
    ("star", "path_following", 16384, 0.15),   # configs[3] (one GPU's shard)
])
def test_baseline_size_fused_launches_match_oracle(sg, oracle, robot, task, n, sigma):
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    seed = 0
    otask = oracle.PATH_FOLLOWING if task == "path_following" else oracle.TARGET_REACHING
    m = oracle.resolve_robot(robot)
    ref = oracle.Env(oracle.env_config(n_envs=n, seed=seed, task=otask, goal_sigma=sigma), m, threads=0)
    env = sg.VecTaskEnv(robots=(robot,), n_envs=n, seed=seed, task=task, goal_sigma=sigma)
    ref.reset()
    env.reset()
    env.bench_begin(seed)
    ar = oracle.make_stream(seed, 0xAC7104)
    A = m.dof
    done = 0
    for k in (1, 149, 150, 10):  # warm-up step, then fused launches across the burst at step 300
        env.bench_step(k)
        for _ in range(k):
            ref.step(oracle.fill_uniform_actions(ar, n, A).astype(np.float32).astype(np.float64))
        done += k
        torch.cuda.synchronize()
        res, r = env._result(), ref.result()
        np.testing.assert_array_equal(res.timed_out.cpu().numpy(), r["timed_out"], err_msg=f"timed_out @{done}")
        np.testing.assert_array_equal(res.terminated.cpu().numpy(), r["terminated"], err_msg=f"terminated @{done}")
        st, c = env.state(), ref.counters()
        keys = ["step_count", "hold_count", "episode_count"] + (["waypoint_idx", "waypoint_len"]
                                                                 if task == "path_following" else [])
        for key in keys:
            np.testing.assert_array_equal(st[key].cpu().numpy(), c[key], err_msg=f"{key} @{done}")
        np.testing.assert_array_equal(st["rng_state"].cpu().numpy(), ref.rng()[0], err_msg=f"rng @{done}")
        sr = ref.state()
        for key in ("q", "qdot", "q_target", "tips", "goals"):
            tol = TOL[key] if key in TOL else TOL["tips"]
            err = np.abs(_soa(st[key]) - sr[key]).max()
            assert err <= tol, f"{robot} {key} err {err:.3e} @ step {done}"
        _compare_obs(res.observations.cpu().numpy(), ref.obs()[0], A, TOL)
        np.testing.assert_allclose(res.rewards.cpu().numpy(), r["rewards"], atol=TOL["reward"])
    assert done == 310 and (ref.counters()["episode_count"] == 1).all()


def test_multitool_16k_fused_launches_match_oracle(sg, oracle):
    """Trimanual MultiToolReaching at 16,384 envs (bench --config multitool):
    fused device launches vs the oracle across the reset burst (flags,
    counters, every tool's stream bit-exact; state / observations within
    tolerance; rewards may differ by exactly the collision penalty where the
    minimum tip separation ties the threshold)."""
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    robots, n, seed = ("psm", "psm", "ecm"), 16384, 0
    ms = [oracle.resolve_robot(r) for r in robots]
    ref = oracle.MultiToolEnv(oracle.env_config(n_envs=n, seed=seed, task=oracle.MULTI_TOOL), ms, threads=0)
    env = sg.VecTaskEnv(robots=robots, n_envs=n, seed=seed, task="multi_tool_reaching")
    ref.reset()
    env.reset()
    env.bench_begin(seed)
    ar = oracle.make_stream(seed, 0xAC7104)
    done = 0
    for k in (1, 149, 150, 10):
        env.bench_step(k)
        for _ in range(k):
            ref.step(oracle.fill_uniform_actions(ar, n, 20).astype(np.float32).astype(np.float64))
        done += k
        torch.cuda.synchronize()
        res, r = env._result(), ref.result()
        np.testing.assert_array_equal(res.timed_out.cpu().numpy(), r["timed_out"], err_msg=f"@{done}")
        np.testing.assert_array_equal(res.terminated.cpu().numpy(), r["terminated"], err_msg=f"@{done}")
        st, c = env.state(), ref.counters()
        for key in ("step_count", "hold_count", "episode_count"):
            np.testing.assert_array_equal(st[key].cpu().numpy(), c[key], err_msg=f"{key} @{done}")
        np.testing.assert_array_equal(st["rng_state"].cpu().numpy(), ref.rng()[0], err_msg=f"rng @{done}")
        sr = ref.state()
        for key in ("q", "qdot", "q_target"):
            assert np.abs(st[key].cpu().numpy().T - sr[key]).max() <= TOL[key], (key, done)
        for key in ("tips", "goals"):
            assert np.abs(st[key].cpu().numpy().T - sr[key]).max() <= TOL["tips"], (key, done)
        d = np.abs(res.rewards.cpu().numpy() - r["rewards"])
        off = d > TOL["reward"]
        assert (np.abs(d[off] - 1.0) <= TOL["reward"]).all() and off.sum() <= 4, (done, d[off][:4])
    assert done == 310 and (ref.counters()["episode_count"] == 1).all()
