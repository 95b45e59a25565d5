"""The C++ surfaces on the device: the fp64 host-matrix drop-in
(include/sg/host_env.hpp, the reference's BatchedEnv / VecTaskEnv / StepResult
names and types, envs.hpp:82-118) driven by the reference's bench_sim loop
with make_stream(seed, 0xac7104) actions (include/sg/rng.hpp), compiled with
g++ against libsg_env.so and checked against the fp64 oracle; and the shipped
C++ examples build and run."""
import os
import subprocess

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2310_04676_b200", "lib")


def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")


def _compile(src, out):
    cmd = ["g++", "-std=c++17", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"), src, "-L", LIBDIR, "-lsg_env",
           f"-Wl,-rpath,{LIBDIR}", "-o", out]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_host_fp64_dropin_matches_oracle(sg, oracle, tmp_path):
    _cuda()
    sg.lib()  # builds libsg_env.so if needed
    exe = str(tmp_path / "host_env_parity")
    _compile(os.path.join(ROOT, "tests", "cpp", "host_env_parity.cpp"), exe)
    n, steps, seed = 64, 310, 0
    out = str(tmp_path / "res.bin")
    r = subprocess.run([exe, out, str(n), str(steps), str(seed)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    raw = open(out, "rb").read()
    head = np.frombuffer(raw[:32], dtype=np.int64)
    assert tuple(head[:2]) == (n, 27)
    off = 32
    first = np.frombuffer(raw[off:off + 8], dtype=np.float64)[0]
    off += 8
    take = lambda count, dt, size: (np.frombuffer(raw[off:off + count * size], dtype=dt), off + count * size)
    obs, off = take(n * 27, np.float64, 8)
    rew, off = take(n, np.float64, 8)
    err, off = take(n, np.float64, 8)
    term, off = take(n, np.uint8, 1)
    tout, off = take(n, np.uint8, 1)
    tobs, off = take(n * 27, np.float64, 8)
    obs, tobs = obs.reshape(n, 27), tobs.reshape(n, 27)

    m = oracle.resolve_robot("psm")
    ref = oracle.Env(oracle.env_config(n_envs=n, seed=seed), m)
    o0 = ref.reset()
    assert abs(first - o0[0, 0]) < 1e-6
    ar = oracle.make_stream(seed, 0xAC7104)
    ended = 0
    for _ in range(steps):
        ref.step(oracle.fill_uniform_actions(ar, n, m.dof).astype(np.float32).astype(np.float64))
        rr = ref.result()
        ended += int((rr["terminated"] | rr["timed_out"]).sum())
    rr = ref.result()
    o_ref, t_ref = ref.obs()
    np.testing.assert_array_equal(term, rr["terminated"])
    np.testing.assert_array_equal(tout, rr["timed_out"])
    assert head[2] == ended == n  # the step-300 burst
    assert head[3] == 0  # uniform actions in [-1, 1) never saturate
    assert np.abs(obs - o_ref).max() < 1e-4
    assert np.abs(rew - rr["rewards"]).max() < 2e-5
    assert np.abs(err - rr["task_error"]).max() < 2e-5


@pytest.mark.parametrize("example", ["bench_sim_cpp"])
def test_cpp_examples_build_and_run(sg, tmp_path, example):
    _cuda()
    sg.lib()
    exe = str(tmp_path / example)
    _compile(os.path.join(ROOT, "examples", f"{example}.cpp"), exe)
    r = subprocess.run([exe, "1024", "20"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr + r.stdout
    assert "env-steps/s" in r.stdout
