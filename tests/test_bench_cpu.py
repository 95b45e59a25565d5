"""bench.py host logic without a GPU: roofline byte accounting, the shard plan
and the reference (CPU) arm."""
import json
import subprocess
import sys
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def test_step_bytes_psm():
    b = bench.step_bytes(7, 27, fused=250, reset_frac=1 / 300)
    assert b["per_launch"] == 3 * 7 * 4 * 2 + 36 + 32
    assert b["per_step"] == 28 + 108 + 8 + 2
    assert abs(b["per_env_step"] - (b["per_launch"] / 250 + 146 + b["per_reset"] / 300)) < 1e-9


def test_shard_plan_covers_global_rows():
    rows = []
    for r in range(8):
        p = bench.shard_plan(r, 8, 16384)
        assert p["global_n_envs"] == 8 * 16384
        rows.extend(range(p["row_offset"], p["row_offset"] + p["n_envs"]))
    assert rows == list(range(8 * 16384))


def test_reference_arm_runs_on_cpu():
    cfg = dict(robot="psm", task="target_reaching", n_envs=512, goal_sigma=0.05)
    rate, lanes, sample = bench.cpu_reference(cfg, steps=20, budget_s=0.5)
    assert rate > 0 and lanes >= 1 and "512 envs" in sample


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "4",
                          "--config", "psm"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "port"
    assert line["e2e"]["h2d_bytes_per_step"] == 0


def test_step_bytes_task_configs():
    """Per-tool state and the ImageMatching target read in the roofline bytes."""
    mt = bench.step_bytes(20, 78, fused=250, reset_frac=1 / 300, tools=3)
    assert mt["per_launch"] == 3 * 20 * 4 * 2 + 3 * 3 * 4 * 3 + 32
    im = bench.step_bytes(7, 2072, fused=250, reset_frac=1 / 300, step_read=4 * 1024)
    assert im["per_step"] == 28 + 2072 * 4 + 10 + 4096


def test_task_reference_arms_run_on_cpu():
    """The CPU baselines of the section-8f configs (oracle ports of the tasks)."""
    for name in ("multitool", "image"):
        cfg = dict(bench.CONFIGS[name], n_envs=64)
        rate, lanes, sample = bench.cpu_reference(cfg, steps=3, budget_s=0.5)
        assert rate > 0 and lanes >= 1 and "64 envs" in sample


def _json_lines(text):
    out = []
    for ln in text.splitlines():
        ln = ln.strip()
        if ln.startswith("{"):
            out.append(json.loads(ln))
    return out


def test_gpus_flag_spawns_ranks_dry_run():
    """`bench.py --gpus 2` outside torchrun launches two ranks itself
    (torch.distributed.run on 127.0.0.1) -- the driver's N>1 entry -- and the
    ranks agree on the shard plan and the max-over-ranks timing (gloo here)."""
    env = dict(os.environ, OMP_NUM_THREADS="1")
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = _json_lines(out.stdout)
    assert len(lines) == 1, out.stdout
    line = lines[0]
    assert line["n_gpus"] == 2 and line["backend"] == "gloo"
    rows = []
    for p in line["plans"]:
        rows.extend(range(p["row_offset"], p["row_offset"] + p["n_envs"]))
        assert p["global_n_envs"] == 2 * 16384
    assert rows == list(range(2 * 16384))
    assert line["max_time"] == 2.0


def test_gpus_flag_reference_arm_prints_one_line():
    """The reference arm under N ranks: rank 0 alone runs and prints."""
    env = dict(os.environ, OMP_NUM_THREADS="1")
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--impl", "reference",
                          "--steps", "3"], capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = _json_lines(out.stdout)
    assert len(lines) == 1 and lines[0]["impl"] == "reference" and lines[0]["n_gpus"] == 2


def test_contract_bytes_match_survey():
    """314 / 278 / 350 B per env-step (PSM / ECM / STAR)."""
    assert bench.contract_bytes(7, 27) == 314
    assert bench.contract_bytes(6, 24) == 278
    assert bench.contract_bytes(8, 30) == 350


def test_ppo_cpu_baseline_runs_on_cpu():
    """Config 5's CPU baseline (bounded sample of whole fp64 PPO iterations)
    runs on the host cores and reports env-steps/s with learning."""
    rate, lanes, sample = bench.cpu_ppo_reference(dict(bench.CONFIGS["ppo"]), budget_s=0.1, n_envs=32)
    assert rate > 0 and lanes >= 1 and "PPO iterations" in sample
