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
