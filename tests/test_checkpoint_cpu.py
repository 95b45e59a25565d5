"""Policy checkpoints in the reference's SCLPCKP1 format (policy.cpp:220-295):
byte layout written by an independent restatement of save_checkpoint, read
by the C-ABI; round trips; the reference's ConfigError cases. CPU only (the
C-ABI file functions need no GPU)."""
import struct

import numpy as np
import pytest

from paper_2310_04676_b200 import sg


def _param_count(obs, act, hidden):
    total = 0
    for trunk in (0, 1):
        i = obs
        for o in list(hidden) + [act if trunk == 0 else 1]:
            total += o * i + o
            i = o
    return total + act


def _write_reference(path, obs, act, hidden, robot, task, params, magic=b"SCLPCKP1", version=1, count=None):
    """save_checkpoint (policy.cpp:220-242), byte for byte."""
    with open(path, "wb") as f:
        f.write(magic)
        f.write(struct.pack("<IIII", version, obs, act, len(hidden)))
        f.write(struct.pack(f"<{len(hidden)}I", *hidden))
        for s in (robot, task):
            f.write(struct.pack("<I", len(s)) + s.encode())
        f.write(struct.pack("<Q", len(params) if count is None else count))
        f.write(np.asarray(params, "<f8").tobytes())


def test_reads_reference_layout_and_round_trips(tmp_path):
    obs, act, hidden = 27, 7, (256, 128, 64)
    n = _param_count(obs, act, hidden)
    assert n == 97167  # PSM policy parameter count
    p = np.random.default_rng(0).normal(size=n)
    ref = tmp_path / "ref.ckpt"
    _write_reference(ref, obs, act, hidden, "psm", "target_reaching", p)
    meta, q = sg.load_checkpoint(str(ref))
    assert meta == dict(obs_dim=obs, action_dim=act, hidden=hidden, robot="psm", task="target_reaching")
    assert np.array_equal(p, q)
    ours = tmp_path / "ours.ckpt"
    sg.save_checkpoint(str(ours), p, obs, act, "psm", "target_reaching")
    assert ours.read_bytes() == ref.read_bytes()  # byte-identical to the reference writer


@pytest.mark.parametrize("case,msg", [
    ("magic", "is not a scalpel checkpoint"),
    ("version", "unsupported version 2"),
    ("count", "parameter count does not match"),
    ("truncated", "is truncated"),
])
def test_reference_errors(tmp_path, case, msg):
    obs, act, hidden = 24, 6, (256, 128, 64)
    p = np.zeros(_param_count(obs, act, hidden))
    path = tmp_path / "bad.ckpt"
    kw = dict(magic=b"NOTACKPT") if case == "magic" else dict(version=2) if case == "version" else \
        dict(count=len(p) + 1) if case == "count" else {}
    _write_reference(path, obs, act, hidden, "ecm", "target_reaching", p, **kw)
    if case == "truncated":
        path.write_bytes(path.read_bytes()[:-8])
    with pytest.raises(sg.ConfigError, match=msg):
        sg.load_checkpoint(str(path))
    with pytest.raises(sg.ConfigError, match="cannot open checkpoint"):
        sg.load_checkpoint(str(tmp_path / "missing.ckpt"))
