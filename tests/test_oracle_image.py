"""Oracle renderer and ImageMatching task (render.cpp:34-67, envs.cpp:269-295,
333-335, 513-523).

The renderer is pinned by the reference's own render tests
(proj/tests/test_render.cpp) re-run against the oracle, plus an independent
vectorised numpy restatement; the task's reset (scene draws, target view) and
reward are pinned by a Python restatement of envs.cpp on the oracle's streams.
"""
import math

import numpy as np
import pytest

W = H = 32
FOV = 1.0471975511965976


def _centroid(img):
    h, w = img.shape
    ys, xs = np.mgrid[0:h, 0:w]
    t = img.sum()
    return (img * (xs + 0.5)).sum() / t, (img * (ys + 0.5)).sum() / t


def _quat_rpy(roll, pitch, yaw):
    # AngleAxis(yaw, Z) * AngleAxis(pitch, Y) * AngleAxis(roll, X) (geometry.hpp:45-49)
    def qmul(a, b):
        w1, x1, y1, z1 = a
        w2, x2, y2, z2 = b
        return np.array([w1 * w2 - x1 * x2 - y1 * y2 - z1 * z2, w1 * x2 + x1 * w2 + y1 * z2 - z1 * y2,
                         w1 * y2 + y1 * w2 + z1 * x2 - x1 * z2, w1 * z2 + z1 * w2 + x1 * y2 - y1 * x2])
    qz = np.array([math.cos(yaw / 2), 0, 0, math.sin(yaw / 2)])
    qy = np.array([math.cos(pitch / 2), 0, math.sin(pitch / 2), 0])
    qx = np.array([math.cos(roll / 2), math.sin(roll / 2), 0, 0])
    return qmul(qmul(qz, qy), qx)


def _np_render(pos, R, spheres, w=W, h=H, fov=FOV, near=0.005, far=2.0):
    """Independent vectorised restatement of render.cpp:42-64."""
    f = 0.5 * w / math.tan(0.5 * fov)
    py, px = np.mgrid[0:h, 0:w]
    d = np.stack([(px + 0.5 - 0.5 * w) / f, -(py + 0.5 - 0.5 * h) / f, -np.ones((h, w))], -1) @ R.T
    d /= np.linalg.norm(d, axis=-1, keepdims=True)
    best = np.full((h, w), far)
    val = np.zeros((h, w))
    for c0, c1, c2, r, alb in spheres:
        oc = pos - np.array([c0, c1, c2])
        b = d @ oc
        disc = b * b - (oc @ oc - r * r)
        with np.errstate(invalid="ignore"):
            t = -b - np.sqrt(disc)
        hit = (disc >= 0) & (t >= near) & (t < best)
        n = (pos + t[..., None] * d - np.array([c0, c1, c2])) / r
        lam = -(n * d).sum(-1)
        best = np.where(hit, t, best)
        val = np.where(hit, np.where(lam > 0, alb * lam, 0.0), val)
    return val


def _rot(q):
    w, x, y, z = q
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                     [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                     [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])


I4 = [1.0, 0.0, 0.0, 0.0]


def test_render_on_axis_sphere_brightest_at_center(oracle):
    img = oracle.render([0, 0, 0], I4, [[0.0, 0.0, -0.5, 0.08, 1.0]])
    by, bx = np.unravel_index(np.argmax(img), img.shape)
    assert abs(bx - W // 2) <= 1 and abs(by - H // 2) <= 1
    assert img.max() > 0.9


def test_render_empty_frustum_is_background(oracle):
    assert (oracle.render([0, 0, 0], I4, [[0.0, 0.0, 0.5, 0.05, 1.0]]) == 0.0).all()


def test_render_lateral_shift_moves_centroid(oracle):
    z, d = 0.6, 0.04
    sph = [[0.0, 0.0, -z, 0.05, 1.0]]
    img0 = oracle.render([0, 0, 0], I4, sph, width=64, height=64)
    img1 = oracle.render([d, 0, 0], I4, sph, width=64, height=64)
    (cx0, cy0), (cx1, cy1) = _centroid(img0), _centroid(img1)
    f = 0.5 * 64 / math.tan(0.5 * FOV)
    assert abs((cx0 - cx1) - f * d / z) < 1.0 and abs(cy1 - cy0) < 0.5


def test_render_mirror_symmetric(oracle):
    sph = [[0.12, 0.03, -0.5, 0.06, 0.8], [-0.12, 0.03, -0.5, 0.06, 0.8], [0.0, -0.08, -0.4, 0.05, 1.0]]
    img = oracle.render([0, 0, 0], I4, sph)
    assert np.array_equal(img, img[:, ::-1])


def test_render_range_determinism_and_nearest(oracle):
    sph = [[0.05, -0.02, -0.3, 0.1, 0.9], [-0.1, 0.1, -0.7, 0.2, 0.4]]
    q = _quat_rpy(0.1, -0.2, 0.3)
    a = oracle.render([0.02, 0.01, 0.05], q, sph)
    b = oracle.render([0.02, 0.01, 0.05], q, sph)
    assert np.array_equal(a, b) and (a >= 0).all() and (a <= 1).all()
    img = oracle.render([0, 0, 0], I4, [[0, 0, -0.8, 0.2, 0.2], [0, 0, -0.3, 0.05, 1.0]])
    assert img[H // 2, W // 2] > 0.9


def test_render_matches_numpy_restatement(oracle):
    rng = np.random.default_rng(3)
    for _ in range(20):
        q = rng.normal(size=4)
        q /= np.linalg.norm(q)
        pos = rng.uniform(-0.05, 0.05, 3)
        sph = np.column_stack([rng.uniform(-0.2, 0.2, (4, 2)), rng.uniform(-0.9, 0.3, 4),
                               rng.uniform(0.02, 0.2, 4), rng.uniform(0.3, 1.0, 4)])
        np.testing.assert_allclose(oracle.render(pos, q, sph), _np_render(pos, _rot(q), sph), atol=1e-9)


def test_render_config_validation(oracle):
    m = oracle.resolve_robot("psm")
    for kw, msg in ((dict(render_w=4), "width and height"), (dict(render_near=0.0), "near < far"),
                    (dict(render_fov=3.2), "fov")):
        with pytest.raises(oracle.OracleError, match=msg):
            oracle.Env(oracle.env_config(n_envs=2, task=oracle.IMAGE_MATCHING, **kw), m)


def test_image_matching_reset_and_reward_restatement(oracle):
    """reset_row for ImageMatching (envs.cpp:304-316, 269-295): q (middle half),
    three spheres below the workspace drawn z, y, x (g++ argument order), radius,
    albedo; then a target q in the middle quarter and the target view; the
    current view from the reset q. Reward = -mean |current - target|."""
    m = oracle.resolve_robot("psm")
    n, seed, sigma = 6, 4, 0.05
    e = oracle.Env(oracle.env_config(n_envs=n, seed=seed, task=oracle.IMAGE_MATCHING), m)
    e.reset()
    im = e.images()
    center, radius = e.workspace()
    for i in range(n):
        r = oracle.make_stream(seed, i)
        q0 = []
        for d in range(m.dof):
            j = m.dof_joint(d)
            quarter = 0.25 * (j.limit_hi - j.limit_lo)
            q0.append(oracle.uniform(r, j.limit_lo + quarter, j.limit_hi - quarter))
        spheres = []
        for _ in range(3):
            z = -(radius + oracle.uniform(r, 0.1, 0.25))
            y = oracle.uniform(r, -2 * sigma, 2 * sigma)
            x = oracle.uniform(r, -2 * sigma, 2 * sigma)
            rad = oracle.uniform(r, 0.02, 0.05)
            alb = oracle.uniform(r, 0.5, 1.0)
            spheres.append([center[0] + x, center[1] + y, center[2] + z, rad, alb])
        np.testing.assert_array_equal(im["scenes"][i], spheres)
        qt = []
        for d in range(m.dof):
            j = m.dof_joint(d)
            margin = 0.5 * (1.0 - 0.25) * (j.limit_hi - j.limit_lo)
            qt.append(oracle.uniform(r, j.limit_lo + margin, j.limit_hi - margin))
        M = oracle.fk_matrix(m, qt)
        np.testing.assert_allclose(im["target_cameras"][i, :3], M[:3, 3], atol=1e-12)
        np.testing.assert_allclose(_rot(im["target_cameras"][i, 3:]), M[:3, :3], atol=1e-12)
        np.testing.assert_allclose(im["target"][i], _np_render(M[:3, 3], M[:3, :3], spheres).ravel(), atol=1e-9)
        M0 = oracle.fk_matrix(m, q0)
        np.testing.assert_allclose(im["current"][i], _np_render(M0[:3, 3], M0[:3, :3], spheres).ravel(), atol=1e-9)
        assert r.state == int(e.rng()[0][i])
    ar = oracle.make_stream(seed, 0xAC7104)
    e.step(oracle.fill_uniform_actions(ar, n, m.dof))
    im = e.images()
    res = e.result()
    err = np.abs(im["current"] - im["target"]).mean(1)
    np.testing.assert_allclose(res["rewards"], -err, atol=1e-15)
    np.testing.assert_allclose(res["task_error"], err, atol=1e-15)
    o = e.obs()[0]
    wh = W * H
    np.testing.assert_array_equal(o[:, 3 * m.dof + 3:3 * m.dof + 3 + wh], im["target"])
    np.testing.assert_array_equal(o[:, 3 * m.dof + 3 + wh:], im["current"])


def test_image_matching_episodes_only_time_out(oracle):
    """goal_met is never set for ImageMatching (envs.cpp:513-523): every env
    times out at step 300 and resets (new scene, new target)."""
    m = oracle.resolve_robot("ecm")
    e = oracle.Env(oracle.env_config(n_envs=8, seed=1, task=oracle.IMAGE_MATCHING, episode_len=20), m)
    e.reset()
    sc0 = e.images()["scenes"].copy()
    ar = oracle.make_stream(1, 0xAC7104)
    for s in range(20):
        e.step(oracle.fill_uniform_actions(ar, 8, m.dof))
        r = e.result()
        assert not r["terminated"].any()
        assert r["timed_out"].all() == (s == 19)
    assert not np.array_equal(e.images()["scenes"], sc0)
    assert (e.counters()["episode_count"] == 1).all()
