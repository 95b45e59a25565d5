"""Oracle spline / waypoint sampler vs the reference's spline tests
(proj/tests/test_spline.cpp)."""
import numpy as np
import pytest


def _coeffs(a=(0, 0, 0), b=(0, 0, 0), c=(0, 0, 0), d=(0, 0, 0)):
    return np.array([*a, *b, *c, *d], dtype=np.float64)


def _eval(cf, t):
    a, b, c, d = cf[0:3], cf[3:6], cf[6:9], cf[9:12]
    return ((a * t + b) * t + c) * t + d


def test_unit_speed_line_exact_multiples(oracle):
    # test_spline.cpp:56-66
    w = oracle.spline_waypoints(_coeffs(c=(1, 0, 0)), 0.25)
    assert len(w) == 5
    for k in range(5):
        assert w[k, 0] == pytest.approx(0.25 * k, rel=1e-6, abs=1e-12)
        assert w[k, 1] == 0 and w[k, 2] == 0


def test_constant_spline_single_point(oracle):
    # test_spline.cpp:68-74
    w = oracle.spline_waypoints(_coeffs(d=(0.1, -0.2, 0.3)), 0.05)
    assert len(w) == 1 and np.array_equal(w[0], [0.1, -0.2, 0.3])


def test_both_endpoints_included(oracle):
    # test_spline.cpp:76-86
    cf = _coeffs((0.2, -0.1, 0.05), (-0.3, 0.2, 0.1), (0.25, 0.15, -0.2), (1, 2, 3))
    w = oracle.spline_waypoints(cf, 0.03)
    assert len(w) >= 2
    assert np.linalg.norm(w[0] - _eval(cf, 0.0)) < 1e-12
    assert np.linalg.norm(w[-1] - _eval(cf, 1.0)) < 1e-12


def _chord(cf, pa, pb):
    ts = np.linspace(0, 1, 20001)
    pts = np.stack([_eval(cf, t) for t in ts])
    ta = ts[np.argmin(((pts - pa) ** 2).sum(1))]
    tb = ts[np.argmin(((pts - pb) ** 2).sum(1))]
    tt = np.linspace(ta, tb, 4001)
    seg = np.stack([_eval(cf, t) for t in tt])
    return np.linalg.norm(np.diff(seg, axis=0), axis=1).sum()


def test_gaps_match_spacing_within_one_percent(oracle):
    # test_spline.cpp:88-106 (20 random cubics from make_stream(99, 1))
    rng = oracle.make_stream(99, 1)
    for _ in range(20):
        cf = np.zeros(12)
        for k in range(3):
            cf[k] = oracle.uniform(rng, -0.5, 0.5)
            cf[3 + k] = oracle.uniform(rng, -0.5, 0.5)
            cf[6 + k] = oracle.uniform(rng, -0.3, 0.3)
            cf[9 + k] = oracle.uniform(rng, -0.1, 0.1)
        w = oracle.spline_waypoints(cf, 0.02)
        assert len(w) >= 3
        for i in range(0, len(w) - 2, 3):  # every 3rd gap keeps the CPU suite fast
            assert _chord(cf, w[i], w[i + 1]) == pytest.approx(0.02, rel=0.01)


def test_validation(oracle):
    # test_spline.cpp:108-115
    cf = _coeffs(c=(1, 0, 0))
    with pytest.raises(oracle.OracleError):
        oracle.spline_waypoints(cf, 0.0)
    with pytest.raises(oracle.OracleError):
        oracle.spline_waypoints(cf, -1.0)
    cf[0] = np.nan
    with pytest.raises(oracle.OracleError):
        oracle.spline_waypoints(cf, 0.1)


def test_arc_length_closed_form(oracle):
    # test_spline.cpp:117-126
    cf = _coeffs(b=(0, 0.4, 0), c=(1, 0, 0))
    expected = 0.5 * (np.sqrt(1.64) + np.arcsinh(0.8) / 0.8)
    assert oracle.spline_arc_length(cf, 200000) == pytest.approx(expected, rel=1e-6)
