"""Generates tests/golden/*.json.

reference_kats.json: known-answer values transcribed from the reference's own
tests (file:line cited). oracle_digests.json: per-50-step digests of oracle
runs at BASELINE config 1 and small ECM / STAR cases; committed so the oracle
cannot drift silently (tests/test_oracle_env.py::test_golden_digests).
Run from the repo root: python tests/golden/make_golden.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from tests.test_oracle_env import _digest  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

kats = {
    "pcg32_42_54_first3": {"values": ["0xa15c02b7", "0x7b47f409", "0xba1d3330"],
                           "source": "proj/tests/test_rng_and_pool.cpp:25-31"},
    "fk_matrix_oracle": {"trials_per_robot": 1000, "stream": [2024, 11], "tol": 1e-9,
                         "source": "proj/tests/test_robot_model.cpp:139-151"},
    "quarter_turn": {"link": 0.37, "q": "pi/2", "tip": [0.0, 0.37, 0.0],
                     "source": "proj/tests/test_robot_model.cpp:129-137"},
    "saturation_count": {"actions": [[0.5, 1.5], [-2.0, 0.0], [1.0, -1.0]], "count": 2,
                         "source": "proj/tests/test_dynamics.cpp:165-173"},
    "straight_line_waypoints": {"c": [1, 0, 0], "spacing": 0.25, "count": 5,
                                "source": "proj/tests/test_spline.cpp:56-66"},
    "arc_length_closed_form": {"b": [0, 0.4, 0], "c": [1, 0, 0], "value": "0.5*(sqrt(1.64)+asinh(0.8)/0.8)",
                               "source": "proj/tests/test_spline.cpp:117-126"},
    "workspace_centres": {"psm": [0, 0, -0.296], "ecm": [0, 0, -0.315], "star": [0.23192, 0, 1.03534],
                          "source": "SURVEY.md Appendix E (probe of envs.cpp:161-162)"},
    "config1_goal_draws": {"value": 264, "source": "SURVEY.md Appendix E (256 resets + 8 rejections)"},
}

cases = [
    dict(name="config1_psm_reach", robot="psm", task=O.TARGET_REACHING, sigma=0.05, n=64, steps=1001, seed=0),
    dict(name="ecm_reach", robot="ecm", task=O.TARGET_REACHING, sigma=0.05, n=48, steps=650, seed=3),
    dict(name="star_path", robot="star", task=O.PATH_FOLLOWING, sigma=0.15, n=32, steps=620, seed=1),
]
for c in cases:
    c["rows"] = _digest(O, c["robot"], c["task"], c["sigma"], c["n"], c["steps"], c["seed"])

with open(os.path.join(HERE, "reference_kats.json"), "w") as f:
    json.dump(kats, f, indent=1)
with open(os.path.join(HERE, "oracle_digests.json"), "w") as f:
    json.dump({"generator": "tests/golden/make_golden.py", "cases": cases}, f, indent=1)
print("wrote", len(cases), "digest cases")
