"""Descriptor parser contract (robot_model.cpp:46-59, 133-161, 191-283): the
product parser (csrc/robot.cpp) and the oracle's independent C parser accept
the same descriptors and reject the rest with the same message and line, over
a corpus of malformed inputs that touches every error path and the number
grammar of `in >> double` (libstdc++ num_get: no inf / nan / hex; a malformed
token at the very end of a value is dropped, elsewhere it is an error)."""
import ctypes as C

import pytest

J = lambda **kw: "".join(f"{k} = {v}\n" for k, v in kw.items())
good_joint = J(name="j", kind="revolute", axis="0 0 1", origin_xyz="0 0 0", origin_rpy="0 0 0", limits="-1 1",
               velocity_limit="1", effort_limit="1")
def doc(*parts):
    return "".join(parts)
R = "[robot]\nname = x\n"
T = "[tool_tip]\nxyz = 0 0 0\n"
cases = [
    R + "[joint]\n" + good_joint + T,
    R + "[joint]\n" + good_joint + T + "[jaw]\njoint = 0\n",
    R + "[joint]\n" + good_joint + T + "[jaw]\njoint = 3\n",
    R + "[joint]\n" + good_joint.replace("revolute", "prismatic") + T + "[jaw]\njoint = 0\n",
    R + "[joint]\n" + good_joint + "[joint]\nname = f\nkind = fixed\norigin_xyz = 0 0 1\norigin_rpy = 0 0 0\n" + T,
    R + "[joint]\nname = f\nkind = fixed\norigin_xyz = 0 0 1\norigin_rpy = 0 0 0\nlimits = 0 1\n" + T,
    R + "[joint]\nname = f\nkind = fixed\naxis = 1 0 0\norigin_xyz = 0 0 1\norigin_rpy = 0 0 0\n" + T,
    R + "[joint]\nname = f\nkind = fixed\naxis = 1 0\norigin_xyz = 0 0 1\norigin_rpy = 0 0 0\n" + T,
    R + "[joint]\n" + good_joint.replace("name = j\n", "") + T,
    R + "[joint]\n" + good_joint.replace("kind = revolute\n", "") + T,
    R + "[joint]\n" + good_joint.replace("revolute", "spherical") + T,
    R + "[joint]\n" + good_joint.replace("axis = 0 0 1\n", "") + T,
    R + "[joint]\n" + good_joint.replace("axis = 0 0 1", "axis = 0 0 2") + T,
    R + "[joint]\n" + good_joint.replace("axis = 0 0 1", "axis = 0 0 1 4") + T,
    R + "[joint]\n" + good_joint.replace("axis = 0 0 1", "axis = 0 0 x") + T,
    R + "[joint]\n" + good_joint.replace("axis = 0 0 1", "axis = 0 0 1x") + T,
    R + "[joint]\n" + good_joint.replace("origin_xyz = 0 0 0\n", "") + T,
    R + "[joint]\n" + good_joint.replace("origin_rpy = 0 0 0\n", "") + T,
    R + "[joint]\n" + good_joint.replace("limits = -1 1\n", "") + T,
    R + "[joint]\n" + good_joint.replace("limits = -1 1", "limits = 1 1") + T,
    R + "[joint]\n" + good_joint.replace("velocity_limit = 1\n", "") + T,
    R + "[joint]\n" + good_joint.replace("velocity_limit = 1", "velocity_limit = 0") + T,
    R + "[joint]\n" + good_joint.replace("effort_limit = 1\n", "") + T,
    R + "[joint]\n" + good_joint.replace("effort_limit = 1", "effort_limit = -1") + T,
    R + "[joint]\n" + good_joint + "zeta = 1\nalpha = 2\n" + T,
    R + "[joint]\n" + good_joint + "name = again\n" + T,
    R + "[joint]\n" + "name = j\nkind = spherical\n" + T,
    R + "[joint]\n" + "kind = spherical\n" + T,
    R + "[joint]\n" + good_joint + "[tool_tip]\nxyz = 0 0 0\nrpy = 0.1 0.2 0.3\n",
    R + "[joint]\n" + good_joint + "[tool_tip]\nfoo = 1\n",
    R + "[joint]\n" + good_joint + "[tool_tip]\nxyz = 1 2\n",
    R + "[joint]\n" + good_joint + T + "[jaw]\nfoo = 1\n",
    R + "[joint]\n" + good_joint + T + "[jaw]\njoint = a\n",
    R + "[joint]\n" + good_joint,
    R + "[joint]\n" + good_joint + T + "[bogus]\n",
    R + "[joint]\n" + good_joint + T + "[jaw\n",
    "name = x\n",
    "[robot]\nname\n",
    "[robot]\nname =\n",
    "[robot]\n= x\n",
    "[robot]\nformat_version = 2\n",
    "[robot]\nformat_version = 1.5\n",
    "[robot]\nformat_version = a\n",
    "[robot]\nfoo = 1\n",
    "[robot]\n[joint]\n" + good_joint + T,
    "[robot]\nname = x\n" + T,
    "",
    "# only comment\n\n   \n",
    "  [robot]  \r\n name = y \r\n[joint]\r\n" + good_joint.replace("\n", "\r\n") + T,
    R + "[joint]\n" + good_joint + "[joint]\n" + good_joint.replace("name = j", "name = k").replace("limits = -1 1", "limits = 3 2") + T,
    R + "[joint]\n[joint]\n" + good_joint + T,
    R + "[joint]\n" + good_joint.replace("limits = -1 1", "limits = -1 1 2") + T,
    R + "[joint]\n" + good_joint.replace("velocity_limit = 1", "velocity_limit = 1 2") + T,
    R + "[joint]\n" + good_joint.replace("origin_rpy = 0 0 0", "origin_rpy = 0.1 0 0") + T,
    R + "[joint]\n" + good_joint.replace("limits = -1 1", "limits = -1e-1 .5") + T,
    R + "[joint]\n" + good_joint.replace("limits = -1 1", "limits = inf 1") + T,
    R + "[joint]\n" + good_joint.replace("limits = -1 1", "limits = 0x10 1") + T,
    R + "[joint]\n" + good_joint + T + "[robot]\nname = z\n",
    R + "[joint]\nname = j\nkind = revolute\naxis = 1 0 0\norigin_xyz = 0 0\n",
    R + "[joint]\n" + good_joint + "= 3\n" + T,
    R + "[joint]\n" + good_joint + "junk line\n" + T,
    R + "[joint]\n" + good_joint.replace("axis = 0 0 1", "axis = 0.6 0.8 0") + T,
]

# number grammar of formatted stream extraction, pinned by a g++ probe of
# `std::istringstream in(s); while (in >> x) ...; in.eof()` (libstdc++ 14)
NUMBER_CASES = {  # value of `limits` -> accepted (two numbers, lo < hi)
    "-1 1": True, "-1e-1 .5": True, "-1 1 -": True, "-1 1 +": True, "-1 1 .": True, "-1 1 1e": True,
    "-1 1 e": False, "-1 1e5x": False, "inf 1": False, "nan 1": False, "0x10 1": False, "- 1 2": False,
    "-1,1": False, "-1.2.3": True, "+-1 1": False, "-1 1 1": False, "-1": False, "-.5 5.": True,
}


def _parse_both(sg, oracle, text):
    try:
        r = sg.Robot.parse(text, "f.robot")
        d, j = C.c_int32(), C.c_int32()
        sg.lib().sg_robot_dof(r._h, C.byref(d), C.byref(j))
        ours = ("ok", d.value, j.value)
    except sg.ConfigError as e:
        ours = ("err", str(e))
    try:
        m = oracle.parse_robot(text, "f.robot")
        theirs = ("ok", m.dof)
    except oracle.OracleError as e:
        theirs = ("err", str(e))
    return ours, theirs


@pytest.mark.parametrize("k", range(len(cases)))
def test_parser_corpus_matches_oracle(sg, oracle, k):
    ours, theirs = _parse_both(sg, oracle, cases[k])
    assert ours[0] == theirs[0], (cases[k], ours, theirs)
    if ours[0] == "err":
        assert ours[1] == theirs[1]
    else:
        assert ours[1] == theirs[1]


@pytest.mark.parametrize("value,accepted", sorted(NUMBER_CASES.items()))
def test_number_grammar(sg, oracle, value, accepted):
    text = R + "[joint]\n" + good_joint.replace("limits = -1 1", "limits = " + value) + T
    ours, theirs = _parse_both(sg, oracle, text)
    assert (ours[0] == "ok") == accepted, (value, ours)
    assert ours[0] == theirs[0] and (ours[0] == "ok" or ours[1] == theirs[1]), (value, ours, theirs)
