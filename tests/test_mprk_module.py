"""`import mprk` (repo-root alias of the GPU-backed module under the
reference's Python module name): the reference's
Python callers find the same entry points and behaviour — tableau helpers and
rounding on the host, `integrate` on the B200 (bindings.cpp:130-147)."""
import json
import math
import os
import sys

import pytest

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def test_module_surface_and_host_helpers():
    import mprk

    for name in ("4s3pA", "4s3pB", "4s3pC"):
        t = mprk.builtin(name)
        assert (t.name, t.q) == (name, 4)
        assert mprk.validate(t) == []
    back = mprk.tableau_from_json(mprk.tableau_to_json(mprk.builtin("4s3pB")))
    assert json.loads(mprk.tableau_to_json(back))["name"] == "4s3pB"
    assert mprk.round_binary32(0.1) != 0.1 and abs(mprk.round_binary32(0.1) - 0.1) < 1e-8
    assert mprk.round_binary16(1.0) == 1.0 and math.isinf(mprk.round_binary16(1.0e6))
    t = mprk.builtin("4s3pA")
    t16 = mprk.truncate_eps(t, "f16")
    assert t16.name == "4s3pA+b16" and t16.a_high == t.a_high
    assert [x for r in t16.a_eps for x in r] != [x for r in t.a_eps for x in r]
    assert all(x == mprk.round_binary16(x) for r in t16.a_eps for x in r)
    for i in range(t16.q):  # (a plain running sum: Python's sum() compensates)
        acc = 0.0
        for j in range(t16.q):
            acc += t16.a_high[i][j] + t16.a_eps[i][j]
        assert t16.c[i] == acc
    with pytest.raises(ValueError):
        mprk.truncate_eps(t, "f8")
    assert issubclass(mprk.MprkError, Exception)


@pytest.mark.gpu
def test_integrate_through_the_alias(gpu):
    import mprk

    r = mprk.integrate(mprk.builtin("4s3pB"), "heat", 8, 0.025, 0.1, tol=1e-6)
    assert r["steps"] == 4 and not r["solver_failure"] and r["mean_iterations"] == 1.0
    assert 0.0 < r["error_l2"] <= r["error_max"] * (1 + 1e-12)
    assert len(r["state"]) == 8 ** 3
    assert r["timings"]["solver"]["count"] == 16
    a = mprk.integrate(mprk.midpoint_corrected(1), "advection", 8, 1.0 / 640.0, 8.0 / 640.0, tol=1e-3)
    assert a["steps"] == 8 and a["error_max"] is None and a["error_l2"] is None and not a["solver_failure"]
    t = mprk.builtin("4s3pB")
    with pytest.raises(ValueError):
        mprk.integrate(t, "plasma", 8, 0.025, 0.1)
    with pytest.raises(mprk.MprkError):
        mprk.integrate(t, "heat", 8, 0.03, 0.1)
    with pytest.raises(mprk.MprkError):
        mprk.integrate(t, "heat", 1, 0.025, 0.1)
