"""Host-side setup of the product (computed on the CPU, uploaded once):
tableaus, problems, analytic solution — bitwise the reference's.
No device needed."""
import numpy as np
import pytest


def test_tableaus_bitwise(mp, ref):
    for name in ("4s3pA", "4s3pB", "4s3pC", "midpoint0", "midpoint1", "midpoint7"):
        t = mp.midpoint_corrected(int(name[8:])) if name.startswith("midpoint") else mp.builtin(name)
        r = ref.tableau(name)
        assert t.q == r["q"]
        assert np.array_equal(np.array(t.a_high), r["a_high"])
        assert np.array_equal(np.array(t.a_eps), r["a_eps"])
        assert np.array_equal(np.array(t.b), r["b"])
        assert np.array_equal(np.array(t.c), r["c"])
        assert mp.validate(t) == []


def test_validate_flags_violations(mp):
    t = mp.builtin("4s3pB")
    t.b = [0.5, 0.5, 0.5, 0.5]
    assert "sum(b) must be 1" in mp.validate(t)
    t = mp.builtin("4s3pB")
    t.a_high[0][0] = 0.25
    assert any("diagonal" in v for v in mp.validate(t))


@pytest.mark.parametrize("eq,n", [(0, 2), (0, 9), (1, 3), (1, 10)])
def test_problem_bitwise(mp, ref, eq, n):
    u0, g, h, gam = mp.make_problem("heat" if eq == 0 else "advection", n)
    ru0, rg, rh, rgam = ref.make_problem(eq, n)
    assert np.array_equal(u0, ru0) and h == rh and gam == rgam
    if eq == 0:
        assert np.array_equal(g, rg)
        assert np.array_equal(mp.heat_exact(n, 0.1), ref.heat_exact(n, 0.1))


def test_problem_too_small(mp):
    with pytest.raises(mp.DimensionTooSmall):
        mp.make_problem("heat", 1)
    with pytest.raises(mp.DimensionTooSmall):
        mp.make_problem("advection", 2)
