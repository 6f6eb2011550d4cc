"""Pin the CPU restatement (oracle/mprk_oracle.c) before trusting it.

1. Against the golden fixtures generated from the reference itself
   (tests/golden/make_golden.py) — always runs.
2. Against the reference library (oracle/_ref) on fresh seeded inputs,
   bit for bit — runs wherever the reference was compiled.
"""
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
G = np.load(os.path.join(HERE, "golden", "golden.npz"))
DT = {0: np.float32, 1: np.float64, 2: np.complex64, 3: np.complex128}


def same_bits(a, b):
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    return a.shape == b.shape and np.array_equal(a.view(np.uint8), b.view(np.uint8))


def tab(name):
    return dict(q=len(G[f"tab_{name}_b"]), a_high=G[f"tab_{name}_ah"], a_eps=G[f"tab_{name}_ae"],
                b=G[f"tab_{name}_b"])


# ---- 1. golden fixtures --------------------------------------------------------
def test_golden_problem(orc):
    for eq in (0, 1):
        u0, g, h, gam = orc.make_problem(eq, 6)
        assert same_bits(u0, G[f"prob{eq}_u0"])
        assert [h, gam] == G[f"prob{eq}_hg"].tolist()
        if eq == 0:
            assert same_bits(g, G["prob0_g"])


@pytest.mark.parametrize("kind", [0, 1, 2, 3])
def test_golden_kernels(orc, kind):
    n = 5
    x, q = G[f"k{kind}_x"], G[f"k{kind}_q"]
    for st in (0, 1):
        assert same_bits(orc.stencil(kind, n, st, 1.0, -0.37, x), G[f"k{kind}_stencil{st}"])
    for side in range(3):
        assert same_bits(orc.tensor(kind, side, n, q, x), G[f"k{kind}_tensor{side}"])
    tau = 0.01 if kind <= 1 else 1.0 / 640.0
    assert same_bits(orc.fastdiag(kind, n, tau, 0.5, x), G[f"k{kind}_fastdiag"])


@pytest.mark.parametrize("kind,solver", [(0, 0), (1, 0), (2, 1), (3, 1)])
@pytest.mark.parametrize("tol", [1e-3, 1e-8])
def test_golden_solves(orc, kind, solver, tol):
    key = f"solve{kind}_{tol:g}"
    tau = 0.025 if kind <= 1 else 1.0 / 640.0
    b = G[key + "_b"].astype(DT[kind])
    x, rep = orc.stage_solve(kind, solver, 6, tau, 0.5, 1, b, b, tol, 40)
    assert same_bits(x, G[key + "_x"])
    assert np.array_equal(rep["history"], G[key + "_hist"])
    meta = G[key + "_meta"]
    assert [rep["iterations"], rep["converged"], rep["failure"], rep["true_residual"]] == meta.tolist()


@pytest.mark.parametrize("name,eq,prec", [("midpoint1", 0, "f32"), ("4s3pB", 0, "f64"), ("4s3pC", 1, "f32")])
def test_golden_steps(orc, name, eq, prec):
    tau = 0.01 if eq == 0 else 1.0 / 640.0
    s = orc.stepper(eq, 6, tab(name), tau, 1e-5, prec)
    u = G[f"step_{name}_{eq}_{prec}_u0"].copy()
    its = []
    for _ in range(2):
        its += s.step(u)["iterations"]
    assert same_bits(u, G[f"step_{name}_{eq}_{prec}_u2"])
    assert its == G[f"step_{name}_{eq}_{prec}_its"].tolist()


def test_golden_config1(orc):
    """Config 1 end to end: heat 32^3 midpoint1 fp32 tol 1e-4, 10 steps."""
    s = orc.stepper(0, 32, tab("midpoint1"), 0.01, 1e-4, "f32")
    u = np.zeros(32 ** 3)
    its = []
    for _ in range(10):
        its += s.step(u)["iterations"]
    assert same_bits(u, G["cfg1_state"])
    assert its == G["cfg1_its"].tolist()
    u0, g, h, gam = orc.make_problem(0, 32)
    exact = orc.heat_exact(32, 0.1, g)
    err = np.abs(u - exact).max()
    assert err == G["cfg1_meta"][0]


# ---- 2. against the reference library itself -------------------------------------
@pytest.mark.parametrize("n", [2, 3, 8])
@pytest.mark.parametrize("kind", [0, 1, 2, 3])
def test_restatement_vs_reference_kernels(ref, orc, n, kind):
    rng = np.random.default_rng(77 + n + kind)

    def rnd(m):
        x = rng.uniform(-1, 1, m)
        if kind >= 2:
            x = x + 1j * rng.uniform(-1, 1, m)
        return x.astype(DT[kind])

    for st in (0, 1):
        if st == 1 and n < 3:
            continue
        x = rnd(n ** 3)
        assert same_bits(orc.stencil(kind, n, st, 1.0, -0.3, x), ref.stencil(kind, n, st, 1.0, -0.3, x))
    for side in range(3):
        q, x = rnd(n * n), rnd(n ** 3)
        assert same_bits(orc.tensor(kind, side, n, q, x), ref.tensor(kind, side, n, q, x))
    if kind >= 2 and n < 3:
        return
    x = rnd(n ** 3)
    assert same_bits(orc.fastdiag(kind, n, 0.01, 0.5, x), ref.fastdiag(kind, n, 0.01, 0.5, x))


@pytest.mark.parametrize("kind,solver", [(0, 0), (1, 0), (1, 1), (2, 1), (3, 1)])
@pytest.mark.parametrize("pre", [0, 1])
def test_restatement_vs_reference_solves(ref, orc, kind, solver, pre):
    n = 8
    rng = np.random.default_rng(5 + kind)
    b = rng.uniform(-1, 1, n ** 3).astype(DT[kind])
    for tol in (1e-3, 1e-8):
        xa, ra = ref.stage_solve(kind, solver, n, 0.01, 0.5, pre, b, b, tol, 40)
        xb, rb = orc.stage_solve(kind, solver, n, 0.01, 0.5, pre, b, b, tol, 40)
        assert same_bits(xa, xb)
        assert ra["iterations"] == rb["iterations"]
        assert np.array_equal(ra["history"], rb["history"])
        assert ra["true_residual"] == rb["true_residual"]


@pytest.mark.parametrize("name", ["midpoint1", "4s3pA", "4s3pB", "4s3pC"])
@pytest.mark.parametrize("eq", [0, 1])
@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_restatement_vs_reference_steps(ref, orc, name, eq, prec):
    t = ref.tableau(name)
    n = 8
    tau = 0.01 if eq == 0 else 1.0 / 640.0
    sa = ref.stepper(eq, n, t, tau, 1e-5, prec)
    sb = orc.stepper(eq, n, t, tau, 1e-5, prec)
    u0, *_ = ref.make_problem(eq, n)
    ua, ub = u0.copy(), u0.copy()
    for _ in range(3):
        ta = sa.step(ua)
        tb = sb.step(ub)
        assert ta["iterations"] == tb["iterations"]
    assert same_bits(ua, ub)


def test_golden_matches_reference(ref):
    """The fixtures are the reference's (regenerate with make_golden.py)."""
    for name in ("4s3pA", "4s3pB", "4s3pC", "midpoint1"):
        t = ref.tableau(name)
        assert same_bits(t["a_high"], G[f"tab_{name}_ah"]) and same_bits(t["b"], G[f"tab_{name}_b"])
    x = G["k1_x"]
    assert same_bits(ref.fastdiag(1, 5, 0.01, 0.5, x), G["k1_fastdiag"])
