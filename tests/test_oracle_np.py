"""Pin oracle/krylov_np.py (the numpy restatements used as oracles for the
north_star extensions) against the UNMODIFIED reference (oracle/_ref) on CPU.
"""
import numpy as np
import pytest

from oracle.krylov_np import AdvDiff, BlockJacobi, gmres_basis16, round16


def _rhs(n, seed=3):
    rng = np.random.default_rng(seed)
    return (rng.uniform(-1, 1, n ** 3) + 1j * rng.uniform(-1, 1, n ** 3)).astype(np.complex64)


@pytest.mark.parametrize("n", [6, 12])
def test_advdiff_operator_is_reference_periodic_stencil(ref, n):
    """nu = 0: AdvDiff.apply is the reference's PeriodicCentralDiff1D
    KronSumOperator (operators.hpp:141-158) up to fp32 summation order."""
    s, g, g2 = AdvDiff.stage(n, 1.0 / 640.0, 0.5, 0.0)
    x = _rhs(n)
    want = ref.stencil(2, n, 1, s, g, x)
    got = AdvDiff(n, s, g, g2).apply(x)
    assert np.abs(got - want).max() <= 4e-7 * (1 + 6 * abs(g)) * np.abs(x).max()


@pytest.mark.parametrize("n", [6, 12])
def test_advdiff_inverse_is_reference_fastdiag(ref, n):
    """nu = 0: the FFT inverse equals the reference's advection FastDiag
    (build_advection_precond, precond.cpp:27-42) — same eigenvalues, same
    convention — to fp64 rounding."""
    tau, a = 1.0 / 640.0, 0.5
    s, g, g2 = AdvDiff.stage(n, tau, a, 0.0)
    x = _rhs(n).astype(np.complex128)
    want = ref.fastdiag(3, n, tau, a, x)
    got = AdvDiff(n, s, g, g2, np.complex128).solve(x)
    assert np.abs(got - want).max() <= 1e-12 * np.abs(want).max()


@pytest.mark.parametrize("nu", [0.0, 0.01])
def test_advdiff_inverse_inverts(nu):
    n = 10
    s, g, g2 = AdvDiff.stage(n, 1.0 / 64.0, 0.5, nu)
    ad = AdvDiff(n, s, g, g2, np.complex128)
    x = _rhs(n).astype(np.complex128)
    assert np.abs(ad.apply(ad.solve(x)) - x).max() <= 1e-12


def test_round16():
    v = np.array([1.0 + 2j, 1e-3 - 3e4j, 0.1 + 0.2j], np.complex64)
    r = round16(v)
    assert r.dtype == np.complex64
    assert np.array_equal(r.real, v.real.astype(np.float16).astype(np.float32))
    assert np.array_equal(r.imag, v.imag.astype(np.float16).astype(np.float32))


@pytest.mark.parametrize("n", [8, 16])
def test_gmres_restatement_matches_reference_gmres(ref, n):
    """With the storage hook set to the identity, the restatement of
    krylov.hpp:181-311 follows the reference's own gmres<complex<float>>
    (its dots accumulate in fp64 instead of fp32, so not bitwise): same
    iteration count, same residual history to a few ulps of the stopping
    test, same solution to the tolerance."""
    tau, a, nu = 1.0 / 160.0, 0.5, 0.01
    s, g, g2 = AdvDiff.stage(n, tau, a, nu)
    ad = AdvDiff(n, s, g, g2)
    bj = BlockJacobi(n, 4, s, g, "f32", np.complex64, gamma2=g2)
    b = _rhs(n, 7)
    tol = 1e-5
    xw, rw = ref.krylov_cb(2, 1, ad.apply, bj, b, np.zeros_like(b), tol, 60)
    xo, ro = gmres_basis16(ad.apply, bj, b, np.zeros_like(b), tol, 60, store=lambda v: v)
    assert rw["converged"] and ro["converged"] and rw["iterations"] > 3
    assert ro["iterations"] == rw["iterations"]
    # (entries near the fp32 floor, ~1e-6 of beta, differ by the dots' rounding)
    np.testing.assert_allclose(ro["history"], rw["history"], rtol=1e-3, atol=2e-6 * rw["history"][0])
    assert np.linalg.norm(xo - xw) <= 1e-4 * np.linalg.norm(xw)
    # fp16 storage: a few more iterations at most, same solution to tol
    x16, r16 = gmres_basis16(ad.apply, bj, b, np.zeros_like(b), 1e-3, 60)
    assert r16["converged"] and r16["iterations"] <= rw["iterations"] + 2
    assert np.linalg.norm(x16 - xw) <= 1e-2 * np.linalg.norm(xw)


def test_block_jacobi_np_matches_reference_cg(ref):
    """The numpy block-Jacobi ApplyFn inside the reference's cg<double>
    converges; its storage rounding is exactly float16 of the fp64 inverse."""
    n, tau, a = 12, 0.01, 0.5
    h = 1.0 / (n - 1)
    s, g = 1.0, -tau * a * (-1.0 / h ** 2)
    bj = BlockJacobi(n, 4, s, g, "f16", np.float64)
    inv = bj.inv[4]
    assert np.array_equal(inv, inv.astype(np.float16).astype(np.float64))
    b = np.random.default_rng(1).uniform(-1, 1, n ** 3)
    x, r = ref.stage_solve_cb(1, 0, n, tau, a, bj, b, b, 1e-8, 200)
    assert r["converged"] and r["iterations"] > 1


def test_cg_storage_restatement_matches_reference_cg(ref):
    """oracle/krylov_np.cg_storage without storage rounding IS the reference's
    cg<double> (krylov.hpp:100-168): same iterations and iterate, with the
    numpy heat stencil and the sequential block-Jacobi in the ApplyFn slots."""
    from oracle.krylov_np import BlockJacobiSeq, cg_storage, heat_apply

    n, tau, a = 16, 0.01, 0.5
    h = 1.0 / (n - 1)
    s, g = 1.0, -tau * a * (-1.0 / h ** 2)
    op = lambda v: heat_apply(v, n, s, g)  # noqa: E731
    bj = BlockJacobiSeq(n, 4, s, g, "f32", np.float64)
    b = np.random.default_rng(3).uniform(-1, 1, n ** 3)
    for pre in (bj, None):
        xw, rw = ref.krylov_cb(1, 0, op, pre, b, np.zeros_like(b), 1e-9, 300)
        xo, ro = cg_storage(op, pre, b, np.zeros_like(b), 1e-9, 300, store=lambda v: v)
        assert rw["converged"] and ro["converged"]
        assert abs(ro["iterations"] - rw["iterations"]) <= 1, (ro["iterations"], rw["iterations"])
        assert np.linalg.norm(xo - xw) <= 1e-8 * np.linalg.norm(xw)
        assert abs(ro["true_residual"] - rw["true_residual"]) <= 1e-6 * np.linalg.norm(b)


def test_cg_storage_fp16_converges_to_its_floor():
    """fp16 vector storage under fp32 compute: CG still reaches tol 1e-3 at
    n = 16 (the fp16 rounding floor of the recurrence is ~1e-3 relative)."""
    from oracle.krylov_np import BlockJacobiSeq, cg_storage, heat_apply, round16

    n, tau, a = 16, 0.01, 0.5
    h = 1.0 / (n - 1)
    s, g = np.float32(1.0), np.float32(-tau * a * (-1.0 / h ** 2))
    op = lambda v: heat_apply(v, n, s, g)  # noqa: E731
    bj = BlockJacobiSeq(n, 8, s, g, "f16", np.float32)
    b = np.random.default_rng(4).uniform(-1, 1, n ** 3).astype(np.float32)
    x, r = cg_storage(op, bj, b, np.zeros_like(b), 1e-3, 200, store=round16)
    assert r["converged"] and r["iterations"] > 3
    assert r["true_residual"] <= 2e-3 * np.linalg.norm(b)
