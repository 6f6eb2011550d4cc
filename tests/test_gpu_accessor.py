"""Accessor-style Krylov vector storage (accessor.cu; north_star (a): the
matrix-free stencil and the CG vectors read fp16 / fp32 storage and compute in
the stage's precision).  No reference counterpart: the oracle is
oracle/krylov_np.cg_storage — the reference's cg<T> (krylov.hpp:100-168,
pinned against the reference's own cg by tests/test_oracle_np.py) with r, z,
p, q stored through the same rounding — run with the same numpy stencil and
the same sequential block-Jacobi sums as the kernels, so the two differ only
in the order of the fp64 dot sums."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _system(n, T, seed=5):
    tau, a = 0.01, 0.5
    h = 1.0 / (n - 1)
    sigma, gamma = 1.0, -tau * a * (-1.0 / h ** 2)
    b = np.random.default_rng(seed).uniform(-1, 1, n ** 3).astype(T)
    return tau, a, sigma, gamma, b


def _store(name, T):
    from oracle.krylov_np import round16

    if name == "f16":
        return round16
    return lambda v: v.astype(np.float32).astype(T)


@pytest.mark.parametrize("dtype,storage", [("f32", "f16"), ("f64", "f16"), ("f64", "f32")])
@pytest.mark.parametrize("precond", ["block-jacobi", None])
def test_cg_vector_storage_matches_restatement(gpu, mp, dtype, storage, precond):
    import torch
    from oracle.krylov_np import BlockJacobiSeq, cg_storage, heat_apply

    n = 64
    T = np.float32 if dtype == "f32" else np.float64
    code = 0 if dtype == "f32" else 1
    tau, a, sigma, gamma, b = _system(n, T)
    tol = 1e-3 if storage == "f16" else 1e-6
    cap = 300
    op = lambda v: heat_apply(v, n, T(sigma), T(gamma))  # noqa: E731
    pre_np = BlockJacobiSeq(n, 8, sigma, gamma, "f32", T) if precond else None
    xo, ro = cg_storage(op, pre_np, b, np.zeros_like(b), tol, cap, store=_store(storage, T))
    A = mp.Operator.stencil(code, n, 0, sigma, gamma)
    P = mp.Operator.block_jacobi(code, "heat", n, tau, a, 8, "f32") if precond else None
    bd = torch.from_numpy(b).cuda()
    xg, rg = mp.cg(A, P, bd, torch.zeros_like(bd), tol, cap, storage=storage)
    assert ro["converged"] and rg["converged"], (ro["iterations"], rg["iterations"])
    assert ro["iterations"] >= 3
    assert abs(rg["iterations"] - ro["iterations"]) <= 1, (rg["iterations"], ro["iterations"])
    h = min(len(rg["history"]), len(ro["history"]))
    np.testing.assert_allclose(rg["history"][:h], ro["history"][:h], rtol=1e-2, atol=1e-4 * ro["history"][0])
    xg = xg.cpu().numpy()
    assert np.linalg.norm(xg - xo) <= 10 * tol * np.linalg.norm(xo)
    # the stored-precision solve reaches the working-precision answer to its tolerance
    xw, rw = mp.cg(A, P, bd, torch.zeros_like(bd), tol, cap)
    assert rw["converged"]
    assert np.linalg.norm(xg - xw.cpu().numpy()) <= 20 * tol * np.linalg.norm(xg)


def test_cg_vector_storage_launches_storage_kernels(gpu, mp):
    """The storage path runs its own kernels (no working-precision fallback)
    and reads 2-byte vectors: the identity-preconditioned fp16 solve performs
    one update and one fused direction + stencil + dot pass per iteration
    (k_acc_pq) plus the initial residual, the first stencil, the exit
    residual and the true-residual checks."""
    import torch

    n = 32
    tau, a, sigma, gamma, b = _system(n, np.float32, seed=9)
    A = mp.Operator.stencil(0, n, 0, sigma, gamma)
    bd = torch.from_numpy(b).cuda()
    l0 = mp.kernel_launches()
    _, r = mp.cg(A, None, bd, torch.zeros_like(bd), 1e-3, 200, storage="f16")
    launched = mp.kernel_launches() - l0
    it = r["iterations"]
    assert r["converged"] and it >= 3
    # resid x2 + first stencil (+1 true-residual check per convergence trigger), per iteration update + pq
    assert 2 * it + 2 <= launched <= 3 * it + 3, (launched, it)


def test_cg_vector_storage_errors(gpu, mp):
    import torch

    n = 16
    tau, a, sigma, gamma, b = _system(n, np.float32)
    A = mp.Operator.stencil(0, n, 0, sigma, gamma)
    P = mp.Operator.fastdiag_stage(0, "heat", n, tau, a)
    bd = torch.from_numpy(b).cuda()
    with pytest.raises(ValueError):  # FastDiag has no storage-precision apply
        mp.cg(A, P, bd, bd.clone(), 1e-3, 10, storage="f16")
    with pytest.raises(ValueError):  # fp32 storage under fp32 compute
        mp.cg(A, None, bd, bd.clone(), 1e-3, 10, storage="f32")
    with pytest.raises(ValueError):
        mp.cg(A, None, bd, bd.clone(), 1e-3, 10, numerics="parity", storage="f16")
    with pytest.raises(ValueError):
        mp.Stepper("heat", n, mp.builtin("4s3pB"), 0.01, 1e-3, "f32", krylov_storage="f16")  # FastDiag


@pytest.mark.parametrize("prec,storage", [("f32", "f16"), ("f64", "f32")])
def test_stepper_vector_storage(gpu, mp, prec, storage):
    """Stepper(..., preconditioner="block-jacobi", krylov_storage=...): the
    stage solves keep r, z, p, q in the storage precision; the stepped state
    agrees with the working-precision stepper to the stage tolerance.  fp16
    vectors put a floor near 2.6e-3 of ||r0|| under the recurrence (measured:
    the second step's solves stall at 2.4e-3 / 0.91 with tol 1e-3), so the
    fp16 case runs at tol 1e-2, above it; iteration counts within twice the
    working-precision count."""
    n = 64
    t = mp.builtin("4s3pB")
    tol = 1e-2 if storage == "f16" else 1e-6
    kw = dict(preconditioner="block-jacobi", block_size=8, block_storage="f32")
    acc = mp.Stepper("heat", n, t, 0.01, tol, prec, 400, krylov_storage=storage, **kw)
    ref = mp.Stepper("heat", n, t, 0.01, tol, prec, 400, **kw)
    tight = mp.Stepper("heat", n, t, 0.01, 1e-6 if prec == "f32" else 1e-10, prec, 400, **kw)
    u0 = mp.heat_exact(n, 0.05)
    a, c, e = u0.copy(), u0.copy(), u0.copy()
    for _ in range(2):
        ta, tc = acc.step(a), ref.step(c)
        tight.step(e)
        assert all(ta["converged"]) and all(tc["converged"])
        for i, j in zip(ta["iterations"], tc["iterations"]):
            assert i <= 2 * j + 5 and j <= 2 * i + 5, (ta["iterations"], tc["iterations"])
    # the state error (against tightly solved stages) is that of the
    # working-precision vectors at the same stage tolerance, within 3x
    assert np.linalg.norm(a - e) <= 3 * np.linalg.norm(c - e) + 1e-6 * np.linalg.norm(e)


@pytest.mark.parametrize("dtype,storage,b", [("f32", "f16", 8), ("f32", "f16", 32), ("f64", "f32", 16),
                                             ("f64", "f16", 4)])
def test_cg_vector_storage_fused_passes(gpu, mp, monkeypatch, dtype, storage, b):
    """The fused accessor passes — the update with the block-Jacobi apply
    (k_acc_update_bj) and p = z + beta p with q = A p, p.q (k_acc_pq) — agree
    with the separate kernels (MPRKB_ACC_FUSED=0): the direction pass is
    bitwise, the fused update only reorders the fp64 partial sums of
    ||r||^2 and r.z (last-bit changes of the working-precision scalars), so
    iterations agree within one and histories / solutions to 1e-5."""
    import torch

    n = 64
    T = np.float32 if dtype == "f32" else np.float64
    code = 0 if dtype == "f32" else 1
    tau, a, sigma, gamma, bv = _system(n, T, seed=11)
    A = mp.Operator.stencil(code, n, 0, sigma, gamma)
    P = mp.Operator.block_jacobi(code, "heat", n, tau, a, b, "f16")
    bd = torch.from_numpy(bv).cuda()
    tol = 1e-3 if storage == "f16" else 1e-7
    xf, rf = mp.cg(A, P, bd, torch.zeros_like(bd), tol, 300, storage=storage)
    monkeypatch.setenv("MPRKB_ACC_FUSED", "0")
    xs, rs = mp.cg(A, P, bd, torch.zeros_like(bd), tol, 300, storage=storage)
    assert rf["converged"] and rs["converged"]
    assert abs(rf["iterations"] - rs["iterations"]) <= 1 and rf["iterations"] >= 3
    h = min(len(rf["history"]), len(rs["history"]))
    np.testing.assert_allclose(rf["history"][:h], rs["history"][:h], rtol=1e-5)
    xf, xs = xf.cpu().numpy(), xs.cpu().numpy()
    assert np.linalg.norm(xf - xs) <= 1e-5 * np.linalg.norm(xs) + 2 * tol * np.linalg.norm(xs)


def test_cg_vector_storage_tma_direction_pass(gpu, mp, monkeypatch):
    """fp16 vectors on a TMA-sized grid (n % 128 == 0): the direction pass
    p = z + beta p, q = A p, p.q runs on the TMA plane pipeline
    (k_acc_pq_tma) with the same element operations as k_acc_pq
    (MPRKB_ACC_PQ_TMA=0); only the fp64 grouping of p.q differs, so the
    iterations agree within one and histories / solutions closely."""
    import torch

    n = 128
    tau, a, sigma, gamma, bv = _system(n, np.float32, seed=5)
    A = mp.Operator.stencil(0, n, 0, sigma, gamma)
    P = mp.Operator.block_jacobi(0, "heat", n, tau, a, 8, "f16")
    bd = torch.from_numpy(bv).cuda()
    xf, rf = mp.cg(A, P, bd, torch.zeros_like(bd), 1e-3, 300, storage="f16")
    monkeypatch.setenv("MPRKB_ACC_PQ_TMA", "0")
    xs, rs = mp.cg(A, P, bd, torch.zeros_like(bd), 1e-3, 300, storage="f16")
    assert rf["converged"] and rs["converged"]
    assert abs(rf["iterations"] - rs["iterations"]) <= 1 and rf["iterations"] >= 3
    h = min(len(rf["history"]), len(rs["history"]))
    np.testing.assert_allclose(rf["history"][:h], rs["history"][:h], rtol=1e-5)
    xf, xs = xf.cpu().numpy(), xs.cpu().numpy()
    assert np.linalg.norm(xf - xs) <= 1e-5 * np.linalg.norm(xs) + 2e-3 * np.linalg.norm(xs)
