"""North-star extensions without a reference counterpart:
block-Jacobi with per-block storage precision, CSR SpMV with fp16/fp32/fp64
values, fp16 Krylov-basis GMRES, the advection-diffusion operator.

Oracle route: a CPU ApplyFn (numpy) plugged into the
reference's OWN cg/gmres through oracle/ref_shim.cpp's callback entry point;
the storage roundings are emulated exactly with numpy's float16/float32.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

DT = {0: np.float32, 1: np.float64, 2: np.complex64, 3: np.complex128}
ST = {"f16": np.float16, "f32": np.float32, "f64": np.float64}


def line_block(n, bs, sigma, gamma, stencil=0, gamma2=0.0):
    A = np.zeros((bs, bs))
    for i in range(bs):
        if stencil == 0:
            d, lo, hi = sigma + 6 * gamma, -gamma, -gamma
        else:
            d, lo, hi = sigma + 6 * gamma2, -gamma - gamma2, gamma - gamma2
        A[i, i] = d
        if i > 0:
            A[i, i - 1] = lo
        if i + 1 < bs:
            A[i, i + 1] = hi
    return A


class NumpyBlockJacobi:
    """z_B = D_B^-1 r_B on x-line blocks, inverse rounded to the storage
    precision, applied in the compute precision (sequential j)."""

    def __init__(self, n, b, sigma, gamma, storage, kind, stencil=0):
        self.n, self.b = n, min(b, n)
        self.inv = {}
        for bs in {self.b, n % self.b} - {0}:
            inv = np.linalg.inv(line_block(n, bs, sigma, gamma, stencil))
            self.inv[bs] = inv.astype(ST[storage]).astype(np.float64)
        self.R = np.float32 if kind in (0, 2) else np.float64
        self.dt = DT[kind]

    def __call__(self, r):
        n, b = self.n, self.b
        X = r.reshape(-1, n)
        Z = np.zeros_like(X)
        for i0 in range(0, n, b):
            bs = min(b, n - i0)
            Dinv = self.inv[bs].astype(self.R)
            Z[:, i0:i0 + bs] = (X[:, i0:i0 + bs] @ Dinv.T.astype(self.dt)).astype(self.dt)
        return Z.ravel()


def stage_params(kind, n, tau, a):
    h = 1.0 / (n - 1) if kind <= 1 else 1.0 / n
    gk = -1.0 / h ** 2 if kind <= 1 else -1.0 / (2 * h)
    return 1.0, -tau * a * gk


@pytest.mark.parametrize("kind", [0, 1, 3])
@pytest.mark.parametrize("storage", ["f16", "f32", "f64"])
@pytest.mark.parametrize("b", [4, 8, 32])
def test_block_jacobi_apply(gpu, mp, kind, storage, b):
    import torch

    n = 12
    tau, a = 0.025, 0.5
    sigma, gamma = stage_params(kind, n, tau, a)
    eq = "heat" if kind <= 1 else "advection"
    P = mp.Operator.block_jacobi(kind, eq, n, tau, a, b, storage)
    rng = np.random.default_rng(b + kind)
    r = rng.uniform(-1, 1, n ** 3)
    if kind >= 2:
        r = r + 1j * rng.uniform(-1, 1, n ** 3)
    r = r.astype(DT[kind])
    got = P.apply(torch.from_numpy(r).cuda()).cpu().numpy()
    want = NumpyBlockJacobi(n, b, sigma, gamma, storage, kind, 0 if kind <= 1 else 1)(r)
    # (the library inverts in fp64 by Gauss-Jordan, numpy by LAPACK: a rare
    # 1-ulp difference survives rounding to fp16 storage)
    tol = 2e-3 if storage == "f16" else {0: 2e-6, 1: 1e-12, 3: 1e-12}[kind]
    assert np.abs(got - want).max() <= tol * max(1.0, np.abs(want).max())
    # accuracy of the stored inverse: exact block solve up to storage rounding
    bs = min(b, n)
    D = line_block(n, bs, sigma, gamma, 0 if kind <= 1 else 1)
    lead = got.reshape(-1, n)[:, :bs].astype(np.complex128 if kind >= 2 else np.float64)
    back = lead @ D.T
    eps = {"f16": 4e-3, "f32": 3e-6, "f64": 1e-12}[storage]
    if kind == 0:
        eps = max(eps, 3e-6)
    assert np.abs(back - r.reshape(-1, n)[:, :bs]).max() <= eps * max(1.0, np.abs(D).sum(1).max())


@pytest.mark.parametrize("storage", ["f16", "f32", "f64"])
@pytest.mark.parametrize("b", [8, 16, 32])
def test_block_jacobi_apply_chunked_bitwise(gpu, mp, storage, b):
    """fp32 block-Jacobi apply with n % b == 0 runs as the chunked two-phase
    kernel (k_block_jacobi_tile); it forms every output with the same
    operations in the same order as the thread-per-block kernel
    (MPRKB_BJ_TILE=0), so the results are bitwise equal, and they match the
    numpy emulation like the generic path."""
    import os

    import torch

    n, tau, a = 64, 0.025, 0.5
    sigma, gamma = stage_params(0, n, tau, a)
    P = mp.Operator.block_jacobi(0, "heat", n, tau, a, b, storage)
    r = np.random.default_rng(b).uniform(-1, 1, n ** 3).astype(np.float32)
    rt = torch.from_numpy(r).cuda()
    got = P.apply(rt).cpu().numpy()
    os.environ["MPRKB_BJ_TILE"] = "0"
    try:
        ref_k = P.apply(rt).cpu().numpy()
    finally:
        os.environ.pop("MPRKB_BJ_TILE", None)
    assert np.array_equal(got.view(np.uint32), ref_k.view(np.uint32))
    want = NumpyBlockJacobi(n, b, sigma, gamma, storage, 0, 0)(r)
    tol = 2e-3 if storage == "f16" else 2e-6
    assert np.abs(got - want).max() <= tol * max(1.0, np.abs(want).max())


@pytest.mark.parametrize("kind,storage", [(1, "f64"), (0, "f32"), (0, "f16")])
def test_cg_block_jacobi_matches_reference_cg(gpu, mp, ref, kind, storage):
    """Block-Jacobi CG on the GPU vs the reference's own cg<T> with the numpy
    block-Jacobi ApplyFn: iteration counts +-1, solutions within tol."""
    import torch

    n, tau, a, b = 16, 0.01, 0.5, 8
    sigma, gamma = stage_params(kind, n, tau, a)
    rng = np.random.default_rng(33)
    rhs = rng.uniform(-1, 1, n ** 3).astype(DT[kind])
    pre = NumpyBlockJacobi(n, b, sigma, gamma, storage, kind)
    tol = 1e-5 if kind == 1 else 1e-4
    xw, rw = ref.stage_solve_cb(kind, 0, n, tau, a, pre, rhs, rhs, tol, 400)
    A = mp.Operator.stencil(kind, n, 0, sigma, gamma)
    P = mp.Operator.block_jacobi(kind, "heat", n, tau, a, b, storage)
    for numerics in ("fast", "parity"):
        xg, rg = mp.cg(A, P, torch.from_numpy(rhs).cuda(), torch.from_numpy(rhs).cuda(), tol, 400, numerics)
        assert rw["converged"] and rg["converged"]
        assert abs(rg["iterations"] - rw["iterations"]) <= 1, (numerics, rg["iterations"], rw["iterations"])
        err = np.linalg.norm(xg.cpu().numpy() - xw) / np.linalg.norm(xw)
        assert err <= 10 * tol


def test_stepper_block_jacobi_heat(gpu, mp, ref):
    """A full 4s3pB step with block-Jacobi stage solves (max_iter raised, as
    SURVEY §0 finding 1 requires) lands on the FastDiag (reference) result
    within the solve tolerance."""
    n, tau = 24, 0.01
    t = mp.builtin("4s3pB")
    fd = mp.Stepper("heat", n, t, tau, 1e-9, "f64")
    bj = mp.Stepper("heat", n, t, tau, 1e-9, "f64", 500, preconditioner="block-jacobi", block_size=8)
    u1 = np.random.default_rng(4).uniform(0, 1, n ** 3)
    u2 = u1.copy()
    tf = fd.step(u1)
    tb = bj.step(u2)
    assert not tb["solver_failure"]
    assert all(i > 1 for i in tb["iterations"]) and all(i == 1 for i in tf["iterations"])
    assert np.linalg.norm(u2 - u1) <= 1e-7 * np.linalg.norm(u1)


@pytest.mark.parametrize("kind", [0, 1])
@pytest.mark.parametrize("storage", ["f16", "f32", "f64"])
def test_csr_stencil(gpu, mp, kind, storage):
    """CSR assembly of the stage operator == the matrix-free stencil up to
    summation order (values stored in fp16/fp32/fp64)."""
    import torch

    n = 10
    sigma, gamma = 1.0, -0.37
    x = np.random.default_rng(5).uniform(-1, 1, n ** 3).astype(DT[kind])
    xd = torch.from_numpy(x).cuda()
    want = mp.stencil_apply(xd, n, 0, sigma, gamma).cpu().numpy().astype(np.float64)
    A = mp.Operator.csr_stencil(kind, n, 0, sigma, gamma, storage)
    got = A.apply(xd).cpu().numpy().astype(np.float64)
    # fp16 storage rounds sigma + 6 gamma and -gamma
    vd = np.float64(np.float16(sigma + 6 * gamma)) if storage == "f16" else None
    tol = {"f16": 2e-3, "f32": 2e-6, "f64": 1e-14}[storage]
    if kind == 0:
        tol = max(tol, 2e-6)
    assert np.abs(got - want).max() <= tol * max(1.0, np.abs(want).max()) * 8
    del vd


@pytest.mark.parametrize("storage", ["f16", "f32", "f64"])
def test_csr_random_vs_scipy(gpu, mp, storage):
    import scipy.sparse as sp
    import torch

    rows = 3000
    M = sp.random(rows, rows, density=0.003, random_state=7, format="csr") + sp.eye(rows, format="csr")
    M = M.tocsr()
    M.sort_indices()
    vals = M.data.astype(ST[storage])
    A = mp.Operator.csr(1, rows, M.indptr, M.indices, vals, storage)
    x = np.random.default_rng(8).uniform(-1, 1, rows)
    got = A.apply(torch.from_numpy(x).cuda()).cpu().numpy()
    M2 = sp.csr_matrix((vals.astype(np.float64), M.indices, M.indptr), shape=M.shape)
    want = M2 @ x
    assert np.abs(got - want).max() <= 1e-12 * max(1.0, np.abs(want).max())


@pytest.mark.parametrize("kind", [2, 3])
def test_gmres_fp16_basis(gpu, mp, kind):
    """GMRES with an fp16 Krylov basis (fp64-accumulated MGS) on an advection
    stage system with block-Jacobi: converges to tol with at most a few more
    iterations than the working-precision basis."""
    import torch

    n, tau, a = 16, 1.0 / 160.0, 0.5
    sigma, gamma = stage_params(kind, n, tau, a)
    A = mp.Operator.stencil(kind, n, 1, sigma, gamma)
    P = mp.Operator.block_jacobi(kind, "advection", n, tau, a, 8, "f32")
    rng = np.random.default_rng(9)
    b = (rng.uniform(-1, 1, n ** 3) + 0j).astype(DT[kind])
    bd = torch.from_numpy(b).cuda()
    x1, r1 = mp.gmres(A, P, bd, torch.zeros_like(bd), 1e-3, 60)
    x2, r2 = mp.gmres(A, P, bd, torch.zeros_like(bd), 1e-3, 60, basis_storage="f16")
    assert r1["converged"] and r2["converged"]
    assert r1["iterations"] > 1
    assert r2["iterations"] <= r1["iterations"] + 3
    res = A.apply(x2) - bd
    assert torch.linalg.norm(res).item() <= 2e-2 * torch.linalg.norm(bd).item()


def dense_adv_diff(n, nu):
    """dense K = K_a + K_d of the periodic advection-diffusion operator."""
    h = 1.0 / n
    m = n ** 3
    K = np.zeros((m, m))
    ga, gd = -1.0 / (2 * h), -nu / h ** 2
    for k in range(n):
        for j in range(n):
            for i in range(n):
                r = i + n * j + n * n * k
                for d, (di, dj, dk) in enumerate(((1, 0, 0), (0, 1, 0), (0, 0, 1))):
                    p = (i + di) % n + n * ((j + dj) % n) + n * n * ((k + dk) % n)
                    q = (i - di) % n + n * ((j - dj) % n) + n * n * ((k - dk) % n)
                    K[r, p] += ga - gd
                    K[r, q] += -ga - gd
                K[r, r] += 6 * gd
    return K


def test_advection_diffusion_step_matches_dense(gpu, mp):
    """One 4s3pC step of the advection-diffusion extension vs a dense
    stage-by-stage fp64 DIRK step (test oracle in the style of
    tests/support/dense_step.hpp)."""
    n, nu, tau = 5, 0.05, 1.0 / 64.0
    t = mp.builtin("4s3pC")
    st = mp.Stepper("advection-diffusion", n, t, tau, 1e-13, "f64", nu=nu)
    u = st.initial_state()
    K = dense_adv_diff(n, nu)
    q = t.q
    Ah, Ae, bb = np.array(t.a_high), np.array(t.a_eps), np.array(t.b)
    f, want = [], u.copy()
    for s in range(q):
        rhs = u + tau * sum((Ah[s, j] + Ae[s, j]) * f[j] for j in range(s))
        a = Ae[s, s]
        y = np.linalg.solve(np.eye(n ** 3) - tau * a * K, rhs) if a != 0 else rhs
        f.append(K @ y)
    for s in range(q):
        want = want + tau * bb[s] * f[s]
    tr = st.step(u)
    assert not tr["solver_failure"]
    assert np.abs(u - want).max() <= 1e-10 * max(1.0, np.abs(want).max())


def test_advection_diffusion_conserves_sum(gpu, mp):
    n = 16
    st = mp.Stepper("advection-diffusion", n, mp.builtin("4s3pC"), 1.0 / 640.0, 1e-12, "f64", nu=0.01)
    u = st.initial_state()
    s0 = u.sum()
    for k in range(4):
        st.step(u)
        assert abs(u.sum() - s0) <= 1e-8 * (k + 1)
