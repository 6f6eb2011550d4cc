"""TEST INFRASTRUCTURE ONLY — numpy restatements for the north_star extensions
that have no reference counterpart; only tests/ import this.

* ``gmres_basis16`` — the reference's left-preconditioned MGS-GMRES
  (/root/reference/proj/include/mprk/krylov.hpp:181-311, line by line: initial
  residual 190-194, stopping test + happy breakdown 199-200 / 277-280, basis
  normalisation 228-231 / 297-300, MGS 236-242, Givens 245-270, candidate veto
  281-296, exit true residual 306-309) with ONE change, the extension under
  test: every Krylov basis vector is STORED in binary16 (real and imaginary
  parts rounded to nearest-even) and widened exactly when read, while the
  Gram-Schmidt coefficients and norms accumulate in fp64 (north_star (a):
  "fp16 Krylov-basis/vector storage and fp64 accumulation").  Vector updates
  run in the working precision T; scalars (Hessenberg, rotations, the
  least-squares solve) in T's scalar type, as the reference's.
* ``AdvDiff`` — the periodic advection-diffusion stage operator
  A = sigma I + gamma D_c + gamma2 L (D_c: central first differences summed
  over the three axes, L: 6x minus the six neighbours) restated from the
  reference's periodic KronSumOperator (operators.hpp:113-161, the advection
  branch) plus the diffusion term, and its exact inverse by FFT (the
  combined-eigenvalue FastDiag preconditioner: the reference's
  spectral_periodic eigenvalues, spectral.cpp:31-51, plus the Laplacian's
  2 - 2cos(2 pi k / n)).
* ``block_jacobi`` — x-line block-Jacobi with the inverse blocks rounded to
  the storage precision (the library's extension).
* ``cg_storage`` — the reference's cg<T> (krylov.hpp:100-168, line by line)
  with ONE change, the accessor-style extension under test: its work vectors
  r, z, p, q are STORED through ``store`` (binary16 / binary32, RNE) and
  widened exactly when read; x and b stay in T, vector arithmetic runs in T,
  dots are fp64 sums of the stored values.  ``heat_apply`` is the reference's
  Dirichlet KronSumOperator point arithmetic (operators.hpp:133-140) in T, and
  ``BlockJacobiSeq`` the block apply with the GPU kernel's sequential sum
  order (ext.cu / accessor.cu).
"""
from __future__ import annotations

import numpy as np

RT = {np.dtype(np.float32): np.float32, np.dtype(np.float64): np.float64,
      np.dtype(np.complex64): np.float32, np.dtype(np.complex128): np.float64}


def round16(v: np.ndarray) -> np.ndarray:
    """binary16 storage of v (each real component RNE), widened back to v's dtype."""
    if np.iscomplexobj(v):
        return (v.real.astype(np.float16).astype(v.real.dtype)
                + 1j * v.imag.astype(np.float16).astype(v.real.dtype)).astype(v.dtype)
    return v.astype(np.float16).astype(v.dtype)


def _dot64(a, b):
    """conj(a) . b accumulated in fp64 (complex128 / float64)."""
    a64 = a.astype(np.complex128 if np.iscomplexobj(a) else np.float64)
    b64 = b.astype(a64.dtype)
    return np.vdot(a64, b64)


def gmres_basis16(op, precond, b, x0, tol, max_iter, store=round16):
    """krylov.hpp:181-311 with the basis stored through ``store`` (default
    binary16) and fp64-accumulated dots; returns (x, report dict)."""
    T = b.dtype.type
    R = RT[b.dtype]
    m = b.size
    x = np.array(x0, dtype=b.dtype, copy=True)
    hist = []

    def norm2(v):
        return R(np.sqrt(R(np.real(_dot64(v, v)))))

    def satisfied(res, ref):  # StoppingCriterion::satisfied (krylov.hpp:21-23)
        return res <= tol or (ref > 0.0 and res / ref <= tol)

    def pre(v):
        return precond(v).astype(b.dtype) if precond is not None else v.copy()

    t = (b - op(x).astype(b.dtype)).astype(b.dtype)
    w = pre(t)
    beta = float(norm2(w))
    hist.append(beta)
    rep = dict(iterations=0, converged=False, failure=0)
    k = 0
    if satisfied(beta, beta) or beta == 0.0:
        rep["converged"] = True
    else:
        basis, h_cols = [], []
        cs = [R(0)] * max_iter
        sn = [T(0)] * max_iter
        s = [T(0)] * (max_iter + 1)
        s[0] = T(beta)
        x_built = False

        def candidate(cols):
            y = [T(0)] * cols
            for i in range(cols - 1, -1, -1):
                acc = s[i]
                for j in range(i + 1, cols):
                    acc = T(acc - h_cols[j][i] * y[j])
                y[i] = T(acc / h_cols[i][i])
            xc = x.copy()
            for j in range(cols):
                xc = (xc + T(y[j]) * basis[j]).astype(b.dtype)
            return xc

        basis.append(store((w * T(T(1.0) / T(beta))).astype(b.dtype)))
        while k < max_iter:
            t = op(basis[k]).astype(b.dtype)
            w = pre(t)
            h = [T(0)] * (k + 2)
            for j in range(k + 1):
                hj = T(_dot64(basis[j], w))
                h[j] = hj
                w = (w - hj * basis[j]).astype(b.dtype)
            wnorm = norm2(w)
            h[k + 1] = T(float(wnorm))
            happy = not (float(wnorm) > 0.0)
            for j in range(k):
                tmp = T(T(cs[j]) * h[j] + sn[j] * h[j + 1])
                h[j + 1] = T(T(cs[j]) * h[j + 1] - np.conj(sn[j]) * h[j])
                h[j] = tmp
            anorm = R(abs(h[k]))
            bnorm = R(abs(h[k + 1]))
            rho = R(np.sqrt(R(anorm * anorm + bnorm * bnorm)))
            if rho == 0:
                cs[k], sn[k] = R(1), T(0)
            elif anorm == 0:
                cs[k], sn[k] = R(0), T(1.0)
            else:
                cs[k] = R(anorm / rho)
                sn[k] = T(T(h[k] / T(float(anorm))) * T(float(R(bnorm / rho))))
            h[k] = T(T(cs[k]) * h[k] + sn[k] * h[k + 1])
            h[k + 1] = T(0)
            s[k + 1] = T(-np.conj(sn[k]) * s[k])
            s[k] = T(T(cs[k]) * s[k])
            h_cols.append(h)
            rep["iterations"] += 1
            k += 1
            est = float(abs(s[k]))
            hist.append(est)
            if happy:
                rep["converged"] = True
                break
            if satisfied(est, beta):
                xc = candidate(k)
                tt = (b - op(xc).astype(b.dtype)).astype(b.dtype)
                rt = float(norm2(pre(tt)))
                if satisfied(rt, beta):
                    x = xc
                    x_built = True
                    rep["converged"] = True
                    break
                hist[-1] = rt
            if k == max_iter:
                break
            basis.append(store((w * T(T(1.0) / T(float(wnorm)))).astype(b.dtype)))
        if not rep["converged"]:
            rep["failure"] = 1
        if not x_built:
            x = candidate(k)
    t = (b - op(x).astype(b.dtype)).astype(b.dtype)
    rep["true_residual"] = float(norm2(t))
    rep["history"] = np.array(hist)
    return x, rep


class AdvDiff:
    """Periodic advection-diffusion stage operator on an n^3 grid (x-fastest,
    idx = i + j n + k n^2) and its exact FFT inverse."""

    def __init__(self, n, sigma, gamma, gamma2, dtype=np.complex64):
        self.n, self.sigma, self.gamma, self.gamma2, self.dtype = n, sigma, gamma, gamma2, dtype
        th = 2 * np.pi * np.arange(n) / n
        adv = 2j * np.sin(th)      # x_{+1} - x_{-1} on mode e^{i th j}
        lap = 2 - 2 * np.cos(th)   # 2x - x_{+1} - x_{-1}
        L = (sigma + gamma * (adv[:, None, None] + adv[None, :, None] + adv[None, None, :])
             + gamma2 * (lap[:, None, None] + lap[None, :, None] + lap[None, None, :]))
        self.lam = L

    @staticmethod
    def stage(n, tau, a, nu):
        """sigma, gamma, gamma2 of I - tau a (K_a + K_d): h = 1/n,
        gamma_K = -1/(2h) (operators.cpp:48-54), K_d = nu/h^2 Laplacian."""
        h = 1.0 / n
        return 1.0, -tau * a * (-1.0 / (2 * h)), -tau * a * (-nu / h ** 2)

    def apply(self, x):
        n = self.n
        X = x.reshape(n, n, n)
        rd = self.dtype
        out = X * rd(self.sigma)
        diff = np.zeros_like(X)
        lap = X * rd(6.0)
        for ax in (2, 1, 0):  # i, j, k
            p = np.roll(X, -1, axis=ax)
            q = np.roll(X, 1, axis=ax)
            diff = diff + (p - q)
            lap = lap - p - q
        out = out + rd(self.gamma) * diff + rd(self.gamma2) * lap
        return out.astype(self.dtype).ravel()

    def solve(self, r):
        """exact inverse (fp64 FFT), rounded to the working precision."""
        n = self.n
        R = np.fft.fftn(r.astype(np.complex128).reshape(n, n, n))
        return np.fft.ifftn(R / self.lam).astype(self.dtype).ravel()


def line_block(bs, sigma, gamma, gamma2=None):
    """x-line block of the stage operator: Dirichlet heat (gamma2 None) or the
    periodic advection(-diffusion) stencil's in-line couplings."""
    A = np.zeros((bs, bs))
    if gamma2 is None:
        d, lo, hi = sigma + 6 * gamma, -gamma, -gamma
    else:
        d, lo, hi = sigma + 6 * gamma2, -gamma - gamma2, gamma - gamma2
    for i in range(bs):
        A[i, i] = d
        if i > 0:
            A[i, i - 1] = lo
        if i + 1 < bs:
            A[i, i + 1] = hi
    return A


class BlockJacobi:
    """z_B = D_B^-1 r_B on x-line blocks of length b; the inverse blocks are
    rounded to the storage precision and applied in the compute precision."""

    def __init__(self, n, b, sigma, gamma, storage, dtype, gamma2=None):
        self.n, self.b = n, min(b, n)
        st = {"f16": np.float16, "f32": np.float32, "f64": np.float64}[storage]
        self.inv = {}
        for bs in {self.b, n % self.b} - {0}:
            self.inv[bs] = np.linalg.inv(line_block(bs, sigma, gamma, gamma2)).astype(st).astype(np.float64)
        self.dtype = np.dtype(dtype)
        self.R = RT[self.dtype]

    def __call__(self, r):
        n, b = self.n, self.b
        X = r.reshape(-1, n)
        Z = np.zeros_like(X)
        for i0 in range(0, n, b):
            bs = min(b, n - i0)
            Dinv = self.inv[bs].astype(self.R)
            Z[:, i0:i0 + bs] = (X[:, i0:i0 + bs] @ Dinv.T.astype(self.dtype)).astype(self.dtype)
        return Z.ravel()


def heat_apply(x, n, sigma, gamma):
    """sigma x + gamma (6 x - six Dirichlet neighbours) in x's dtype, the
    reference's order of roundings (operators.hpp:133-140; numpy never fuses)."""
    T = x.dtype.type
    X = x.reshape(n, n, n)  # [k][j][i]
    P = np.zeros((n + 2, n + 2, n + 2), dtype=x.dtype)
    P[1:-1, 1:-1, 1:-1] = X
    c = P[1:-1, 1:-1, 1:-1]
    acc = T(6.0) * c
    acc = acc - P[1:-1, 1:-1, :-2]
    acc = acc - P[1:-1, 1:-1, 2:]
    acc = acc - P[1:-1, :-2, 1:-1]
    acc = acc - P[1:-1, 2:, 1:-1]
    acc = acc - P[:-2, 1:-1, 1:-1]
    acc = acc - P[2:, 1:-1, 1:-1]
    return (T(sigma) * c + T(gamma) * acc).ravel()


class BlockJacobiSeq(BlockJacobi):
    """BlockJacobi with each output summed over the block's inputs in
    ascending order in the compute precision (the kernels' order)."""

    def __call__(self, r):
        n, b = self.n, self.b
        T = self.dtype.type
        X = r.reshape(-1, n)
        Z = np.zeros_like(X)
        for i0 in range(0, n, b):
            bs = min(b, n - i0)
            D = self.inv[bs].astype(self.R)  # D[ii][jj] = inverse (row ii, column jj)
            for ii in range(bs):
                acc = np.zeros(X.shape[0], dtype=self.dtype)
                for jj in range(bs):
                    acc = acc + T(D[ii, jj]) * X[:, i0 + jj]
                Z[:, i0 + ii] = acc
        return Z.ravel()


def cg_storage(op, precond, b, x0, tol, max_iter, store):
    """krylov.hpp:100-168 with r, z, p, q stored through ``store`` (a function
    rounding a T vector to the storage precision and widening it back);
    precond None = identity.  Returns (x, report dict)."""
    T = b.dtype.type
    x = np.array(x0, dtype=b.dtype, copy=True)
    hist = []

    def dot(a, c):
        return float(np.dot(a.astype(np.float64), c.astype(np.float64)))

    def norm(sq):
        return float(T(np.sqrt(T(sq))))

    def satisfied(res, ref):  # StoppingCriterion::satisfied (krylov.hpp:21-23)
        return res <= tol or (ref > 0 and res / ref <= tol)

    def pre(r):
        return r if precond is None else store(precond(r))

    rep = dict(iterations=0, converged=False, failure=0)
    r = store(b - op(x))
    r_sq = dot(r, r)
    r0 = norm(r_sq)
    hist.append(r0)
    rnorm = r0
    if satisfied(rnorm, r0):
        rep["converged"] = True
    else:
        z = pre(r)
        p = z.copy()
        rz = T(dot(r, z))
        for _ in range(max_iter):
            if not rz > 0:
                rep["failure"] = 2
                break
            q = store(op(p))
            pq = T(dot(p, q))
            if not pq > 0:
                rep["failure"] = 2
                break
            alpha = T(rz / pq)
            x = x + alpha * p
            r = store(r - alpha * q)
            rep["iterations"] += 1
            rnorm = norm(dot(r, r))
            hist.append(rnorm)
            if satisfied(rnorm, r0):
                q = store(b - op(x))
                rtnorm = norm(dot(q, q))
                if satisfied(rtnorm, r0):
                    rep["converged"] = True
                    break
                r = q
                hist[-1] = rtnorm
                z = pre(r)
                p = z.copy()
                rz = T(dot(r, z))
                continue
            z = pre(r)
            rz_next = T(dot(r, z))
            beta = T(rz_next / rz)
            rz = rz_next
            p = store(z + beta * p)
        if not rep["converged"] and rep["failure"] == 0:
            rep["failure"] = 1
    q = b - op(x)
    rep["true_residual"] = norm(dot(store(q), store(q)))
    rep["history"] = np.array(hist)
    return x, rep
