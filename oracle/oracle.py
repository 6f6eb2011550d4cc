"""TEST INFRASTRUCTURE ONLY — ctypes access to the two CPU checkers.

* ``Restatement`` — oracle/liboracle.so, the plain-C restatement of the
  reference hot path (oracle/mprk_oracle.c).
* ``Reference``  — oracle/_ref/libmprk_ref.so, the UNMODIFIED reference sources
  (/root/reference/proj) compiled by oracle/Makefile with ref_shim.cpp.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm import this module.  The product (paper_2412_16638_b200/) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libmprk_ref.so")

DT = {0: np.float32, 1: np.float64, 2: np.complex64, 3: np.complex128}
KIND = {"f32": 0, "f64": 1, "c32": 2, "c64": 3}


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def ensure_built(ref: bool = True) -> None:
    """Build liboracle.so (and _ref when the reference sources are present)."""
    if not os.path.exists(ORACLE_SO):
        subprocess.run(["make", "-C", HERE, "liboracle.so"], check=True, capture_output=True)
    if ref and not os.path.exists(REF_SO) and os.path.isdir("/root/reference/proj/src"):
        subprocess.run(["make", "-C", HERE, "ref"], check=True, capture_output=True)


def have_reference() -> bool:
    return os.path.exists(REF_SO)


class OracleError(RuntimeError):
    def __init__(self, code, msg=""):
        super().__init__(f"code {code}: {msg}")
        self.code = code


class Reference:
    """The reference library itself (bit-exact ground truth)."""

    def __init__(self, path: str = REF_SO):
        self.lib = C.CDLL(path)
        L = self.lib
        L.ref_last_error.restype = C.c_char_p
        L.ref_max_threads.restype = C.c_int
        for name in ("ref_make_problem", "ref_stencil_apply", "ref_apply_tensor",
                     "ref_fastdiag_apply", "ref_stage_solve", "ref_stepper_create",
                     "ref_stepper_step", "ref_integrate", "ref_tableau", "ref_apply_f",
                     "ref_heat_exact", "ref_spectral", "ref_stepper_history"):
            getattr(L, name).restype = C.c_int

    def _chk(self, rc):
        if rc:
            raise OracleError(rc, self.lib.ref_last_error().decode())

    def set_threads(self, t: int) -> None:
        self.lib.ref_set_threads(C.c_int(t))

    def max_threads(self) -> int:
        return self.lib.ref_max_threads()

    def tableau(self, name: str):
        ah = np.zeros(64 * 64); ae = np.zeros(64 * 64); b = np.zeros(64); c = np.zeros(64)
        q = C.c_int()
        self._chk(self.lib.ref_tableau(name.encode(), C.byref(q), _p(ah), _p(ae), _p(b), _p(c)))
        q = q.value
        return dict(q=q, a_high=ah[: q * q].reshape(q, q).copy(), a_eps=ae[: q * q].reshape(q, q).copy(),
                    b=b[:q].copy(), c=c[:q].copy())

    def make_problem(self, eq: int, n: int):
        m = n ** 3
        u0 = np.zeros(m); g = np.zeros(m) if eq == 0 else None
        h = C.c_double(); gam = C.c_double()
        self._chk(self.lib.ref_make_problem(eq, n, _p(u0), _p(g), C.byref(h), C.byref(gam)))
        return u0, g, h.value, gam.value

    def heat_exact(self, n, t):
        out = np.zeros(n ** 3)
        self._chk(self.lib.ref_heat_exact(n, C.c_double(t), _p(out)))
        return out

    def stencil(self, kind: int, n: int, stencil: int, sigma: float, gamma: float, x):
        x = np.ascontiguousarray(x, dtype=DT[kind]); out = np.empty_like(x)
        self._chk(self.lib.ref_stencil_apply(kind, n, stencil, C.c_double(sigma), C.c_double(gamma), _p(x), _p(out)))
        return out

    def apply_f(self, eq, n, prec, u):
        u = np.ascontiguousarray(u, dtype=np.float64); out = np.empty_like(u)
        self._chk(self.lib.ref_apply_f(eq, n, prec, _p(u), _p(out)))
        return out

    def tensor(self, kind: int, side: int, n: int, q, x):
        q = np.ascontiguousarray(q, dtype=DT[kind]); x = np.ascontiguousarray(x, dtype=DT[kind])
        out = np.empty_like(x)
        self._chk(self.lib.ref_apply_tensor(kind, side, n, _p(q), _p(x), _p(out)))
        return out

    def fastdiag(self, kind: int, n: int, tau: float, a: float, x):
        x = np.ascontiguousarray(x, dtype=DT[kind]); out = np.empty_like(x)
        self._chk(self.lib.ref_fastdiag_apply(kind, n, C.c_double(tau), C.c_double(a), _p(x), _p(out)))
        return out

    def spectral(self, periodic: int, n: int, sigma: float, gamma: float):
        dt = np.complex128 if periodic else np.float64
        q = np.zeros(n * n, dt); qi = np.zeros(n * n, dt); lam = np.zeros(n, dt)
        self._chk(self.lib.ref_spectral(periodic, n, C.c_double(sigma), C.c_double(gamma), _p(q), _p(qi), _p(lam)))
        return q, qi, lam

    def stage_solve(self, kind, solver, n, tau, a, precond, b, x0, tol, max_iter):
        b = np.ascontiguousarray(b, dtype=DT[kind]); x0 = np.ascontiguousarray(x0, dtype=DT[kind])
        x = np.empty_like(b)
        it = C.c_int(); cv = C.c_int(); fl = C.c_int(); tr = C.c_double(); hl = C.c_int()
        hist = np.zeros(max_iter + 8)
        self._chk(self.lib.ref_stage_solve(kind, solver, n, C.c_double(tau), C.c_double(a), precond,
                                           _p(b), _p(x0), C.c_double(tol), max_iter, _p(x),
                                           C.byref(it), C.byref(cv), C.byref(fl), C.byref(tr),
                                           _p(hist), len(hist), C.byref(hl)))
        return x, dict(iterations=it.value, converged=bool(cv.value), failure=fl.value,
                       true_residual=tr.value, history=hist[: hl.value].copy())

    CB = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p, C.c_void_p)

    def stage_solve_cb(self, kind, solver, n, tau, a, precond, b, x0, tol, max_iter):
        """The reference's own cg/gmres with a Python preconditioner
        precond(x: ndarray) -> ndarray (the ApplyFn slot, krylov.hpp:38-39)."""
        b = np.ascontiguousarray(b, dtype=DT[kind]); x0 = np.ascontiguousarray(x0, dtype=DT[kind])
        m = b.size
        x = np.empty_like(b)

        def tramp(ctx, xp, op):
            xin = np.ctypeslib.as_array(C.cast(xp, C.POINTER(C.c_byte)), shape=(m * b.itemsize,)).view(b.dtype)
            out = np.ctypeslib.as_array(C.cast(op, C.POINTER(C.c_byte)), shape=(m * b.itemsize,)).view(b.dtype)
            out[:] = precond(xin.copy())

        cb = self.CB(tramp)
        it = C.c_int(); cv = C.c_int(); fl = C.c_int(); tr = C.c_double(); hl = C.c_int()
        hist = np.zeros(max_iter + 8)
        self.lib.ref_stage_solve_cb.restype = C.c_int
        self._chk(self.lib.ref_stage_solve_cb(kind, solver, n, C.c_double(tau), C.c_double(a), cb, None, _p(b),
                                              _p(x0), C.c_double(tol), max_iter, _p(x), C.byref(it), C.byref(cv),
                                              C.byref(fl), C.byref(tr), _p(hist), len(hist), C.byref(hl)))
        return x, dict(iterations=it.value, converged=bool(cv.value), failure=fl.value,
                       true_residual=tr.value, history=hist[: hl.value].copy())

    def krylov_cb(self, kind, solver, op, precond, b, x0, tol, max_iter):
        """The reference's own cg (solver 0) / gmres (1) on a caller-defined
        system: op(x) and precond(x) (None: identity) are numpy callables
        (the ApplyFn slot, krylov.hpp:38-39)."""
        b = np.ascontiguousarray(b, dtype=DT[kind]); x0 = np.ascontiguousarray(x0, dtype=DT[kind])
        m = b.size
        x = np.empty_like(b)

        def wrap(fn):
            def tramp(ctx, xp, outp):
                xin = np.ctypeslib.as_array(C.cast(xp, C.POINTER(C.c_byte)), shape=(m * b.itemsize,)).view(b.dtype)
                out = np.ctypeslib.as_array(C.cast(outp, C.POINTER(C.c_byte)), shape=(m * b.itemsize,)).view(b.dtype)
                out[:] = fn(xin.copy())
            return self.CB(tramp)

        cbo = wrap(op)
        cbp = wrap(precond) if precond is not None else self.CB()
        it = C.c_int(); cv = C.c_int(); fl = C.c_int(); tr = C.c_double(); hl = C.c_int()
        hist = np.zeros(max_iter + 8)
        self.lib.ref_krylov_cb.restype = C.c_int
        self._chk(self.lib.ref_krylov_cb(kind, solver, C.c_longlong(m), cbo, None, cbp, None, _p(b), _p(x0),
                                         C.c_double(tol), max_iter, _p(x), C.byref(it), C.byref(cv), C.byref(fl),
                                         C.byref(tr), _p(hist), len(hist), C.byref(hl)))
        return x, dict(iterations=it.value, converged=bool(cv.value), failure=fl.value,
                       true_residual=tr.value, history=hist[: hl.value].copy())

    def stepper(self, eq, n, tab, tau, tol, precision, max_iter=40, t_end=0.1):
        return RefStepper(self, eq, n, tab, tau, tol, precision, max_iter, t_end)

    def integrate(self, eq, n, tab, tau, t_end, tol, precision, max_iter=40, reference=None):
        m = n ** 3
        state = np.zeros(m)
        em = C.c_double(); el = C.c_double(); mi = C.c_double(); ti = C.c_longlong()
        its = np.zeros(100000, np.int32); ns = C.c_int(); st = C.c_int(); sf = C.c_int(); ws = C.c_double()
        ref = None if reference is None else np.ascontiguousarray(reference, np.float64)
        q = tab["q"]
        self._chk(self.lib.ref_integrate(eq, n, q, _p(np.ascontiguousarray(tab["a_high"], np.float64)),
                                         _p(np.ascontiguousarray(tab["a_eps"], np.float64)),
                                         _p(np.ascontiguousarray(tab["b"], np.float64)),
                                         C.c_double(tau), C.c_double(t_end), C.c_double(tol),
                                         0 if precision == "f32" else 1, max_iter, _p(ref), _p(state),
                                         C.byref(em), C.byref(el), C.byref(mi), C.byref(ti), _p(its),
                                         len(its), C.byref(ns), C.byref(st), C.byref(sf), C.byref(ws)))
        nan = float("nan")
        return dict(state=state, error_max=None if np.isnan(em.value) else em.value,
                    error_l2=None if np.isnan(el.value) else el.value, mean_iterations=mi.value,
                    total_iterations=ti.value, solve_iterations=its[: ns.value].tolist(),
                    steps=st.value, solver_failure=bool(sf.value), wall_seconds=ws.value)


def _ref_temporal_order(self, eq, n, tab, taus, t_end, tol, precision, max_iter=40):
    taus = np.ascontiguousarray(taus, np.float64)
    em = np.zeros(taus.size); el = np.zeros(taus.size); slope = C.c_double(); sf = C.c_int()
    self._chk(self.lib.ref_temporal_order(eq, n, tab["q"], _p(np.ascontiguousarray(tab["a_high"], np.float64)),
                                          _p(np.ascontiguousarray(tab["a_eps"], np.float64)),
                                          _p(np.ascontiguousarray(tab["b"], np.float64)), C.c_double(t_end),
                                          C.c_double(tol), 0 if precision == "f32" else 1, max_iter, _p(taus),
                                          taus.size, _p(em), _p(el), C.byref(slope), C.byref(sf)))
    return dict(taus=taus.tolist(), errors_max=em.tolist(), errors_l2=el.tolist(), slope=slope.value,
                solver_failure=bool(sf.value))


Reference.temporal_order = _ref_temporal_order


class RefStepper:
    def __init__(self, R: Reference, eq, n, tab, tau, tol, precision, max_iter, t_end):
        self.R = R
        self.h = C.c_void_p()
        q = tab["q"]
        R._chk(R.lib.ref_stepper_create(eq, n, q, _p(np.ascontiguousarray(tab["a_high"], np.float64)),
                                        _p(np.ascontiguousarray(tab["a_eps"], np.float64)),
                                        _p(np.ascontiguousarray(tab["b"], np.float64)), C.c_double(tau),
                                        C.c_double(t_end), C.c_double(tol), 0 if precision == "f32" else 1,
                                        max_iter, C.byref(self.h)))

    def step(self, u):
        ns = C.c_int(); it = np.zeros(64, np.int32); cv = np.zeros(64, np.int32); sf = C.c_int()
        self.R._chk(self.R.lib.ref_stepper_step(self.h, _p(u), C.byref(ns), _p(it), _p(cv), 64, C.byref(sf)))
        return dict(iterations=it[: ns.value].tolist(), converged=[bool(c) for c in cv[: ns.value]],
                    solver_failure=bool(sf.value))

    def history(self, idx):
        h = np.zeros(256); ln = C.c_int()
        self.R._chk(self.R.lib.ref_stepper_history(self.h, idx, _p(h), 256, C.byref(ln)))
        return h[: ln.value].copy()

    def __del__(self):
        try:
            self.R.lib.ref_stepper_destroy(self.h)
        except Exception:
            pass


class _OrcReport(C.Structure):
    _fields_ = [("iterations", C.c_int), ("converged", C.c_int), ("failure", C.c_int),
                ("true_residual", C.c_double), ("history", C.POINTER(C.c_double)),
                ("history_len", C.c_int), ("history_cap", C.c_int)]


class Restatement:
    """The plain-C restatement (the oracle proper)."""

    SFX = {0: "f32", 1: "f64", 2: "c32", 3: "c64"}

    def __init__(self, path: str = ORACLE_SO):
        self.lib = C.CDLL(path)

    def make_problem(self, eq, n):
        m = n ** 3
        u0 = np.zeros(m); g = np.zeros(m) if eq == 0 else None
        h = C.c_double(); gam = C.c_double()
        rc = self.lib.orc_make_problem(eq, n, _p(u0), _p(g), C.byref(h), C.byref(gam))
        if rc:
            raise OracleError(rc)
        return u0, g, h.value, gam.value

    def heat_exact(self, n, t, g):
        out = np.zeros(n ** 3)
        self.lib.orc_heat_exact(n, C.c_double(t), _p(np.ascontiguousarray(g, np.float64)), _p(out))
        return out

    def stencil(self, kind, n, stencil, sigma, gamma, x):
        x = np.ascontiguousarray(x, dtype=DT[kind]); out = np.empty_like(x)
        getattr(self.lib, "orc_stencil_" + self.SFX[kind])(n, stencil, C.c_double(sigma), C.c_double(gamma), _p(x), _p(out))
        return out

    def tensor(self, kind, side, n, q, x):
        q = np.ascontiguousarray(q, dtype=DT[kind]); x = np.ascontiguousarray(x, dtype=DT[kind])
        out = np.empty_like(x)
        getattr(self.lib, "orc_tensor_" + self.SFX[kind])(side, n, _p(q), _p(x), _p(out))
        return out

    def spectral(self, periodic, n, sigma, gamma):
        dt = np.complex128 if periodic else np.float64
        q = np.zeros(n * n, dt); qi = np.zeros(n * n, dt); lam = np.zeros(n, dt)
        fn = self.lib.orc_spectral_periodic if periodic else self.lib.orc_spectral_dirichlet
        fn(n, C.c_double(sigma), C.c_double(gamma), _p(q), _p(qi), _p(lam))
        return q, qi, lam

    def stage_solve(self, kind, solver, n, tau, a, precond, b, x0, tol, max_iter):
        b = np.ascontiguousarray(b, dtype=DT[kind]); x = np.array(x0, dtype=DT[kind], copy=True)
        hist = np.zeros(max_iter + 8)
        rep = _OrcReport(0, 0, 0, 0.0, hist.ctypes.data_as(C.POINTER(C.c_double)), 0, len(hist))
        rc = self.lib.orc_stage_solve(kind, solver, n, C.c_double(tau), C.c_double(a), precond, _p(b), _p(x),
                                      C.c_double(tol), max_iter, C.byref(rep))
        if rc:
            raise OracleError(rc)
        return x, dict(iterations=rep.iterations, converged=bool(rep.converged), failure=rep.failure,
                       true_residual=rep.true_residual, history=hist[: rep.history_len].copy())

    def fastdiag(self, kind, n, tau, a, x):
        """One stage-preconditioner apply of make_problem(eq, n) (eq from kind)."""
        x = np.ascontiguousarray(x, dtype=DT[kind]); out = np.empty_like(x)
        h = 1.0 / (n - 1) if kind <= 1 else 1.0 / n
        gk = -1.0 / (h * h) if kind <= 1 else -1.0 / (2.0 * h)
        buf = (C.c_byte * 128)()
        rc = self.lib.orc_precond_build(kind, n, C.c_double(tau), C.c_double(a), C.c_double(gk), buf)
        if rc:
            raise OracleError(rc)
        self.lib.orc_precond_apply(buf, _p(x), _p(out))
        self.lib.orc_precond_free(buf)
        return out

    def stepper(self, eq, n, tab, tau, tol, precision, max_iter=40):
        return OrcStepper(self, eq, n, tab, tau, tol, precision, max_iter)


class OrcStepper:
    def __init__(self, O: Restatement, eq, n, tab, tau, tol, precision, max_iter):
        self.O = O
        self.h = C.c_void_p()
        rc = O.lib.orc_stepper_create(eq, n, tab["q"], _p(np.ascontiguousarray(tab["a_high"], np.float64)),
                                      _p(np.ascontiguousarray(tab["a_eps"], np.float64)),
                                      _p(np.ascontiguousarray(tab["b"], np.float64)), C.c_double(tau),
                                      C.c_double(tol), 1 if precision == "f32" else 0, max_iter, C.byref(self.h))
        if rc:
            raise OracleError(rc)

    def step(self, u):
        rc = self.O.lib.orc_stepper_step(self.h, _p(u))
        if rc:
            raise OracleError(rc)
        ns = C.c_int(); it = np.zeros(64, np.int32); cv = np.zeros(64, np.int32); sf = C.c_int()
        self.O.lib.orc_stepper_trace(self.h, C.byref(ns), _p(it), _p(cv), C.byref(sf))
        return dict(iterations=it[: ns.value].tolist(), converged=[bool(c) for c in cv[: ns.value]],
                    solver_failure=bool(sf.value))

    def history(self, idx):
        h = np.zeros(64); ln = C.c_int()
        self.O.lib.orc_stepper_history(self.h, idx, _p(h), 64, C.byref(ln))
        return h[: ln.value].copy()

    def __del__(self):
        try:
            self.O.lib.orc_stepper_destroy(self.h)
        except Exception:
            pass
