"""B200-native mixed-precision DIRK time stepping (arXiv 2412.16638).

Drop-in for the reference ``mprk`` Python module (proj/python/bindings.cpp,
proj/python/mprk/__init__.py): ``builtin``, ``midpoint_corrected``,
``Tableau``, ``validate``, ``integrate`` and ``MprkError`` keep the
reference's names, argument meaning and error behaviour; the time stepping
runs on the GPU through include/mprk_b200.h (libmprk_b200.so).

Lower-level device entry points (the reference's C++ plug-in boundary, the
``ApplyFn`` slot of ``cg``/``gmres``) take torch CUDA tensors:
``stencil_apply``, ``tensor_apply``, ``dot``, ``Operator``, ``cg``, ``gmres``
and the ``Stepper`` class.  torch is only device-memory plumbing here.
"""
from __future__ import annotations

import ctypes as C
import math
from typing import Optional

import numpy as np

from . import _capi as _c
from ._capi import (CudaError, DimensionTooSmall, LengthMismatch, MprkError, NoDevice, NonFiniteState,
                    OverflowToInfinity, WrongEquation, ZeroEigenvalueSum, check)

__all__ = [
    "MprkError", "LengthMismatch", "DimensionTooSmall", "OverflowToInfinity", "ZeroEigenvalueSum",
    "WrongEquation", "NonFiniteState", "CudaError", "NoDevice",
    "Tableau", "builtin", "midpoint_corrected", "validate", "integrate", "make_problem", "heat_exact",
    "Stepper", "Operator", "stencil_apply", "tensor_apply", "dot", "cg", "gmres", "kernel_launches",
    "device_count", "Comm", "LocalGroup", "slab_plan", "run_ranks", "set_device", "temporal_order",
    "tableau_from_json", "tableau_to_json",
]


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


# ---- tableaus (tableau.hpp / tableau.cpp) ---------------------------------------
class Tableau:
    """ButcherTableau (tableau.hpp:18-25): A = A_high + A_eps split."""

    def __init__(self, name: str = "", q: int = 0, c=None, a_high=None, a_eps=None, b=None):
        self.name = name
        self.q = q
        self.c = list(c or [])
        self.a_high = [list(r) for r in (a_high or [])]
        self.a_eps = [list(r) for r in (a_eps or [])]
        self.b = list(b or [])

    def __repr__(self) -> str:
        return f"<Tableau '{self.name}' with {self.q} stages>"

    def _arrays(self):
        q = self.q
        ah = np.ascontiguousarray(np.asarray(self.a_high, dtype=np.float64).reshape(q, q))
        ae = np.ascontiguousarray(np.asarray(self.a_eps, dtype=np.float64).reshape(q, q))
        b = np.ascontiguousarray(np.asarray(self.b, dtype=np.float64).reshape(q))
        return ah, ae, b


def _tableau_from_lib(name: str) -> Tableau:
    cap = 64 * 64
    ah = np.zeros(cap); ae = np.zeros(cap); b = np.zeros(64); c = np.zeros(64); q = C.c_int()
    check(_c.lib.mprkb_builtin_tableau(name.encode(), cap, C.byref(q), _dp(ah), _dp(ae), _dp(b), _dp(c)))
    q = q.value
    return Tableau(name, q, c[:q].tolist(), ah[: q * q].reshape(q, q).tolist(),
                   ae[: q * q].reshape(q, q).tolist(), b[:q].tolist())


def builtin(name: str) -> Tableau:
    """builtin_tableau(method_from_name(name)) (tableau.cpp:116-134)."""
    if name not in ("4s3pA", "4s3pB", "4s3pC"):
        raise MprkError("unknown method name: " + name)
    return _tableau_from_lib(name)


def midpoint_corrected(p: int) -> Tableau:
    """Implicit midpoint rule with p explicit corrector stages (tableau.cpp:135-144)."""
    if p < 0:
        raise MprkError("midpoint_corrected: corrector count must be nonnegative")
    return _tableau_from_lib(f"midpoint{int(p)}")


def _derive_c(a_high, a_eps):
    return [sum(a_high[i][j] + a_eps[i][j] for j in range(len(a_high[i]))) for i in range(len(a_high))]


def tableau_to_json(t: Tableau) -> str:
    """tableau_to_json (tableau.cpp:192-201): name, q, c, A_high, A_eps, b."""
    import json

    return json.dumps({"name": t.name, "q": t.q, "c": list(t.c), "A_high": [list(r) for r in t.a_high],
                       "A_eps": [list(r) for r in t.a_eps], "b": list(t.b)}, indent=2)


def tableau_from_json(text: str) -> Tableau:
    """tableau_from_json (tableau.cpp:203-233): a user tableau for the stepper;
    "c" is optional (row sums of A_high + A_eps).  Errors are MprkError with
    the reference's messages."""
    import json

    try:
        j = json.loads(text)
    except ValueError as e:
        raise MprkError(f"tableau JSON does not parse: {e}") from None
    try:
        name, q = str(j["name"]), j["q"]
        if not isinstance(q, int) or isinstance(q, bool):
            raise TypeError("q must be an integer")
        ah = [[float(v) for v in r] for r in j["A_high"]]
        ae = [[float(v) for v in r] for r in j["A_eps"]]
        b = [float(v) for v in j["b"]]
        c = [float(v) for v in j["c"]] if "c" in j else _derive_c(ah, ae)
    except (KeyError, TypeError, ValueError) as e:
        raise MprkError(f"tableau JSON has a wrong field: {e}") from None
    if q <= 0 or len(b) != q or len(ah) != q or len(ae) != q:
        raise MprkError("tableau JSON dimensions are inconsistent with q")
    if any(len(r) != q for r in ah):
        raise MprkError("A_high rows must have length q")
    if any(len(r) != q for r in ae):
        raise MprkError("A_eps rows must have length q")
    if len(c) != q:
        raise MprkError("c must have length q")
    return Tableau(name, q, c, ah, ae, b)


def validate(t: Tableau) -> list:
    """Structural checks (tableau.cpp:146-190); one line per violation."""
    tol = 1e-13
    out = []
    q = t.q
    if q <= 0:
        out.append("stage count must be positive")

    def shape_ok(m):
        return len(m) == q and all(len(r) == q for r in m)

    if not shape_ok(t.a_high) or not shape_ok(t.a_eps) or len(t.b) != q or len(t.c) != q:
        out.append("coefficient blocks must all be q-by-q and q-long")
        return out
    for i in range(q):
        row = 0.0
        for j in range(q):
            row += t.a_high[i][j] + t.a_eps[i][j]
        if abs(row - t.c[i]) > tol:
            out.append(f"c[{i}] does not match the row sum of A_high + A_eps")
    bsum = 0.0
    for w in t.b:
        bsum += w
    if abs(bsum - 1.0) > tol:
        out.append("sum(b) must be 1")
    if any(t.a_high[i][j] != 0.0 or t.a_eps[i][j] != 0.0 for i in range(q) for j in range(i + 1, q)):
        out.append("A_high + A_eps must be lower triangular")
    if any(t.a_high[i][i] != 0.0 for i in range(q)):
        out.append("diagonal (implicit) coefficients must live in A_eps only")
    return out


# ---- problems -------------------------------------------------------------------------
_EQ = {"heat": _c.HEAT, "advection": _c.ADVECTION, "advection-diffusion": _c.ADVECTION_DIFFUSION,
       "advection_diffusion": _c.ADVECTION_DIFFUSION}
_PREC = {"f32": _c.F32, "f64": _c.F64}
_NUM = {"fast": _c.FAST, "parity": _c.PARITY}
_PRE = {"fastdiag": _c.PRECOND_FASTDIAG, "none": _c.PRECOND_NONE, "block-jacobi": _c.PRECOND_BLOCK_JACOBI,
        "block_jacobi": _c.PRECOND_BLOCK_JACOBI}
_STORE = {None: -1, "f16": _c.F16, "f32": _c.F32, "f64": _c.F64}


def _parse(table, key, what, want):
    if key not in table:
        raise ValueError(f"unknown {what}: {key} (want {want})")
    return table[key]


def make_problem(equation: str, n: int):
    """make_problem (operators.cpp:29-65) -> (u0, forcing or None, h, gamma_K)."""
    eq = _parse(_EQ, equation, "equation", "heat or advection")
    m = n ** 3 if n > 0 else 0
    u0 = np.zeros(max(m, 1)); g = np.zeros(max(m, 1))
    h = C.c_double(); gam = C.c_double()
    check(_c.lib.mprkb_make_problem(eq, n, _dp(u0), _dp(g), C.byref(h), C.byref(gam)))
    return u0[:m], (g[:m] if eq == _c.HEAT else None), h.value, gam.value


def heat_exact(n: int, t: float) -> np.ndarray:
    out = np.zeros(n ** 3)
    check(_c.lib.mprkb_heat_exact(n, t, _dp(out)))
    return out


def _config(tableau: Tableau, equation, n, tau, t_end, tol, precision, max_iter, numerics, preconditioner,
            block_size, block_storage, nu, timings, basis_storage=None, krylov_storage=None):
    cfg = _c.Config()
    _c.lib.mprkb_config_init(C.byref(cfg))
    cfg.equation = _parse(_EQ, equation, "equation", "heat or advection")
    cfg.n = int(n)
    ah, ae, b = tableau._arrays()
    cfg.q = tableau.q
    keep = (ah, ae, b)
    cfg.a_high = ah.ctypes.data_as(C.POINTER(C.c_double))
    cfg.a_eps = ae.ctypes.data_as(C.POINTER(C.c_double))
    cfg.b = b.ctypes.data_as(C.POINTER(C.c_double))
    cfg.tau = float(tau)
    cfg.t_end = float(t_end)
    cfg.tol = float(tol)
    cfg.implicit_precision = _parse(_PREC, precision, "precision", "f32 or f64")
    cfg.max_iter = int(max_iter)
    cfg.numerics = _parse(_NUM, numerics, "numerics", "fast or parity")
    cfg.preconditioner = _parse(_PRE, preconditioner, "preconditioner", "fastdiag, none or block-jacobi")
    cfg.block_size = int(block_size)
    cfg.block_storage = _parse(_STORE, block_storage, "storage", "f16, f32 or f64")
    cfg.nu = float(nu)
    cfg.record_timings = 1 if timings else 0
    cfg.basis_storage = _parse({None: -1, "f16": _c.F16}, basis_storage, "basis storage", "None or f16")
    cfg.krylov_storage = _parse({None: -1, "f16": _c.F16, "f32": _c.F32}, krylov_storage, "krylov storage",
                                "None, f16 or f32")
    return cfg, keep


class Stepper:
    """Stepper(problem, cfg) (stepper.hpp:53-65) on the GPU.

    ``step(u)`` takes a numpy float64 vector (host, updated in place, copied
    in/out each call); ``step_device(u)`` a torch CUDA float64 tensor that
    stays resident in HBM.

    With ``comm`` (a :class:`Comm`) the grid is split into k-slabs across the
    communicator's ranks: every vector argument is this rank's slab
    (``size`` = n*n*nz elements starting at plane ``k0``) and all ranks must
    call every method together.
    """

    def __init__(self, equation: str, n: int, tableau: Tableau, tau: float, tol: float = 1e-6,
                 precision: str = "f64", max_iter: int = 40, *, t_end: float = 0.1, numerics: str = "fast",
                 preconditioner: str = "fastdiag", block_size: int = 8, block_storage: Optional[str] = None,
                 nu: float = 0.0, timings: bool = False, basis_storage: Optional[str] = None,
                 krylov_storage: Optional[str] = None, comm: Optional["Comm"] = None):
        cfg, keep = _config(tableau, equation, n, tau, t_end, tol, precision, max_iter, numerics,
                            preconditioner, block_size, block_storage, nu, timings, basis_storage,
                            krylov_storage)
        self._h = C.c_void_p()
        self._comm = comm  # keeps the communicator alive as long as the stepper
        if comm is None:
            check(_c.lib.mprkb_stepper_create(C.byref(cfg), C.byref(self._h)))
        else:
            check(_c.lib.mprkb_stepper_create_split(C.byref(cfg), comm._h, C.byref(self._h)))
        self.n = int(n)
        k0, nz, m = C.c_int(), C.c_int(), C.c_size_t()
        check(_c.lib.mprkb_stepper_slab(self._h, C.byref(k0), C.byref(nz), C.byref(m)))
        self.k0, self.nz, self.size = k0.value, nz.value, m.value
        self._trace = _c.StepTrace()

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _c is not None and _c.lib is not None:  # (module globals are gone at shutdown)
            _c.lib.mprkb_stepper_destroy(h)
            self._h = None

    @property
    def stream(self) -> int:
        return _c.lib.mprkb_stepper_stream(self._h) or 0

    def initial_state(self) -> np.ndarray:
        u = np.zeros(self.size)
        check(_c.lib.mprkb_stepper_initial_state(self._h, _dp(u)))
        return u

    def _trace_dict(self):
        t = self._trace
        k = t.n_solves
        return dict(iterations=list(t.iterations[:k]), converged=[bool(c) for c in t.converged[:k]],
                    failure=list(t.failure[:k]), true_residual=list(t.true_residual[:k]),
                    solver_failure=bool(t.solver_failure))

    def step(self, u: np.ndarray) -> dict:
        if u.dtype != np.float64 or not u.flags.c_contiguous or u.size != self.size:
            raise LengthMismatch("step: u must be a contiguous float64 vector of length n^3 (split: the slab)")
        check(_c.lib.mprkb_stepper_step(self._h, _dp(u), C.byref(self._trace)))
        return self._trace_dict()

    def step_device(self, u) -> dict:
        """One step on a CUDA float64 tensor (no host copies)."""
        if u.dtype.is_complex or u.element_size() != 8 or u.numel() != self.size or not u.is_contiguous():
            raise LengthMismatch("step_device: u must be a contiguous CUDA float64 tensor of length n^3")
        # ordered after torch's current stream (whatever produced u)
        import torch
        cs = torch.cuda.current_stream(u.device).cuda_stream
        check(_c.lib.mprkb_stepper_step_device_on(self._h, C.c_void_p(u.data_ptr()), C.byref(self._trace),
                                                  C.c_void_p(cs)))
        return self._trace_dict()

    def history(self, idx: int) -> np.ndarray:
        buf = np.zeros(4096); ln = C.c_int()
        check(_c.lib.mprkb_stepper_history(self._h, idx, buf.ctypes.data_as(C.POINTER(C.c_double)), 4096,
                                           C.byref(ln)))
        return buf[: ln.value].copy()

    def timings(self) -> dict:
        out = {}
        label = C.c_char_p(); cnt = C.c_longlong(); sec = C.c_double()
        n = _c.lib.mprkb_stepper_timing(self._h, -1, None, None, None)
        for i in range(n):
            _c.lib.mprkb_stepper_timing(self._h, i, C.byref(label), C.byref(cnt), C.byref(sec))
            out[label.value.decode()] = dict(count=cnt.value, total_seconds=sec.value,
                                             seconds_per_call=sec.value / cnt.value if cnt.value else 0.0)
        return out

    def integrate(self, reference: Optional[np.ndarray] = None) -> dict:
        state = np.zeros(self.size)
        its = np.zeros(1 << 20, dtype=np.int32)
        res = _c.Result()
        res.solve_iterations = its.ctypes.data_as(C.POINTER(C.c_int))
        res.solve_iterations_capacity = len(its)
        ref = None if reference is None else np.ascontiguousarray(reference, dtype=np.float64)
        check(_c.lib.mprkb_stepper_integrate(self._h, None if ref is None else _dp(ref),
                                             0 if ref is None else ref.size, _dp(state), C.byref(res)))
        return _result_dict(res, its, state)


# ---- split grid: communicators ----------------------------------------------------------
def set_device(device: int) -> None:
    """cudaSetDevice for the calling thread inside libmprk_b200."""
    check(_c.lib.mprkb_set_device(int(device)))


def slab_plan(n: int, size: int, rank: int) -> dict:
    """k-slab (state) and j-slab (FastDiag transpose) of `rank` in a `size`-way split."""
    k0, nz, j0, ny = C.c_int(), C.c_int(), C.c_int(), C.c_int()
    check(_c.lib.mprkb_slab_plan(int(n), int(size), int(rank), C.byref(k0), C.byref(nz), C.byref(j0),
                                 C.byref(ny)))
    return dict(k0=k0.value, nz=nz.value, j0=j0.value, ny=ny.value)


class Comm:
    """One rank's communicator: NCCL (one process per GPU) or the in-process
    group (ranks = threads sharing one GPU)."""

    def __init__(self, handle, rank: int, size: int, keep=None):
        self._h = handle
        self.rank, self.size = rank, size
        self._keep = keep

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        check(_c.lib.mprkb_nccl_unique_id(buf))
        return buf.raw

    @classmethod
    def nccl(cls, rank: int, size: int, unique_id: bytes) -> "Comm":
        h = C.c_void_p()
        check(_c.lib.mprkb_comm_create_nccl(int(rank), int(size), C.c_char_p(bytes(unique_id)), C.byref(h)))
        return cls(h, rank, size)

    def allreduce_sum(self, values) -> np.ndarray:
        v = np.ascontiguousarray(values, dtype=np.float64).copy()
        check(_c.lib.mprkb_comm_allreduce_sum(self._h, v.ctypes.data_as(C.POINTER(C.c_double)), v.size))
        return v

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _c is not None and _c.lib is not None:  # (module globals are gone at shutdown)
            _c.lib.mprkb_comm_destroy(h)
            self._h = None


class LocalGroup:
    """`size` ranks in this process on one device (every split code path on a
    single GPU); ``comm(rank)`` is called from that rank's thread."""

    def __init__(self, size: int):
        self._h = C.c_void_p()
        check(_c.lib.mprkb_comm_group_create(int(size), C.byref(self._h)))
        self.size = int(size)

    def comm(self, rank: int) -> Comm:
        h = C.c_void_p()
        check(_c.lib.mprkb_comm_create_local(self._h, int(rank), C.byref(h)))
        return Comm(h, rank, self.size, keep=self)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _c is not None and _c.lib is not None:  # (module globals are gone at shutdown)
            _c.lib.mprkb_comm_group_destroy(h)
            self._h = None


def run_ranks(size: int, fn, device: int = 0) -> list:
    """Run fn(rank, comm) for `size` in-process ranks (one thread each, all on
    `device`) and return the results in rank order; re-raises the first
    rank's exception."""
    import threading

    group = LocalGroup(size)
    out = [None] * size
    errs = [None] * size

    def body(r):
        try:
            set_device(device)
            comm = group.comm(r)
            try:
                out[r] = fn(r, comm)
            finally:
                del comm
        except BaseException as e:  # noqa: BLE001 - re-raised below
            errs[r] = e

    ts = [threading.Thread(target=body, args=(r,)) for r in range(size)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for e in errs:
        if e is not None:
            raise e
    return out


def _result_dict(res, its, state):
    em = None if math.isnan(res.error_max) else res.error_max
    el = None if math.isnan(res.error_l2) else res.error_l2
    return dict(steps=res.steps, solver_failure=bool(res.solver_failure), mean_iterations=res.mean_iterations,
                total_iterations=res.total_iterations, solve_iterations=its[: res.n_solves].tolist(),
                wall_seconds=res.wall_seconds, state=state, error_max=em, error_l2=el)


def integrate(tableau: Tableau, equation: str, n: int, tau: float, t_end: float, tol: float = 1e-6,
              precision: str = "f64", max_iter: int = 40, *, numerics: str = "fast",
              preconditioner: str = "fastdiag", block_size: int = 8, block_storage: Optional[str] = None,
              nu: float = 0.0, reference: Optional[np.ndarray] = None,
              basis_storage: Optional[str] = None) -> dict:
    """mprk.integrate (bindings.cpp:130-147): run the split-tableau integrator
    on a built-in problem; returns the reference's result dict (steps,
    solver_failure, mean_iterations, total_iterations, solve_iterations,
    wall_seconds, state, error_max, error_l2, timings)."""
    eq = _parse(_EQ, equation, "equation", "heat or advection")
    _parse(_PREC, precision, "precision", "f32 or f64")
    if int(n) < (2 if eq == _c.HEAT else 3):
        raise DimensionTooSmall("make_problem: grid too small for the requested equation")
    # tau-divides-t_end check before building anything (stepper.cpp:220-225)
    if not tau > 0.0:
        raise MprkError("integrate: tau must be positive")
    steps = round(t_end / tau)
    if steps < 1 or abs(steps * tau - t_end) > 1e-9 * max(1.0, abs(t_end)):
        raise MprkError("integrate: tau must divide t_end")
    st = Stepper(equation, n, tableau, tau, tol, precision, max_iter, t_end=t_end, numerics=numerics,
                 preconditioner=preconditioner, block_size=block_size, block_storage=block_storage, nu=nu,
                 timings=True, basis_storage=basis_storage)
    out = st.integrate(reference)
    out["timings"] = st.timings()
    return out


def temporal_order(tableau: Tableau, equation: str, n: int, taus, t_end: float = 0.1, tol: float = 1e-6,
                   precision: str = "f64", max_iter: int = 40, *, numerics: str = "fast",
                   preconditioner: str = "fastdiag", nu: float = 0.0) -> dict:
    """temporal_order(problem, cfg, taus) (stepper.cpp:271-310) on the GPU:
    errors of each tau against one tiny-tau fp64 run and the least-squares
    log-log slope.  Returns dict(taus, errors_max, errors_l2, slope,
    solver_failure)."""
    taus = np.ascontiguousarray(list(taus), dtype=np.float64)
    if taus.size == 0:
        raise MprkError("temporal_order: tau list must not be empty")
    cfg, keep = _config(tableau, equation, n, float(taus[0]), t_end, tol, precision, max_iter, numerics,
                        preconditioner, 8, None, nu, False)
    em = np.zeros(taus.size); el = np.zeros(taus.size); slope = C.c_double(); sf = C.c_int()
    check(_c.lib.mprkb_temporal_order(C.byref(cfg), taus.ctypes.data_as(C.POINTER(C.c_double)), taus.size,
                                      em.ctypes.data_as(C.POINTER(C.c_double)),
                                      el.ctypes.data_as(C.POINTER(C.c_double)), C.byref(slope), C.byref(sf)))
    return dict(taus=taus.tolist(), errors_max=em.tolist(), errors_l2=el.tolist(), slope=slope.value,
                solver_failure=bool(sf.value))


# ---- device-level entry points (torch CUDA tensors) ---------------------------------
def _torch():
    import torch  # plumbing only: device memory and the current stream
    return torch


def _dtype_code(t) -> int:
    torch = _torch()
    m = {torch.float32: _c.F32, torch.float64: _c.F64, torch.complex64: _c.C32, torch.complex128: _c.C64}
    if t.dtype not in m:
        raise ValueError(f"unsupported dtype {t.dtype}")
    if not t.is_cuda or not t.is_contiguous():
        raise ValueError("expected a contiguous CUDA tensor")
    return m[t.dtype]


def _stream() -> C.c_void_p:
    torch = _torch()
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t) -> C.c_void_p:
    return C.c_void_p(t.data_ptr())


def stencil_apply(x, n: int, stencil: int, sigma: float, gamma: float):
    """KronSumOperator{n, stencil, sigma, gamma}.apply(x) (operators.hpp:113-161)."""
    dt = _dtype_code(x)
    if x.numel() != n ** 3:
        raise LengthMismatch("KronSumOperator: input length != n^3")
    out = _torch().empty_like(x)
    check(_c.lib.mprkb_stencil_apply(dt, n, stencil, sigma, gamma, _ptr(x), _ptr(out), _stream()))
    return out


def tensor_apply(side: int, n: int, q, x, numerics: str = "fast"):
    """apply_tensor(side, n, Q, x) (precond.hpp:69-122); side 0 L, 1 M, 2 R."""
    dt = _dtype_code(x)
    if q.numel() != n * n:
        raise LengthMismatch("apply_tensor: Q must be n*n")
    if x.numel() != n ** 3:
        raise LengthMismatch("apply_tensor: x must be n^3")
    out = _torch().empty_like(x)
    check(_c.lib.mprkb_tensor_apply(dt, side, n, _ptr(q), _ptr(x), _ptr(out), _NUM[numerics], _stream()))
    return out


def dot(a, b, conjugate: bool = False, numerics: str = "fast"):
    """detail::dot_real / dot (krylov.hpp:43-66)."""
    dt = _dtype_code(a)
    res = (C.c_double * 2)()
    check(_c.lib.mprkb_dot(dt, a.numel(), _ptr(a), _ptr(b), 1 if conjugate else 0, _NUM[numerics], res,
                           _stream()))
    if dt >= 2 and conjugate:
        return complex(res[0], res[1])
    return res[0]


class Operator:
    """An ApplyFn<T> (krylov.hpp:38-39) living on the device."""

    def __init__(self, handle: C.c_void_p, dtype: int, size: int, keep=None):
        self._h = handle
        self.dtype = dtype
        self.size = size
        self._keep = keep

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _c is not None and _c.lib is not None:  # (module globals are gone at shutdown)
            _c.lib.mprkb_op_destroy(h)
            self._h = None

    def apply(self, x):
        out = _torch().empty_like(x)
        check(_c.lib.mprkb_op_apply(self._h, _ptr(x), _ptr(out), _stream()))
        return out

    @staticmethod
    def stencil(dtype: int, n: int, stencil: int, sigma: float, gamma: float) -> "Operator":
        h = C.c_void_p()
        check(_c.lib.mprkb_op_stencil(dtype, n, stencil, sigma, gamma, C.byref(h)))
        return Operator(h, dtype, n ** 3)

    @staticmethod
    def stage_operator(dtype: int, equation: str, n: int, tau: float, a: float, nu: float = 0.0) -> "Operator":
        """stage_operator(make_problem(equation, n), tau, a) = I - tau a K (operators.cpp:77-79);
        nu: diffusion coefficient of the advection-diffusion extension."""
        h = C.c_void_p()
        check(_c.lib.mprkb_op_stage_operator(dtype, _EQ[equation], n, nu, tau, a, C.byref(h)))
        return Operator(h, dtype, n ** 3)

    @staticmethod
    def fastdiag_stage(dtype: int, equation: str, n: int, tau: float, a: float,
                       numerics: str = "fast", nu: float = 0.0) -> "Operator":
        """build_heat_precond(_f32) / build_advection_precond(_f32) (precond.cpp:14-42)."""
        h = C.c_void_p()
        check(_c.lib.mprkb_op_fastdiag_stage_nu(dtype, _EQ[equation], n, nu, tau, a, _NUM[numerics], C.byref(h)))
        return Operator(h, dtype, n ** 3)

    @staticmethod
    def fastdiag(dtype: int, n: int, qa, qa_inv, qb, qb_inv, qc, qc_inv, la, lb, lc,
                 numerics: str = "fast") -> "Operator":
        """FastDiagPreconditioner<T>(n, qa, ..., lambda_c) (precond.hpp:36-39); numpy host arrays."""
        npdt = {0: np.float32, 1: np.float64, 2: np.complex64, 3: np.complex128}[dtype]
        arrs = [np.ascontiguousarray(a, dtype=npdt) for a in (qa, qa_inv, qb, qb_inv, qc, qc_inv, la, lb, lc)]
        h = C.c_void_p()
        check(_c.lib.mprkb_op_fastdiag(dtype, n, *[_dp(a) for a in arrs], _NUM[numerics], C.byref(h)))
        return Operator(h, dtype, n ** 3)

    @staticmethod
    def block_jacobi(dtype: int, equation: str, n: int, tau: float, a: float, block: int,
                     storage: str = "f32", nu: float = 0.0) -> "Operator":
        h = C.c_void_p()
        check(_c.lib.mprkb_op_block_jacobi_nu(dtype, _EQ[equation], n, nu, tau, a, block, _STORE[storage],
                                              C.byref(h)))
        return Operator(h, dtype, n ** 3)

    @staticmethod
    def csr_stencil(dtype: int, n: int, stencil: int, sigma: float, gamma: float,
                    storage: str = "f32") -> "Operator":
        h = C.c_void_p()
        check(_c.lib.mprkb_op_csr_stencil(dtype, n, stencil, sigma, gamma, _STORE[storage], C.byref(h)))
        return Operator(h, dtype, n ** 3)

    @staticmethod
    def csr(dtype: int, rows: int, row_ptr, cols, values, storage: str = "f32") -> "Operator":
        rp = np.ascontiguousarray(row_ptr, dtype=np.int32)
        cl = np.ascontiguousarray(cols, dtype=np.int32)
        vdt = {"f16": np.float16, "f32": np.float32, "f64": np.float64}[storage]
        vl = np.ascontiguousarray(values, dtype=vdt)
        h = C.c_void_p()
        check(_c.lib.mprkb_op_csr(dtype, rows, _dp(rp), _dp(cl), _dp(vl), _STORE[storage], C.byref(h)))
        return Operator(h, dtype, rows)

    @staticmethod
    def callback(dtype: int, size: int, fn) -> "Operator":
        """Wrap fn(x_ptr, out_ptr, stream) -> None (device pointers) as an ApplyFn."""

        def tramp(ctx, x, out, stream):
            try:
                fn(x, out, stream)
                return 0
            except Exception:  # surfaced as mprk::Error by the library
                return 1

        cb = _c.APPLY_FN(tramp)
        h = C.c_void_p()
        check(_c.lib.mprkb_op_callback(dtype, size, cb, None, C.byref(h)))
        return Operator(h, dtype, size, keep=cb)


def _krylov(fn, op: Operator, precond: Optional[Operator], b, x0, tol, max_iter, numerics, extra=()):
    dt = _dtype_code(b)
    x = x0.clone()
    hist = np.zeros(max_iter + 8)
    rep = _c.SolveReport(0, 0, 0, 0.0, hist.ctypes.data_as(C.POINTER(C.c_double)), len(hist), 0)
    check(fn(dt, b.numel(), op._h, precond._h if precond is not None else None, _ptr(b), _ptr(x), tol, max_iter,
             _NUM[numerics], *extra, C.byref(rep), _stream()))
    return x, dict(iterations=rep.iterations, converged=bool(rep.converged), failure=rep.failure,
                   true_residual=rep.true_residual, history=hist[: rep.history_length].copy())


def cg(op: Operator, precond: Optional[Operator], b, x0, tol: float = 1e-6, max_iter: int = 40,
       numerics: str = "fast", storage: Optional[str] = None):
    """cg<T>(op, precond, b, x0, crit, report) (krylov.hpp:100-168) -> (x, report).
    storage="f16" (or "f32" for float64 systems) keeps r, z, p, q in that
    precision and computes in the system's (accessor-style extension:
    heat stencil operator, block-Jacobi or no preconditioner)."""
    if storage is None:
        return _krylov(_c.lib.mprkb_cg, op, precond, b, x0, tol, max_iter, numerics)
    code = _parse({"f16": _c.F16, "f32": _c.F32}, storage, "vector storage", "None, f16 or f32")
    return _krylov(_c.lib.mprkb_cg_ex, op, precond, b, x0, tol, max_iter, numerics, extra=(code,))


def gmres(op: Operator, precond: Optional[Operator], b, x0, tol: float = 1e-6, max_iter: int = 40,
          numerics: str = "fast", basis_storage: Optional[str] = None):
    """gmres<T>(op, precond, b, x0, crit, report) (krylov.hpp:181-311) -> (x, report).
    basis_storage="f16" keeps the Krylov basis in fp16 (extension)."""
    if basis_storage is None:
        return _krylov(_c.lib.mprkb_gmres, op, precond, b, x0, tol, max_iter, numerics)
    code = _parse({"f16": _c.F16}, basis_storage, "basis storage", "None or f16")
    return _krylov(_c.lib.mprkb_gmres_ex, op, precond, b, x0, tol, max_iter, numerics, extra=(code,))


def kernel_launches() -> int:
    return _c.lib.mprkb_kernel_launches()


def device_count() -> int:
    n = C.c_int()
    check(_c.lib.mprkb_device_count(C.byref(n)))
    return n.value
