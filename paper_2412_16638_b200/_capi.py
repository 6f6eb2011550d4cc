"""ctypes binding of include/mprk_b200.h (the C-ABI of libmprk_b200.so).

This is the reference-side binding a Python user of the reference's
``mprk`` module (proj/python/bindings.cpp) switches to.  The shared library
must exist: there is no fallback of any kind.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MPRKB_LIB", os.path.join(_HERE, "libmprk_b200.so"))

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "or `make` at the repo root (the B200 path has no CPU fallback)")

lib = C.CDLL(LIB_PATH)

# ---- status codes -> exceptions (errors.hpp:9-58) ----------------------------
OK, ERROR, LENGTH_MISMATCH, DIMENSION_TOO_SMALL = 0, 1, 2, 3
SINGULAR_SYSTEM, POLE_AT_TWO, OVERFLOW_TO_INFINITY, ZERO_EIGENVALUE_SUM = 4, 5, 6, 7
WRONG_EQUATION, NONFINITE_STATE, INVALID_ARGUMENT, CUDA_ERROR, NO_DEVICE = 8, 9, 10, 20, 21

F32, F64, C32, C64, F16 = 0, 1, 2, 3, 4
FAST, PARITY = 0, 1
HEAT, ADVECTION, ADVECTION_DIFFUSION = 0, 1, 2
PRECOND_FASTDIAG, PRECOND_NONE, PRECOND_BLOCK_JACOBI = 0, 1, 2
MAX_STAGES = 16


class MprkError(RuntimeError):
    """mprk::Error (the reference's pybind11 exception is also MprkError)."""


class LengthMismatch(MprkError):
    pass


class DimensionTooSmall(MprkError):
    pass


class SingularSystem(MprkError):
    pass


class PoleAtTwo(MprkError):
    pass


class OverflowToInfinity(MprkError):
    pass


class ZeroEigenvalueSum(MprkError):
    pass


class WrongEquation(MprkError):
    pass


class NonFiniteState(MprkError):
    pass


class CudaError(RuntimeError):
    pass


class NoDevice(RuntimeError):
    pass


_EXC = {ERROR: MprkError, LENGTH_MISMATCH: LengthMismatch, DIMENSION_TOO_SMALL: DimensionTooSmall,
        SINGULAR_SYSTEM: SingularSystem, POLE_AT_TWO: PoleAtTwo, OVERFLOW_TO_INFINITY: OverflowToInfinity,
        ZERO_EIGENVALUE_SUM: ZeroEigenvalueSum, WRONG_EQUATION: WrongEquation,
        NONFINITE_STATE: NonFiniteState, INVALID_ARGUMENT: ValueError, CUDA_ERROR: CudaError,
        NO_DEVICE: NoDevice}


def check(rc: int) -> None:
    if rc != OK:
        msg = lib.mprkb_last_error().decode(errors="replace")
        raise _EXC.get(rc, MprkError)(msg)


# ---- structs -------------------------------------------------------------------
class SolveReport(C.Structure):
    _fields_ = [("iterations", C.c_int), ("converged", C.c_int), ("failure", C.c_int),
                ("true_residual", C.c_double), ("residual_history", C.POINTER(C.c_double)),
                ("history_capacity", C.c_int), ("history_length", C.c_int)]


class Config(C.Structure):
    _fields_ = [("equation", C.c_int), ("n", C.c_int), ("q", C.c_int),
                ("a_high", C.POINTER(C.c_double)), ("a_eps", C.POINTER(C.c_double)),
                ("b", C.POINTER(C.c_double)), ("tau", C.c_double), ("t_end", C.c_double),
                ("tol", C.c_double), ("implicit_precision", C.c_int), ("max_iter", C.c_int),
                ("numerics", C.c_int), ("preconditioner", C.c_int), ("block_size", C.c_int),
                ("block_storage", C.c_int), ("nu", C.c_double), ("record_timings", C.c_int),
                ("basis_storage", C.c_int), ("krylov_storage", C.c_int)]


class StepTrace(C.Structure):
    _fields_ = [("n_solves", C.c_int), ("solver_failure", C.c_int),
                ("iterations", C.c_int * MAX_STAGES), ("converged", C.c_int * MAX_STAGES),
                ("failure", C.c_int * MAX_STAGES), ("true_residual", C.c_double * MAX_STAGES)]


class Result(C.Structure):
    _fields_ = [("error_max", C.c_double), ("error_l2", C.c_double), ("mean_iterations", C.c_double),
                ("total_iterations", C.c_longlong), ("steps", C.c_int), ("solver_failure", C.c_int),
                ("wall_seconds", C.c_double), ("solve_iterations", C.POINTER(C.c_int)),
                ("solve_iterations_capacity", C.c_int), ("n_solves", C.c_int)]


APPLY_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p)
TIMING_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_char_p, C.c_longlong, C.c_double)

vp, i32, sz, f64 = C.c_void_p, C.c_int, C.c_size_t, C.c_double
dptr = C.POINTER(C.c_double)
ip = C.POINTER(C.c_int)
SIGNATURES = {
    "mprkb_last_error": (C.c_char_p, []),
    "mprkb_version": (i32, []),
    "mprkb_device_count": (i32, [ip]),
    "mprkb_malloc": (i32, [C.POINTER(vp), sz]),
    "mprkb_free": (i32, [vp]),
    "mprkb_memcpy_h2d": (i32, [vp, vp, sz, vp]),
    "mprkb_memcpy_d2h": (i32, [vp, vp, sz, vp]),
    "mprkb_memset": (i32, [vp, i32, sz, vp]),
    "mprkb_stream_synchronize": (i32, [vp]),
    "mprkb_device_synchronize": (i32, []),
    "mprkb_kernel_launches": (C.c_longlong, []),
    "mprkb_measure_fma_peak": (i32, [i32, dptr]),
    "mprkb_kernel_bench": (i32, [C.c_char_p, i32, i32, dptr, dptr]),
    "mprkb_make_problem": (i32, [i32, i32, vp, vp, dptr, dptr]),
    "mprkb_heat_exact": (i32, [i32, f64, vp]),
    "mprkb_builtin_tableau": (i32, [C.c_char_p, i32, ip, vp, vp, vp, vp]),
    "mprkb_stencil_apply": (i32, [i32, i32, i32, f64, f64, vp, vp, vp]),
    "mprkb_tensor_apply": (i32, [i32, i32, i32, vp, vp, vp, i32, vp]),
    "mprkb_dot": (i32, [i32, sz, vp, vp, i32, i32, dptr, vp]),
    "mprkb_tensor_apply_tc": (i32, [i32, i32, vp, vp, vp, vp]),
    "mprkb_tensor_apply_tc_fold": (i32, [i32, i32, vp, vp, vp, vp]),
    "mprkb_op_stencil": (i32, [i32, i32, i32, f64, f64, C.POINTER(vp)]),
    "mprkb_op_fastdiag": (i32, [i32, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp, i32, C.POINTER(vp)]),
    "mprkb_op_fastdiag_stage": (i32, [i32, i32, i32, f64, f64, i32, C.POINTER(vp)]),
    "mprkb_op_block_jacobi": (i32, [i32, i32, i32, f64, f64, i32, i32, C.POINTER(vp)]),
    "mprkb_op_block_jacobi_nu": (i32, [i32, i32, i32, f64, f64, f64, i32, i32, C.POINTER(vp)]),
    "mprkb_op_fastdiag_stage_nu": (i32, [i32, i32, i32, f64, f64, f64, i32, C.POINTER(vp)]),
    "mprkb_op_stage_operator": (i32, [i32, i32, i32, f64, f64, f64, C.POINTER(vp)]),
    "mprkb_op_csr": (i32, [i32, i32, vp, vp, vp, i32, C.POINTER(vp)]),
    "mprkb_op_csr_stencil": (i32, [i32, i32, i32, f64, f64, i32, C.POINTER(vp)]),
    "mprkb_op_callback": (i32, [i32, sz, APPLY_FN, vp, C.POINTER(vp)]),
    "mprkb_op_apply": (i32, [vp, vp, vp, vp]),
    "mprkb_op_destroy": (None, [vp]),
    "mprkb_cg": (i32, [i32, sz, vp, vp, vp, vp, f64, i32, i32, C.POINTER(SolveReport), vp]),
    "mprkb_gmres": (i32, [i32, sz, vp, vp, vp, vp, f64, i32, i32, C.POINTER(SolveReport), vp]),
    "mprkb_gmres_ex": (i32, [i32, sz, vp, vp, vp, vp, f64, i32, i32, i32, C.POINTER(SolveReport), vp]),
    "mprkb_cg_ex": (i32, [i32, sz, vp, vp, vp, vp, f64, i32, i32, i32, C.POINTER(SolveReport), vp]),
    "mprkb_config_init": (None, [C.POINTER(Config)]),
    "mprkb_stepper_create": (i32, [C.POINTER(Config), C.POINTER(vp)]),
    "mprkb_stepper_step": (i32, [vp, vp, C.POINTER(StepTrace)]),
    "mprkb_stepper_step_device": (i32, [vp, vp, C.POINTER(StepTrace)]),
    "mprkb_stepper_step_device_on": (i32, [vp, vp, C.POINTER(StepTrace), vp]),
    "mprkb_stepper_initial_state": (i32, [vp, vp]),
    "mprkb_stepper_history": (i32, [vp, i32, dptr, i32, ip]),
    "mprkb_stepper_stream": (vp, [vp]),
    "mprkb_stepper_timing": (i32, [vp, i32, C.POINTER(C.c_char_p), C.POINTER(C.c_longlong), dptr]),
    "mprkb_stepper_destroy": (None, [vp]),
    "mprkb_integrate": (i32, [C.POINTER(Config), vp, sz, vp, C.POINTER(Result)]),
    "mprkb_stepper_integrate": (i32, [vp, vp, sz, vp, C.POINTER(Result)]),
    "mprkb_temporal_order": (i32, [C.POINTER(Config), dptr, i32, dptr, dptr, dptr, ip]),
    "mprkb_stepper_integrate_from": (i32, [vp, vp, vp, sz, vp, C.POINTER(Result)]),
    # instrumentation and host helpers
    "mprkb_kron_apply_count": (C.c_longlong, [i32]),
    "mprkb_reset_kron_apply_counts": (None, []),
    "mprkb_spectral": (i32, [i32, i32, f64, f64, vp, vp, vp]),
    "mprkb_apply_f": (i32, [i32, i32, f64, f64, vp, i32, vp, vp, vp]),
    "mprkb_op_apply_timed": (i32, [vp, vp, vp, vp, TIMING_FN, vp]),
    # split grid (k-slab decomposition)
    "mprkb_set_device": (i32, [i32]),
    "mprkb_slab_plan": (i32, [i32, i32, i32, ip, ip, ip, ip]),
    "mprkb_nccl_unique_id": (i32, [C.c_char_p]),
    "mprkb_comm_create_nccl": (i32, [i32, i32, C.c_char_p, C.POINTER(vp)]),
    "mprkb_comm_group_create": (i32, [i32, C.POINTER(vp)]),
    "mprkb_comm_create_local": (i32, [vp, i32, C.POINTER(vp)]),
    "mprkb_comm_group_destroy": (None, [vp]),
    "mprkb_comm_destroy": (None, [vp]),
    "mprkb_comm_allreduce_sum": (i32, [vp, dptr, i32]),
    "mprkb_stepper_create_split": (i32, [C.POINTER(Config), vp, C.POINTER(vp)]),
    "mprkb_stepper_slab": (i32, [vp, ip, ip, C.POINTER(sz)]),
}

for _name, (_res, _args) in SIGNATURES.items():
    _f = getattr(lib, _name)  # AttributeError here = the library misses a declared symbol
    _f.restype = _res
    _f.argtypes = _args
