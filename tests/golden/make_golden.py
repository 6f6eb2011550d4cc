"""Generate tests/golden/golden.npz from the UNMODIFIED reference.

Run in the build container (where /root/reference exists):
    make ref && python tests/golden/make_golden.py
The fixtures pin the C restatement (oracle/liboracle.so) even where the
reference library cannot be built; tests/test_oracle.py checks both against
them.  Every array is produced by oracle/_ref/libmprk_ref.so (the reference's
own sources compiled by oracle/Makefile) through oracle/ref_shim.cpp.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle.oracle import Reference  # noqa: E402


def main():
    R = Reference()
    R.set_threads(1)
    out = {}
    rng = np.random.default_rng(20241216)
    for name in ("4s3pA", "4s3pB", "4s3pC", "midpoint0", "midpoint1", "midpoint3"):
        t = R.tableau(name)
        out[f"tab_{name}_ah"] = t["a_high"]
        out[f"tab_{name}_ae"] = t["a_eps"]
        out[f"tab_{name}_b"] = t["b"]
        out[f"tab_{name}_c"] = t["c"]
    for eq, n in ((0, 6), (1, 6)):
        u0, g, h, gam = R.make_problem(eq, n)
        out[f"prob{eq}_u0"] = u0
        out[f"prob{eq}_hg"] = np.array([h, gam])
        if g is not None:
            out[f"prob{eq}_g"] = g
    DT = {0: np.float32, 1: np.float64, 2: np.complex64, 3: np.complex128}
    for kind in range(4):
        n = 5
        x = rng.uniform(-1, 1, n ** 3)
        if kind >= 2:
            x = x + 1j * rng.uniform(-1, 1, n ** 3)
        x = x.astype(DT[kind])
        q = rng.uniform(-1, 1, n * n)
        if kind >= 2:
            q = q + 1j * rng.uniform(-1, 1, n * n)
        q = q.astype(DT[kind])
        out[f"k{kind}_x"] = x
        out[f"k{kind}_q"] = q
        for st in (0, 1):
            out[f"k{kind}_stencil{st}"] = R.stencil(kind, n, st, 1.0, -0.37, x)
        for side in range(3):
            out[f"k{kind}_tensor{side}"] = R.tensor(kind, side, n, q, x)
        tau = 0.01 if kind <= 1 else 1.0 / 640.0
        out[f"k{kind}_fastdiag"] = R.fastdiag(kind, n, tau, 0.5, x)
    for kind, solver in ((0, 0), (1, 0), (2, 1), (3, 1)):
        n = 6
        b = rng.uniform(-1, 1, n ** 3).astype(DT[kind])
        tau = 0.025 if kind <= 1 else 1.0 / 640.0
        for tol in (1e-3, 1e-8):
            x, rep = R.stage_solve(kind, solver, n, tau, 0.5, 1, b, b, tol, 40)
            key = f"solve{kind}_{tol:g}"
            out[key + "_b"] = b
            out[key + "_x"] = x
            out[key + "_hist"] = rep["history"]
            out[key + "_meta"] = np.array([rep["iterations"], rep["converged"], rep["failure"], rep["true_residual"]])
    for name, eq, prec in (("midpoint1", 0, "f32"), ("4s3pB", 0, "f64"), ("4s3pC", 1, "f32")):
        t = R.tableau(name)
        n = 6
        tau = 0.01 if eq == 0 else 1.0 / 640.0
        s = R.stepper(eq, n, t, tau, 1e-5, prec)
        u, *_ = R.make_problem(eq, n)
        u = rng.uniform(0, 1, n ** 3) if eq == 0 else u
        out[f"step_{name}_{eq}_{prec}_u0"] = u.copy()
        its = []
        for _ in range(2):
            its += s.step(u)["iterations"]
        out[f"step_{name}_{eq}_{prec}_u2"] = u
        out[f"step_{name}_{eq}_{prec}_its"] = np.array(its)
    # config 1: heat 32^3 midpoint1, fp32 implicit, tau 0.01, 10 steps, tol 1e-4
    t = R.tableau("midpoint1")
    r = R.integrate(0, 32, t, 0.01, 0.1, 1e-4, "f32")
    out["cfg1_state"] = r["state"]
    out["cfg1_meta"] = np.array([r["error_max"], r["error_l2"], r["mean_iterations"]])
    out["cfg1_its"] = np.array(r["solve_iterations"])
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)
    print("wrote", os.path.join(HERE, "golden.npz"), len(out), "arrays")


if __name__ == "__main__":
    main()
