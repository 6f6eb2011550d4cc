"""Generate tests/golden/configs.npz — BASELINE.json configs[1] pinned by the
UNMODIFIED reference (oracle/_ref/libmprk_ref.so, the reference's own sources
compiled by oracle/Makefile, driven through oracle/ref_shim.cpp).

Run in the build container (where /root/reference exists; ~30 min on 8 cores):
    make ref && python tests/golden/make_golden_configs.py

What it records (consumed by tests/test_gpu_configs.py):
* ``c2_*``  heat 256^3, 4s3pB, tau 0.01, t_end 0.1 (10 steps), F32 implicit
  stages at tol 1e-3 and F64 at tol 1e-5 through the
  reference's ``integrate`` (stepper.cpp:218-269): error_max / error_l2 against
  heat_exact, the per-solve iteration counts, and the final state subsampled on
  every 8th grid line in each direction (32^3 points) plus full-grid moments.
* ``m1_*``  heat 256^3, midpoint1, one step (t_end = tau = 0.01) at F32 tol 1e-3
  and F64 tol 1e-5 (SURVEY.md §8(c) golden values 1.312229e-02 / 1.012499e-04).
"""
import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle.oracle import Reference  # noqa: E402

N = 256
SUB = 8


def sub(state):
    return state.reshape(N, N, N)[::SUB, ::SUB, ::SUB].copy()


def record(out, key, r):
    out[f"{key}_err"] = np.array([r["error_max"], r["error_l2"], r["mean_iterations"]])
    out[f"{key}_iters"] = np.array(r["solve_iterations"], np.int32)
    out[f"{key}_sub"] = sub(r["state"])
    s = r["state"]
    out[f"{key}_moments"] = np.array([s.sum(), np.dot(s, s), np.abs(s).max()])
    # bitwise fingerprint of the whole state (portable, unlike numpy sums)
    out[f"{key}_sha256"] = np.frombuffer(hashlib.sha256(np.ascontiguousarray(s).tobytes()).digest(), np.uint8)
    out[f"{key}_wall"] = np.array([r["wall_seconds"], R.max_threads()])


if __name__ == "__main__":
    R = Reference()
    R.set_threads(os.cpu_count() or 1)
    path = os.path.join(HERE, "configs.npz")
    only = sys.argv[1:]  # e.g. "m1_f32 m1_f64": recompute these keys, keep the rest
    out = dict(np.load(path)) if only and os.path.exists(path) else {"n": np.array([N, SUB])}
    runs = [
        ("m1_f32", "midpoint1", 0.01, 1e-3, "f32"),
        ("m1_f64", "midpoint1", 0.01, 1e-5, "f64"),
        ("c2_f32", "4s3pB", 0.1, 1e-3, "f32"),
        ("c2_f64", "4s3pB", 0.1, 1e-5, "f64"),
    ]
    for key, meth, t_end, tol, prec in runs:
        if only and key not in only:
            continue
        t0 = time.time()
        r = R.integrate(0, N, R.tableau(meth), 0.01, t_end, tol, prec, 40)
        record(out, key, r)
        print(f"{key}: err_max {r['error_max']:.6e} err_l2 {r['error_l2']:.6e} iters {r['solve_iterations']} "
              f"({time.time() - t0:.0f} s)", flush=True)
        np.savez_compressed(path, **out)
