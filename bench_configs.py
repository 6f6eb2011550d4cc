#!/usr/bin/env python3
"""The other BASELINE.json configurations, measured on one B200 (bench.py
measures configs[1], the headline, and configs[2] under torchrun).

  --config 1  heat 32^3, midpoint1 (fp64 explicit / fp32 implicit), CG +
              FastDiag and CG + block-Jacobi, 10 steps; the reference's own
              CPU run of the same integrate() beside it (it runs in seconds).
  --config 2  the fp64-policy "baseline stepper" companion of configs[1]:
              heat 256^3 4s3pB with fp64 stages, tol 1e-5, next to the mixed
              fp32-stage step.
  --config 4  advection-diffusion 256^3, 4s3pC, GMRES stage solves with the
              fp16 Krylov basis (fp64-accumulated dots): FastDiag and
              block-Jacobi (multi-iteration) preconditioners.
  --config 5  solver-parameter sweep at 384^3: stage tol x block-Jacobi block
              size x block storage precision, one 4s3pB step each (bounded:
              --sweep-limit runs).

One JSON line per measurement: metric, value (DOF-updates/s), ms_per_step,
iterations, and what was run.  Device-resident state, CUDA-event timing on
the stepper's stream after warm-up steps.
"""
from __future__ import annotations

import argparse
import itertools
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def time_steps(mp, torch, st, steps, warmup):
    u = torch.from_numpy(st.initial_state()).cuda()
    s = torch.cuda.ExternalStream(st.stream)
    its = []
    for _ in range(warmup):
        st.step_device(u)
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(steps):
        its.append(st.step_device(u)["iterations"])
    b.record(s)
    b.synchronize()
    return a.elapsed_time(b) / steps, its


def line(**kw):
    print(json.dumps(kw), flush=True)


def config1(mp, torch):
    from oracle.oracle import Reference, ensure_built, have_reference

    n, tau, t_end = 32, 0.01, 0.1
    tab = mp.midpoint_corrected(1)
    for pre, tol in (("fastdiag", 1e-4), ("block-jacobi", 1e-4)):
        kw = dict(preconditioner=pre, block_size=8, block_storage="f32") if pre != "fastdiag" else {}
        t0 = time.perf_counter()
        r = mp.integrate(tab, "heat", n, tau, t_end, tol, "f32", 300 if pre != "fastdiag" else 40, **kw)
        wall = time.perf_counter() - t0
        ms, its = time_steps(mp, torch, mp.Stepper("heat", n, tab, tau, tol, "f32", 300, **kw), 50, 5)
        out = dict(config=1, workload=f"heat {n}^3 midpoint1 f32 stages, CG + {pre}, tau={tau}, t_end={t_end}, "
                                      f"tol={tol}", metric="DOF-updates/s", value=n ** 3 / (ms * 1e-3),
                   ms_per_step=ms, iterations_per_solve=sorted(set(i for x in its for i in x)),
                   error_max=r["error_max"], mean_iterations=r["mean_iterations"], integrate_wall_s=wall)
        if pre == "fastdiag":
            ensure_built(ref=True)
            if have_reference():
                R = Reference()
                R.set_threads(os.cpu_count() or 1)
                tabd = dict(q=tab.q, a_high=np.array(tab.a_high), a_eps=np.array(tab.a_eps), b=np.array(tab.b))
                rr = R.integrate(0, n, tabd, tau, t_end, tol, "f32")
                out["reference"] = dict(error_max=rr["error_max"], mean_iterations=rr["mean_iterations"],
                                        wall_s=rr["wall_seconds"], cores=os.cpu_count(),
                                        value=n ** 3 * rr["steps"] / rr["wall_seconds"])
        line(**out)


def config2(mp, torch):
    n, tau = 256, 0.01
    tab = mp.builtin("4s3pB")
    for prec, tol in (("f32", 1e-3), ("f64", 1e-5)):
        st = mp.Stepper("heat", n, tab, tau, tol, prec, 40)
        ms, its = time_steps(mp, torch, st, 20, 3)
        line(config=2, workload=f"heat {n}^3 4s3pB {prec} stages tol={tol}", metric="DOF-updates/s",
             value=n ** 3 / (ms * 1e-3), ms_per_step=ms, iterations_per_solve=sorted(set(i for x in its for i in x)))
        del st


def config4(mp, torch):
    n, tau, nu = 256, 1.0 / 640.0, 1e-2
    tab = mp.builtin("4s3pC")
    for pre, basis in (("fastdiag", "f16"), ("block-jacobi", "f16"), ("block-jacobi", None)):
        kw = dict(preconditioner=pre, block_size=8, block_storage="f16") if pre != "fastdiag" else {}
        st = mp.Stepper("advection-diffusion", n, tab, tau, 1e-3, "f32", 40, nu=nu, basis_storage=basis, **kw)
        ms, its = time_steps(mp, torch, st, 3, 2)  # (2 warm-up steps: the Krylov basis is allocated on first use)
        line(config=4, workload=(f"advection-diffusion {n}^3 nu={nu} 4s3pC, GMRES (complex fp32) + {pre}, "
                                 f"Krylov basis {basis or 'fp32 (working precision)'}, tau=1/640, tol=1e-3"),
             metric="DOF-updates/s", value=n ** 3 / (ms * 1e-3), ms_per_step=ms,
             iterations_per_solve=sorted(set(i for x in its for i in x)))
        del st


def config5(mp, torch, limit):
    n, tau = 384, 0.01
    tab = mp.builtin("4s3pB")
    # (module loading / first-launch setup outside the timed single steps)
    for store in ("f16", "f32", "f64"):
        w = mp.Stepper("heat", 128, tab, tau, 1e-4, "f32", 300, preconditioner="block-jacobi", block_size=4,
                       block_storage=store)
        time_steps(mp, torch, w, 1, 1)
        del w
    runs = list(itertools.product((1e-4, 1e-6, 1e-8, 1e-10), (4, 8, 16, 32), ("f16", "f32", "f64")))
    for tol, b, store in runs[:limit]:
        st = mp.Stepper("heat", n, tab, tau, tol, "f32", 300, preconditioner="block-jacobi", block_size=b,
                        block_storage=store)
        ms, its = time_steps(mp, torch, st, 1, 0)
        line(config=5, workload=f"heat {n}^3 4s3pB f32 stages, CG + block-Jacobi b={b} ({store}), tol={tol}",
             metric="DOF-updates/s", value=n ** 3 / (ms * 1e-3), ms_per_step=ms,
             iterations=its[0], ms_per_cg_iteration=ms / max(1, sum(its[0])))
        del st
    # accessor-style CG vectors (r, z, p, q in fp16; accessor.cu) beside the
    # working-precision vectors, b = 8 fp16 blocks, tol 1e-4
    for kst in (None, "f16"):
        st = mp.Stepper("heat", n, tab, tau, 1e-4, "f32", 300, preconditioner="block-jacobi", block_size=8,
                        block_storage="f16", krylov_storage=kst)
        ms, its = time_steps(mp, torch, st, 1, 1)
        line(config=5, workload=(f"heat {n}^3 4s3pB f32 stages, CG + block-Jacobi b=8 (f16), tol=1e-4, "
                                 f"CG vectors {kst or 'fp32 (working precision)'}"),
             metric="DOF-updates/s", value=n ** 3 / (ms * 1e-3), ms_per_step=ms, iterations=its[0],
             ms_per_cg_iteration=ms / max(1, sum(its[0])))
        del st


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, nargs="+", default=[1, 2, 4, 5])
    ap.add_argument("--sweep-limit", type=int, default=48)
    args = ap.parse_args()
    import torch

    torch.cuda.set_device(0)
    import paper_2412_16638_b200 as mp

    for c in args.config:
        {1: lambda: config1(mp, torch), 2: lambda: config2(mp, torch), 4: lambda: config4(mp, torch),
         5: lambda: config5(mp, torch, args.sweep_limit)}[c]()


if __name__ == "__main__":
    main()
