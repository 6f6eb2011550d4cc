"""Small-size driver for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): the bench path (fused speculative fp32 pipeline, tcgen05
FastDiag) and its neighbours at n = 128, the fp64 DMMA path, block-Jacobi
pipelined CG with the device loop, accessor-storage CG, GMRES with the fp16
basis, and a 2-rank in-process split step.
Usage: compute-sanitizer --tool memcheck python profiles/sanitize.py"""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2412_16638_b200 as mp  # noqa: E402


def step(*args, steps=1, **kw):
    st = mp.Stepper(*args, **kw)
    u = st.initial_state()
    for _ in range(steps):
        tr = st.step(u)
    assert np.isfinite(u).all()
    return tr


n = 128
t = mp.builtin("4s3pB")
print("fp32 fused/speculative", step("heat", n, t, 0.01, 1e-3, "f32", steps=2)["iterations"])
print("fp32 forced miss", step("heat", n, t, 0.01, 1e-7, "f32", 12)["iterations"])
print("fp64 dmma", step("heat", n, t, 0.01, 1e-6, "f64")["iterations"])
print("block-jacobi devloop", step("heat", n, t, 0.01, 1e-5, "f32", 300, preconditioner="block-jacobi",
                                   block_size=8, block_storage="f16")["iterations"])
print("accessor f16", step("heat", 64, t, 0.01, 1e-2, "f32", 400, preconditioner="block-jacobi", block_size=8,
                           block_storage="f32", krylov_storage="f16")["iterations"])
print("advection gmres", step("advection", 32, mp.builtin("4s3pC"), 1.0 / 640.0, 1e-4, "f32")["iterations"])
print("parity", step("heat", 16, t, 0.01, 1e-5, "f32", numerics="parity")["iterations"])


def body(rank, comm):
    st = mp.Stepper("heat", n, t, 0.01, 1e-3, "f32", comm=comm)
    u = st.initial_state()
    return st.step(u)["iterations"]


print("split P=2", mp.run_ranks(2, body))
torch.cuda.synchronize()
print("ok")
