"""A few block-Jacobi (b = 32, fp16 blocks) fp32 CG iterations at 384^3 — a
short driver for ncu captures of the chunked fused update
(k_cg_update_bj_tile).  Usage: python profiles/bj32_iters.py"""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2412_16638_b200 as mp  # noqa: E402

n, tau, a = 384, 0.01, 0.5
h = 1.0 / (n - 1)
A = mp.Operator.stencil(0, n, 0, 1.0, -tau * a * (-1.0 / h ** 2))
P = mp.Operator.block_jacobi(0, "heat", n, tau, a, 32, "f16")
b = torch.from_numpy(np.random.default_rng(3).uniform(-1, 1, n ** 3).astype(np.float32)).cuda()
x, r = mp.cg(A, P, b, torch.zeros_like(b), 1e-2, 12)
torch.cuda.synchronize()
print("iterations", r["iterations"])
