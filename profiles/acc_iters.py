"""A few accessor-storage (fp16 vectors) block-Jacobi CG solves at 384^3 — a
short driver for ncu launch lists.  Usage: python profiles/acc_iters.py [n]"""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2412_16638_b200 as mp  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 384
tau, a = 0.01, 0.5
h = 1.0 / (n - 1)
sigma, gamma = 1.0, -tau * a * (-1.0 / h ** 2)
b = torch.from_numpy(np.random.default_rng(3).uniform(-1, 1, n ** 3).astype(np.float32)).cuda()
A = mp.Operator.stencil(0, n, 0, sigma, gamma)
P = mp.Operator.block_jacobi(0, "heat", n, tau, a, 8, "f16")
for _ in range(2):
    x, r = mp.cg(A, P, b, torch.zeros_like(b), 1e-2, 12, storage="f16")
torch.cuda.synchronize()
print("iterations", r["iterations"])
