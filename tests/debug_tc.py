"""Ad-hoc GPU check of the tcgen05 contraction per side (not collected by pytest)."""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2412_16638_b200 as mp  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128


def run(side, q, x):
    xd = torch.from_numpy(x).cuda()
    out = torch.zeros_like(xd)
    qq = np.ascontiguousarray(q, dtype=np.float32)
    mp.check(mp._c.lib.mprkb_tensor_apply_tc(side, n, qq.ctypes.data_as(C.c_void_p), C.c_void_p(xd.data_ptr()),
                                             C.c_void_p(out.data_ptr()), None))
    return out.cpu().numpy()


def ref(side, q, x):
    X = x.reshape(n, n, n).astype(np.float64)  # [k][j][i]
    Q = q.astype(np.float64)
    if side == 2:
        return np.einsum("aq,kjq->kja", Q, X).ravel()
    if side == 1:
        return np.einsum("aq,kqi->kai", Q, X).ravel()
    return np.einsum("aq,qji->aji", Q, X).ravel()


import os  # noqa: E402

print("MN variant", os.environ.get("MPRKB_TC_MN_VARIANT", "0"))
rng = np.random.default_rng(1)
x = rng.uniform(-1, 1, n ** 3).astype(np.float32)
for name, q in (("identity", np.eye(n, dtype=np.float32)), ("random", rng.uniform(-1, 1, (n, n)).astype(np.float32)),
                ("e01", np.eye(n, k=1, dtype=np.float32))):
    for side in (2, 1, 0):
        got = run(side, q, x)
        want = ref(side, q, x)
        err = np.abs(got - want).max() / max(np.abs(want).max(), 1e-30)
        print(f"{name:9s} side {side}: rel err {err:.3e}  |got| {np.abs(got).max():.3e}")
        if err > 1e-5 and name != "random":
            G = got.reshape(n, n, n)
            W = want.reshape(n, n, n)
            bad = np.argwhere(np.abs(G - W) > 1e-5)
            print("   first bad", bad[:5].tolist(), "got", [G[tuple(b)] for b in bad[:5]], "want",
                  [W[tuple(b)] for b in bad[:5]])
            # where does got's value come from?  find x index with same value for identity
            if name == "identity":
                for b in bad[:3]:
                    v = G[tuple(b)]
                    idx = np.argwhere(np.abs(x.reshape(n, n, n) - v) < 1e-7)
                    print("   value", v, "found at x", idx[:3].tolist())
