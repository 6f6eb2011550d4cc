"""Ad-hoc GPU check of each FAST component across sizes (not collected by pytest)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2412_16638_b200 as mp  # noqa: E402
from oracle.oracle import Reference  # noqa: E402

R = Reference()
for n in [int(a) for a in sys.argv[1:]] or [128, 256]:
    rng = np.random.default_rng(n)
    for kind, dt in ((0, np.float32), (1, np.float64)):
        x = rng.uniform(-1, 1, n ** 3).astype(dt)
        xd = torch.from_numpy(x).cuda()
        got = mp.stencil_apply(xd, n, 0, 1.0, -0.37).cpu().numpy()
        want = R.stencil(kind, n, 0, 1.0, -0.37, x)
        print(n, kind, "stencil bitwise", np.array_equal(got, want), np.abs(got - want).max())
        for side in range(3):
            q = rng.uniform(-1, 1, n * n).astype(dt)
            qd = torch.from_numpy(q).cuda()
            a = mp.tensor_apply(side, n, qd, xd, "parity").cpu().numpy()
            b = mp.tensor_apply(side, n, qd, xd, "fast").cpu().numpy()
            print(n, kind, "tensor side", side, "fast-vs-parity", np.abs(a - b).max(), np.isfinite(b).all())
        P = mp.Operator.fastdiag_stage(kind, "heat", n, 0.01, 0.5, "parity")
        F = mp.Operator.fastdiag_stage(kind, "heat", n, 0.01, 0.5, "fast")
        a = P.apply(xd).cpu().numpy()
        b = F.apply(xd).cpu().numpy()
        print(n, kind, "fastdiag fast-vs-parity", np.abs(a - b).max() / np.abs(a).max(), np.isfinite(b).all())
    for prec in ("f32", "f64"):
        st = mp.Stepper("heat", n, mp.midpoint_corrected(1), 0.01, 1e-3, prec)
        u = st.initial_state()
        try:
            tr = st.step(u)
            print(n, prec, "step ok", tr["iterations"], np.abs(u).max())
        except Exception as e:  # noqa: BLE001
            print(n, prec, "step FAILED", type(e).__name__, e)
