"""Split-grid overhead on ONE GPU: heat n^3 4s3pB fp32 stages stepped by P
in-process ranks (LocalComm: every multi-rank code path, device copies for
transport) vs the undivided stepper.  All P ranks share the GPU, so the
wall time of one global step (device-resident slabs, barrier-synchronised)
against the undivided step is the split path's overhead.
Usage: python profiles/split_local.py [n] [steps] [P ...]"""
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2412_16638_b200 as mp  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
Ps = [int(p) for p in sys.argv[3:]] or [1, 2, 4, 8]
tab = mp.builtin("4s3pB")
out = {"n": n, "steps": steps}


def timed(step_fn, warm=2):
    for _ in range(warm):
        step_fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        step_fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / steps * 1e3


st = mp.Stepper("heat", n, tab, 0.01, 1e-3, "f32")
u = torch.from_numpy(st.initial_state()).cuda()
out["undivided_ms"] = timed(lambda: st.step_device(u))
del st
for P in Ps:
    def body(rank, comm):
        s = mp.Stepper("heat", n, tab, 0.01, 1e-3, "f32", comm=comm)
        v = torch.from_numpy(s.initial_state()).cuda()
        ms = timed(lambda: s.step_device(v))
        return ms
    res = mp.run_ranks(P, body)
    out[f"P{P}_ms"] = max(res)
    out[f"P{P}_over_undivided"] = max(res) / out["undivided_ms"]
print(json.dumps(out))
