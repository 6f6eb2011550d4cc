"""Per-label device times of the bench step (CUDA-event brackets,
record_timings): tensor-r/m/l (the FastDiag contractions), diag, stencil,
precond, solver, axpy — next to the same contractions timed alone
(kernel_bench tc_fold_*).  Usage: python profiles/step_timings.py [steps]"""
import ctypes as C
import json
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2412_16638_b200 as mp  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
n = 256
st = mp.Stepper("heat", n, mp.builtin("4s3pB"), 0.01, 1e-3, "f32", timings=True)
u = torch.from_numpy(mp.heat_exact(n, 0.05)).cuda()
for _ in range(3):
    st.step_device(u)
st2 = mp.Stepper("heat", n, mp.builtin("4s3pB"), 0.01, 1e-3, "f32", timings=True)
for _ in range(steps):
    st2.step_device(u)
torch.cuda.synchronize()
out = {"in_step": {k: {"calls_per_step": v["count"] / steps, "us_per_call": 1e6 * v["seconds_per_call"],
                       "us_per_step": 1e6 * v["total_seconds"] / steps} for k, v in st2.timings().items()}}
alone = {}
for name in ("tc_fold_R", "tc_fold_M", "tc_fold_L", "tc_fold_Lpd"):
    ms, by = C.c_double(), C.c_double()
    mp.check(mp._c.lib.mprkb_kernel_bench(name.encode(), n, 200, C.byref(ms), C.byref(by)))
    alone[name] = ms.value * 1e3
out["alone_us"] = alone
print(json.dumps(out, indent=1))
