"""Steps heat 256^3 4s3pB with fp64 stages (the fp64 "baseline stepper" of
configs[1], tol 1e-5) — a short driver for an ncu launch list of its step.
Usage: python profiles/step_f64.py [steps]"""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2412_16638_b200 as mp  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
st = mp.Stepper("heat", 256, mp.builtin("4s3pB"), 0.01, 1e-5, "f64")
u = torch.from_numpy(mp.heat_exact(256, 0.05)).cuda()
for _ in range(steps):
    tr = st.step_device(u)
torch.cuda.synchronize()
print("ok", tr["iterations"])
