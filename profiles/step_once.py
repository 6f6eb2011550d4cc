"""Steps the bench workload (heat 256^3 4s3pB, fp32 stages, device-resident
state) a few times — a short driver for ncu launch lists of one step.
Usage: python profiles/step_once.py [steps] [n]"""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2412_16638_b200 as mp  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
n = int(sys.argv[2]) if len(sys.argv) > 2 else 256
st = mp.Stepper("heat", n, mp.builtin("4s3pB"), 0.01, 1e-3, "f32")
u = torch.from_numpy(mp.heat_exact(n, 0.05)).cuda()
for _ in range(steps):
    st.step_device(u)
torch.cuda.synchronize()
print("ok", float(u.abs().max()))
