import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2412_16638_b200 as mp
n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
for eq, prec, nu in (("advection", "f32", 0.0), ("advection-diffusion", "f32", 1e-2), ("heat", "f64", 0.0)):
    tab = mp.builtin("4s3pC")
    tau = 1 / 640 if eq != "heat" else 0.01
    st = mp.Stepper(eq, n, tab, tau, 1e-3 if prec == "f32" else 1e-5, prec, 40, nu=nu, timings=True)
    u = torch.from_numpy(st.initial_state()).cuda()
    tr = st.step_device(u); torch.cuda.synchronize()
    t0 = time.time()
    for _ in range(3): tr = st.step_device(u)
    torch.cuda.synchronize()
    print(eq, prec, "ms/step", (time.time() - t0) / 3 * 1e3, tr["iterations"], flush=True)
    print({k: round(v["seconds_per_call"] * 1e3, 3) for k, v in st.timings().items()})
