"""Steps config 4 with block-Jacobi stage preconditioners (advection-diffusion
256^3 4s3pC, complex fp32 GMRES, fp16 Krylov basis) once — a short driver
for an ncu launch list.  Usage: python profiles/step_cfg4_bj.py"""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2412_16638_b200 as mp  # noqa: E402

st = mp.Stepper("advection-diffusion", 256, mp.builtin("4s3pC"), 1.0 / 640.0, 1e-3, "f32", 40, nu=1e-2,
                preconditioner="block-jacobi", block_size=8, basis_storage="f16")
u = torch.from_numpy(st.initial_state()).cuda()
tr = st.step_device(u)
torch.cuda.synchronize()
print("ok", tr["iterations"])
