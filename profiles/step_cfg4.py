"""One config-4 step (advection-diffusion 256^3, 4s3pC, complex-fp32 GMRES +
FastDiag on the DFT basis, fp16 Krylov basis) for ncu launch lists."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2412_16638_b200 as mp  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
st = mp.Stepper("advection-diffusion", 256, mp.builtin("4s3pC"), 1.0 / 640.0, 1e-3, "f32", 40, nu=1e-2,
                basis_storage="f16")
u = torch.from_numpy(st.initial_state()).cuda()
for _ in range(steps):
    print(st.step_device(u)["iterations"])
torch.cuda.synchronize()
