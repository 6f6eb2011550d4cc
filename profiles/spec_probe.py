"""Host-side view of one bench step with and without speculative stage
solves: wall time per step_device() and the histories it reports."""
import os
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2412_16638_b200 as mp  # noqa: E402

st = mp.Stepper("heat", 256, mp.builtin("4s3pB"), 0.01, 1e-3, "f32")
u = torch.from_numpy(st.initial_state()).cuda()
for _ in range(3):
    st.step_device(u)
torch.cuda.synchronize()
ts = []
for _ in range(20):
    t0 = time.perf_counter()
    tr = st.step_device(u)
    ts.append(time.perf_counter() - t0)
print(os.environ.get("MPRKB_SPECULATE", "1"), "host ms/step", round(1e3 * sum(ts) / len(ts), 4),
      "min", round(1e3 * min(ts), 4), tr["iterations"], [list(st.history(i)) for i in range(4)][0])
