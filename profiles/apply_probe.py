"""FastDiag apply (6 folded tcgen05 contractions) timed three ways on a 256^3
grid: CUDA events around 20 applies (bench.py's roofline measure), host
enqueue time of the same loop (is the stream host-bound?), and the six
sides alone through kbench.  Usage: python profiles/apply_probe.py"""
import ctypes as C
import sys
import time

sys.path.insert(0, ".")
import torch

import paper_2412_16638_b200 as mp

n, reps = 256, 20
P = mp.Operator.fastdiag_stage(0, "heat", n, 0.01, 0.5, "fast")
x = torch.randn(n ** 3, dtype=torch.float32, device="cuda")
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for _ in range(3):
        P.apply(x)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    t0 = time.perf_counter()
    for _ in range(reps):
        P.apply(x)
    t_host = (time.perf_counter() - t0) / reps
    b.record(s)
    b.synchronize()
print(f"apply: {a.elapsed_time(b) / reps * 1e3:.1f} us per apply ({a.elapsed_time(b) / reps / 6 * 1e3:.2f} per contraction),"
      f" host enqueue {t_host * 1e6:.1f} us per apply")
tot = 0.0
for k in ("tc_fold_L", "tc_fold_M", "tc_fold_R", "tc_fold_Rpd", "tc_fold_M", "tc_fold_L"):
    ms, by = C.c_double(), C.c_double()
    mp.check(mp._c.lib.mprkb_kernel_bench(k.encode(), n, 30, C.byref(ms), C.byref(by)))
    tot += ms.value * 1e3
    print(f"  {k:12s} {ms.value * 1e3:.2f} us")
print(f"kbench sum {tot:.1f} us per apply-equivalent ({tot / 6:.2f} per contraction)")
