"""Run one kernel_bench entry (for ncu captures).  Usage: kbench_loop.py name [n] [reps]"""
import ctypes as C
import sys

sys.path.insert(0, ".")
import paper_2412_16638_b200 as mp  # noqa: E402

name = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 256
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
ms, by = C.c_double(), C.c_double()
mp.check(mp._c.lib.mprkb_kernel_bench(name.encode(), n, reps, C.byref(ms), C.byref(by)))
print(name, ms.value * 1e3, "us")
