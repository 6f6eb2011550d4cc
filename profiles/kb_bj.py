import sys, ctypes as C
sys.path.insert(0, ".")
import paper_2412_16638_b200 as mp
out = []
for k in ("block_jacobi_f16", "cg_bj_f16"):
    ms, by = C.c_double(), C.c_double()
    mp.check(mp._c.lib.mprkb_kernel_bench(k.encode(), 256, 30, C.byref(ms), C.byref(by)))
    out.append("%s %.2f us (%.3f of 6534.5 GB/s)" % (k, ms.value * 1e3, by.value / (ms.value * 1e-3) / 1e9 / 6534.5))
print(" | ".join(out))
