import sys, ctypes as C
sys.path.insert(0, ".")
import paper_2412_16638_b200 as mp
for k in sys.argv[1:]:
    ms, by = C.c_double(), C.c_double()
    mp.check(mp._c.lib.mprkb_kernel_bench(k.encode(), 256, 2, C.byref(ms), C.byref(by)))
    print(k, ms.value, by.value / ms.value / 1e6)
