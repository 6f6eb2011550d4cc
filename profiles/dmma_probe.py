"""fp64 DMMA FastDiag contraction per side at 256^3 (kbench tensor_f64_{R,M,L})
for the in-tree library and every profiles/_variants/*/ library."""
import glob
import os
import subprocess
import sys

code = r'''
import sys, ctypes as C
sys.path.insert(0, ".")
import paper_2412_16638_b200 as mp
out = []
for sd in "RML":
    ms, by = C.c_double(), C.c_double()
    mp.check(mp._c.lib.mprkb_kernel_bench(("tensor_f64_" + sd).encode(), 256, 20, C.byref(ms), C.byref(by)))
    out.append("%s %.1f" % (sd, ms.value * 1e3))
print(" | ".join(out))
'''
libs = [("base", "paper_2412_16638_b200/libmprk_b200.so")]
libs += [(os.path.basename(os.path.dirname(p)), p) for p in sorted(glob.glob("profiles/_variants/*/libmprk_b200.so"))]
for name, lib in libs:
    env = dict(os.environ, MPRKB_LIB=os.path.abspath(lib))
    for rep in range(2):
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
        print(f"{name:10s} {r.stdout.strip() or r.stderr.strip()[-300:]}", flush=True)
