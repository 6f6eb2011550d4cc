"""Time the folded contraction (R, M, L, L with the diagonal) for every
variant library built by profiles/tc_variants.sh.  Usage: python
profiles/tc_variants.py [n] [reps]"""
import glob
import os
import subprocess
import sys

n = sys.argv[1] if len(sys.argv) > 1 else "256"
reps = sys.argv[2] if len(sys.argv) > 2 else "30"
code = r'''
import sys, ctypes as C
sys.path.insert(0, ".")
import paper_2412_16638_b200 as mp
out = []
for k in ("tc_fold_R", "tc_fold_M", "tc_fold_L", "tc_fold_Lpd", "tc_fold_Rpd"):
    try:
        ms, by = C.c_double(), C.c_double()
        mp.check(mp._c.lib.mprkb_kernel_bench(k.encode(), %s, %s, C.byref(ms), C.byref(by)))
        out.append("%%s %%.2f" %% (k[8:], ms.value * 1e3))
    except Exception as e:
        out.append("%%s ERR %%s" %% (k, str(e)[:60]))
print(" | ".join(out))
''' % (n, reps)
libs = [("base", "paper_2412_16638_b200/libmprk_b200.so")]
libs += [(os.path.basename(os.path.dirname(p)), p) for p in sorted(glob.glob("profiles/_variants/*/libmprk_b200.so"))]
for name, lib in libs:
    env = dict(os.environ, MPRKB_LIB=os.path.abspath(lib))
    flags = open(os.path.join(os.path.dirname(lib), "flags.txt")).read().strip() if name != "base" else ""
    for rep in range(2):
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
        print(f"{name:10s} {r.stdout.strip() or r.stderr.strip()[-300:]}   [{flags}]", flush=True)
