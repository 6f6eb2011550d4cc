"""Time the folded tcgen05 FastDiag contraction per side under the
MPRKB_TC_DBG stage-removal knobs (results invalid when a knob is set; timing
only).  Usage: python profiles/tc_experiments.py [n] [dbg ...]"""
import os
import subprocess
import sys

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
dbgs = sys.argv[2:] or ["0", "1", "2", "4", "8", "16", "12", "31"]
code = r'''
import sys, ctypes as C
sys.path.insert(0, ".")
import paper_2412_16638_b200 as mp
out = []
for k in ("tc_fold_R", "tc_fold_M", "tc_fold_L", "tc_fold_Lpd"):
    ms, by = C.c_double(), C.c_double()
    mp.check(mp._c.lib.mprkb_kernel_bench(k.encode(), %d, 20, C.byref(ms), C.byref(by)))
    out.append("%%s %%.2f us %%.0f GB/s" %% (k, ms.value * 1e3, by.value / ms.value / 1e6))
print(" | ".join(out))
''' % n
for d in dbgs:
    env = dict(os.environ, MPRKB_TC_DBG=d)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    print(f"dbg={d:>3}:", r.stdout.strip() or r.stderr.strip()[-300:], flush=True)
