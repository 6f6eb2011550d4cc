for d in 0 1 2 4 8 16 3 9 10 11 27 31; do
  echo -n "dbg=$d: "; MPRKB_TC_DBG=$d python -c "
import sys, ctypes as C
sys.path.insert(0, '.')
import paper_2412_16638_b200 as mp
out=[]
for k in ('tc_fold_R','tc_fold_M','tc_fold_L','tc_fold_Rpd'):
    ms, by = C.c_double(), C.c_double()
    mp.check(mp._c.lib.mprkb_kernel_bench(k.encode(), 256, 30, C.byref(ms), C.byref(by)))
    out.append('%s %.2f' % (k[8:], ms.value*1e3))
print(' | '.join(out))
"
done
