import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["PE_IV_DEBUG"] = "1"
import numpy as np
import paper_1307_5655_b200 as pe
from paper_1307_5655_b200 import workloads as W
wl = W.c5()
prog = pe.compile(wl.poly, wl.schemes)
lo, hi = wl.points(4096)
olo, ohi = pe.Evaluator(pe.IntervalDomain(), prog).evaluate((lo, hi))
acc = ohi.view(np.uint64)
print("slow fraction", np.mean(acc >> np.uint64(63)))
for i in range(5):
    print(hex(int(acc[i])), lo[0][i])
slow = np.nonzero(acc >> np.uint64(63))[0]
print("slow idx", slow[:20])
print("slow x", lo[0][slow[:20]])
