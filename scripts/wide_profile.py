"""Target process for ncu captures of the wide-integer walk (pe_eval_wide):
  python scripts/wide_profile.py <bits> <degree> <points> <scheme> [tuning]
Device-resident inputs and outputs; prints points/s (CUDA events)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import ctypes as C  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1307_5655_b200 as pe  # noqa: E402
from paper_1307_5655_b200 import _lib as L_  # noqa: E402
from paper_1307_5655_b200 import workloads as W  # noqa: E402

bits, degree, n = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
scheme = sys.argv[4] if len(sys.argv) > 4 else "balanced"
exps, coefs, pts = W.fig1(degree, bits, bits, n)
L = pe.limbs_for(pts)
prog = pe.compile_wide(exps, coefs, pe.builtin_scheme(scheme))
if len(sys.argv) > 5:  # pe_tuning fields, e.g. block=32,min_ctas=8
    prog.set_tuning(**{k: int(v) for k, v in (kv.split("=") for kv in sys.argv[5].split(","))})
k = pe.wide_limbs(prog, L)
dev = torch.device("cuda:0")
words = torch.from_numpy(pe.ints_to_words(pts, L).view(np.int64)).to(dev)
out = torch.empty((n, k), dtype=torch.int64, device=dev)
ptrs = (C.c_void_p * 1)(words.data_ptr())
ex = L_.pe_exec()
ex.device = -1
ex.synchronize = 0


def call():
    L_.check(L_.lib().pe_eval_wide(prog.handle, ptrs, L, n, out.data_ptr(), k, C.byref(ex)))


call()
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
best = 1e30
for _ in range(3):
    s.record()
    call()
    e.record()
    torch.cuda.synchronize()
    best = min(best, s.elapsed_time(e))
print(json.dumps({"bits": bits, "degree": degree, "points": n, "scheme": scheme, "result_limbs": k,
                  "tuning": sys.argv[5] if len(sys.argv) > 5 else "",
                  "ms": best, "points_per_s": n / (best * 1e-3)}))
