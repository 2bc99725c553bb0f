"""Probe: C4 as K separate kernels over x-exponent ranges of the terms
(sub-polynomials with their own trees, summed on the device) vs the one
sectioned kernel of the reference tree. Prints ms per evaluate of 4e6 points."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1307_5655_b200 as pe  # noqa: E402
from paper_1307_5655_b200 import workloads as W  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4_000_000
wl = W.c4()
dev = torch.device("cuda:0")
x = [torch.from_numpy(v).to(dev) for v in wl.points(n)]
e, c = wl.poly.exponents, wl.poly.coefficients
xs = np.unique(e[:, 0])


def timed(fn, reps=3):
    s, t = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        s.record()
        fn()
        t.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(t))
    return best


for K in ([int(k) for k in sys.argv[2].split(",")] if len(sys.argv) > 2 else (1, 2, 4, 6, 8)):
    evs = []
    for q in range(K):
        lo = xs[len(xs) * q // K]
        hi = xs[len(xs) * (q + 1) // K] if q + 1 < K else 10**9
        sel = (e[:, 0] >= lo) & (e[:, 0] < hi)
        p = pe.compile(pe.Polynomial(e[sel], c[sel]), wl.schemes)
        p.set_tuning(section_ops=2**32 - 1, jit_mode=1)
        evs.append(pe.Evaluator(pe.DoubleDomain(), p))
    outs = [torch.empty(n, dtype=torch.float64, device=dev) for _ in evs]

    def run():
        for ev, o in zip(evs, outs):
            ev.evaluate(x, out=o)
    print(json.dumps({"split_kernels": K, "ms": round(timed(run), 4)}), flush=True)
