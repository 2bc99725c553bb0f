"""Experiment: does splitting a wide program into K slices by the outer
variable's exponent (K kernels, partial sums) beat one huge kernel?"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1307_5655_b200 as pe
from paper_1307_5655_b200 import workloads as W

wl = W.c4()
n = 4_000_000
dev = torch.device("cuda:0")
x = [torch.from_numpy(a).to(dev) for a in wl.points(n)]
e, c = wl.poly.exponents, wl.poly.coefficients
for K in [int(k) for k in sys.argv[1:]] or [1, 2, 4, 8, 16]:
    order = np.argsort(e[:, 0], kind="stable")
    groups = np.array_split(order, K)
    progs = [pe.compile(pe.Polynomial(e[g], c[g], ("x", "y", "z")), wl.schemes) for g in groups]
    outs = [torch.empty(n, dtype=torch.float64, device=dev) for _ in progs]
    evs = [pe.Evaluator(pe.DoubleDomain(), p) for p in progs]
    for ev, o in zip(evs, outs):
        ev.evaluate(x, out=o)
    torch.cuda.synchronize()
    s, t = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for rep in range(3):
        s.record()
        for ev, o in zip(evs, outs):
            ev.evaluate(x, out=o)
        t.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(t))
    print(f"K={K}: {best:.3f} ms for {n} points ({n / best * 1e3:.3e} pts/s)", flush=True)
