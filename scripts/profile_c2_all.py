"""Evaluates the four C2 programs (d1000/d1023 x Estrin/balanced) in bench
order, `--reps` times, on one shared 1e7-point device batch — for ncu
captures of every C2 kernel (`-s 4 -c 4` skips the first, JIT-warm rep)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1307_5655_b200 as pe  # noqa: E402
from paper_1307_5655_b200 import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
wls = W.c2_all()
dev = torch.device("cuda:0")
x = [torch.from_numpy(v).to(dev) for v in wls[0].points()]
evs = [pe.Evaluator(pe.DoubleDomain(), pe.compile(w.poly, w.schemes)) for w in wls]
outs = [torch.empty_like(x[0]) for _ in wls]
for r in range(a.reps):
    for e, o in zip(evs, outs):
        e.evaluate(x, out=o)
    torch.cuda.synchronize()
print("programs:", ",".join(w.name for w in wls))
