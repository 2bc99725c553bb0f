"""Runs one config program a few times on device buffers (for ncu captures)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1307_5655_b200 as pe  # noqa: E402
from paper_1307_5655_b200 import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2e1000")
ap.add_argument("--points", type=int, default=10_000_000)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--strict", action="store_true")
a = ap.parse_args()
wl = {"c1": W.c1, "c2e1000": lambda: W.c2(1000, "estrin"), "c2b1000": lambda: W.c2(1000, "balanced"),
      "c2e1023": lambda: W.c2(1023, "estrin"), "c3": W.c3, "c4": W.c4, "c5": W.c5}[a.config]()
prog = pe.compile(wl.poly, wl.schemes)
dev = torch.device("cuda:0")
if wl.domain == "interval":
    lo, hi = wl.points(a.points)
    x = ([torch.from_numpy(v).to(dev) for v in lo], [torch.from_numpy(v).to(dev) for v in hi])
    ev = pe.Evaluator(pe.IntervalDomain(), prog, deferred_checks=True)
elif wl.domain == "i64":
    x = [torch.from_numpy(v).to(dev) for v in wl.points(a.points)]
    ev = pe.Evaluator(pe.BigIntDomain(), prog, deferred_checks=True)
else:
    x = [torch.from_numpy(v).to(dev) for v in wl.points(a.points)]
    ev = pe.Evaluator(pe.DoubleDomain(strict=a.strict), prog)
start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for r in range(a.reps):
    start.record()
    out = ev.evaluate(x)
    end.record()
    torch.cuda.synchronize()
    if ev.deferred_checks:
        ev.synchronize()
    print(f"{wl.name} rep {r}: {start.elapsed_time(end):.3f} ms")
