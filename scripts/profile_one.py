"""Runs one config's program on device buffers: timing sweeps over
code-generation options, and the target process of ncu captures.

  python scripts/profile_one.py --config c4 --points 4000000 --reps 3 \
      --tune section_ops=2000 --tune section_ops=3000,group_tiles=4

Each --tune (comma-separated pe_tuning fields) compiles the program afresh
and prints one JSON line {config, tune, ms (best of reps), points/s, sections}.
Timing: CUDA events on torch's current stream around one evaluate call.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1307_5655_b200 as pe  # noqa: E402
from paper_1307_5655_b200 import workloads as W  # noqa: E402

CONFIGS = {"c1": W.c1, "c2e1000": lambda: W.c2(1000, "estrin"),
           "c2b1000": lambda: W.c2(1000, "balanced"), "c2e1023": lambda: W.c2(1023, "estrin"),
           "c2b1023": lambda: W.c2(1023, "balanced"), "c3": W.c3, "c4": W.c4, "c5": W.c5}

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2e1000", choices=sorted(CONFIGS))
ap.add_argument("--points", type=int, default=10_000_000)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--strict", action="store_true")
ap.add_argument("--tune", action="append", default=[])
a = ap.parse_args()
wl = CONFIGS[a.config]()
dev = torch.device("cuda:0")
if wl.domain == "interval":
    lo, hi = wl.points(a.points)
    x = ([torch.from_numpy(v).to(dev) for v in lo], [torch.from_numpy(v).to(dev) for v in hi])
else:
    x = [torch.from_numpy(v).to(dev) for v in wl.points(a.points)]


def parse_tune(text):
    out = {}
    for kv in filter(None, text.split(",")):
        k, v = kv.split("=")
        out[k.strip()] = int(v)
    return out


for tune in a.tune or [""]:
    opts = parse_tune(tune)
    prog = pe.compile(wl.poly, wl.schemes)
    if opts:
        prog.set_tuning(**opts)
    if wl.domain == "interval":
        ev = pe.Evaluator(pe.IntervalDomain(), prog, deferred_checks=True)
    elif wl.domain == "i64":
        ev = pe.Evaluator(pe.BigIntDomain(), prog, deferred_checks=True)
    else:
        ev = pe.Evaluator(pe.DoubleDomain(strict=a.strict), prog)
    # wait for the specialised kernel (a new program's first calls would
    # otherwise run the walk VM while it compiles)
    for dc in {"f64": [pe.DOMAIN_F64_STRICT if a.strict else pe.DOMAIN_F64],
               "interval": [pe.DOMAIN_INTERVAL], "i64": [pe.DOMAIN_I64F, pe.DOMAIN_I64]}[wl.domain]:
        prog.compile_only(dc)
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = None
    for r in range(a.reps + 1):  # first call: JIT + load
        start.record()
        ev.evaluate(x)
        end.record()
        torch.cuda.synchronize()
        if ev.deferred_checks:
            ev.synchronize()
        if r:
            ms = start.elapsed_time(end)
            best = ms if best is None else min(best, ms)
    print(json.dumps({"config": a.config, "tune": opts, "points": a.points, "ms": round(best, 4),
                      "points_per_s": a.points / (best * 1e-3),
                      "sections": prog.f64_slices() if wl.domain == "f64" else None}), flush=True)
