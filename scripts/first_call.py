"""Time to first result on a fresh program (no cubin cache): compile + first
evaluate (walk VM, the library default) vs waiting for the specialised
kernel (ptxas), and the unmodified reference's own setup (build + compile,
reference bench.hpp:39-41 setup_ns) for the same polynomial. Also the VM's
and the kernel's throughput at the config's size. One JSON line per config.

  PE_CACHE_DIR=off python scripts/first_call.py [c1 c2e c2b c3 c4 c5]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
os.environ.setdefault("PE_CACHE_DIR", "off")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1307_5655_b200 as pe  # noqa: E402
from paper_1307_5655_b200 import workloads as W  # noqa: E402
import pyoracle  # noqa: E402

CFG = {"c1": W.c1, "c2e": lambda: W.c2(1000, "estrin"), "c2b": lambda: W.c2(1000, "balanced"),
       "c3": W.c3, "c4": W.c4, "c5": W.c5}
dev = torch.device("cuda:0")


def sync_time(fn):
    torch.cuda.synchronize()
    t = time.perf_counter()
    out = fn()
    torch.cuda.synchronize()
    return time.perf_counter() - t, out


def run(name):
    wl = CFG[name]()
    n = min(wl.n_points, 10_000_000)
    if wl.domain == "interval":
        lo, hi = wl.points(n)
        x = ([torch.from_numpy(a).to(dev) for a in lo], [torch.from_numpy(a).to(dev) for a in hi])
        dom, dc = pe.IntervalDomain(), pe.DOMAIN_INTERVAL
    elif wl.domain == "i64":
        x = [torch.from_numpy(a).to(dev) for a in wl.points(n)]
        dom, dc = pe.BigIntDomain(), pe.DOMAIN_I64F
    else:
        x = [torch.from_numpy(a).to(dev) for a in wl.points(n)]
        dom, dc = pe.DoubleDomain(), pe.DOMAIN_F64
    t0 = time.perf_counter()
    prog = pe.compile(wl.poly, wl.schemes)
    t_front = time.perf_counter() - t0
    ev = pe.Evaluator(dom, prog)
    t_first, _ = sync_time(lambda: ev.evaluate(x))
    t_first += t_front
    t_vm, _ = sync_time(lambda: ev.evaluate(x)) if not prog.kernel_ready(dc) else (None, None)
    t1 = time.perf_counter()
    prog.compile_only(dc)
    t_jit_wait = time.perf_counter() - t1
    ev.evaluate(x)
    t_kernel, _ = sync_time(lambda: ev.evaluate(x))
    # the JIT-only path (what a first call cost before the VM)
    t2 = time.perf_counter()
    p2 = pe.compile(wl.poly, wl.schemes)
    p2.set_tuning(jit_mode=1, sched_window=0)
    p2.compile_only(dc)
    t_jit = time.perf_counter() - t2
    t3 = time.perf_counter()
    pyoracle.Reference(wl.poly, wl.schemes)
    t_ref = time.perf_counter() - t3
    print(json.dumps({"config": name, "points": n, "front_end_s": t_front,
                      "first_result_s": t_first, "vm_call_s": t_vm, "kernel_call_s": t_kernel,
                      "jit_compile_s": t_jit, "jit_left_after_first_call_s": t_jit_wait,
                      "reference_setup_s": t_ref}), flush=True)


for c in sys.argv[1:] or list(CFG):
    run(c)
