"""Throughput of the K-limb exact integer kernels (pe_eval_limbs) on the C3
program (bivariate total degree 40, |c| <= 8) at coordinate spans that need
K = 2 / 4 / 7 limbs, device buffers, CUDA events; beside it the unmodified
reference BigInt evaluator (oracle/_ref) on all host threads."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1307_5655_b200 as pe  # noqa: E402
from paper_1307_5655_b200 import workloads as W  # noqa: E402
import pyoracle  # noqa: E402

wl = W.c3()
prog = pe.compile(wl.poly, wl.schemes)
ev = pe.Evaluator(pe.BigIntDomain(), prog)
threads = len(os.sched_getaffinity(0))
for span in (4, 60, 1000):
    n = 4_000_000
    rng = np.random.default_rng(span)
    x = [torch.from_numpy(rng.integers(-span, span + 1, n).astype(np.int64)).cuda() for _ in range(2)]
    k, _ = ev.evaluate_limbs(x)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    a.record()
    for _ in range(reps):
        ev.evaluate_limbs(x, limbs=k)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    ref = pyoracle.Reference(wl.poly, wl.schemes)
    m = 20_000
    xs = [c[:m].cpu().numpy() for c in x]
    t = time.perf_counter()
    ref.eval_limbs(xs, k, threads)
    cpu = m / (time.perf_counter() - t)
    print(json.dumps({"span": span, "limbs": k, "points": n, "ms_per_call": round(ms, 3),
                      "gpu_points_per_s": n / (ms * 1e-3), "ref_bigint_points_per_s": cpu,
                      "ref_threads": threads,
                      "note": "ms includes the per-call max|x| reduction and proof"}), flush=True)
