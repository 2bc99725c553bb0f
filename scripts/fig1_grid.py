"""The paper's Figure-1 workload on the GPU (pe_eval_wide) next to the
unmodified reference BigInt walk (oracle/_ref): dense degree-d polynomials
with 64-bit (run_grid defaults, reference bench.hpp:22-23) or 2048-bit
(acceptance_test.cpp C09 staircase) coefficients and points, schemes
balanced / estrin / horner. Per case: GPU points/s over a batch — the whole
call with host words in and out (wall clock), and the walk alone with
device-resident buffers (CUDA events) — results checked word for word
against the reference, reference
points/s on 1 thread and on all host threads, and the estrin / balanced
time ratio — the paper's Figure-1 quantity — on both.

  python scripts/fig1_grid.py [--quick]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import ctypes as C  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1307_5655_b200 as pe  # noqa: E402
from paper_1307_5655_b200 import _lib as L_  # noqa: E402
from paper_1307_5655_b200 import workloads as W  # noqa: E402
import pyoracle  # noqa: E402

quick = "--quick" in sys.argv
threads = len(os.sched_getaffinity(0))
grid = [(64, d, 4096) for d in (16, 64, 128, 255, 256, 512, 1000)] + \
       [(2048, d, 296) for d in (64, 255, 256)]
if quick:
    grid = [(64, 64, 1024), (2048, 255, 148), (2048, 256, 148)]
rows = {}
for bits, degree, n in grid:
    exps, coefs, pts = W.fig1(degree, bits, bits, n)
    L = pe.limbs_for(pts)
    cols = [pe.ints_to_words(pts, L)]
    cw = pe.ints_to_words(coefs, pe.limbs_for(coefs))
    for scheme in ("balanced", "estrin", "horner"):
        sch = pe.builtin_scheme(scheme)
        prog = pe.compile_wide(exps, coefs, sch)
        k = pe.wide_limbs(prog, L)
        got = pe.evaluate_wide(prog, cols, as_words=True)  # warm-up + checked result
        ref = pyoracle.ReferenceWide(exps, cw, [sch])
        bad = ref.mismatches(cols, got, threads=threads)
        gpu_s = 1e30
        for _ in range(3):  # best of 3 (host staging + one launch + D2H per call)
            torch.cuda.synchronize()
            t = time.perf_counter()
            pe.evaluate_wide(prog, cols, as_words=True)
            gpu_s = min(gpu_s, time.perf_counter() - t)
        # the walk alone: device-resident words in and out, CUDA events
        dev_in = torch.from_numpy(cols[0].view(np.int64)).to("cuda:0")
        dev_out = torch.empty((n, k), dtype=torch.int64, device="cuda:0")
        ptrs = (C.c_void_p * 1)(dev_in.data_ptr())
        ex = L_.pe_exec()
        ex.device = -1
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        kern_ms = 1e30
        for _ in range(3):
            e0.record()
            L_.check(L_.lib().pe_eval_wide(prog.handle, ptrs, L, n, dev_out.data_ptr(), k, C.byref(ex)))
            e1.record()
            torch.cuda.synchronize()
            kern_ms = min(kern_ms, e0.elapsed_time(e1))
        assert np.array_equal(dev_out.cpu().numpy().view(np.uint64), got)
        m = min(n, 64 if bits == 64 else 8)
        sub = [c[:m] for c in cols]
        ref1 = m / ref.seconds(sub, threads=1)
        reft = min(n, 16 * threads) if bits == 64 else min(n, 2 * threads)
        refT = reft / ref.seconds([c[:reft] for c in cols], threads=threads)
        row = {"coeff_bits": bits, "point_bits": bits, "degree": degree, "scheme": scheme,
               "points": n, "result_limbs": k, "mismatches": bad,
               "gpu_points_per_s": n / gpu_s, "gpu_call_s": gpu_s,
               "gpu_kernel_points_per_s": n / (kern_ms * 1e-3), "gpu_kernel_ms": kern_ms,
               "ref_points_per_s_1thread": ref1, "ref_points_per_s_all": refT,
               "ref_threads": threads}
        rows[(bits, degree, scheme)] = row
        print(json.dumps(row), flush=True)
# Figure-1 quantity: scheme time / balanced time, GPU and reference (1 thread)
for (bits, degree, scheme), row in rows.items():
    b = rows.get((bits, degree, "balanced"))
    if b and scheme != "balanced":
        print(json.dumps({"ratio_vs_balanced": scheme, "bits": bits, "degree": degree,
                          "gpu": b["gpu_points_per_s"] / row["gpu_points_per_s"],
                          "reference": b["ref_points_per_s_1thread"] / row["ref_points_per_s_1thread"]}),
              flush=True)
