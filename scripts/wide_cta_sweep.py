"""Wide-integer walk: CTA size sweep on the Figure-1 shapes (pe_tuning.block
overrides the width-based choice). Prints one JSON line per (case, block)."""
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

cases = [(64, 64, 4096), (64, 256, 4096), (64, 1000, 4096), (2048, 64, 296), (2048, 256, 296)]
blocks = [int(b) for b in sys.argv[1].split(",")] if len(sys.argv) > 1 else [0, 32, 64, 128, 256]
for bits, degree, n in cases:
    exps, coefs, pts = W.fig1(degree, bits, bits, n)
    L = pe.limbs_for(pts)
    cols = [pe.ints_to_words(pts, L)]
    for scheme in ("balanced", "horner"):
        base = None
        for b in blocks:
            prog = pe.compile_wide(exps, coefs, pe.builtin_scheme(scheme))
            if b:
                prog.set_tuning(block=b)
            got = pe.evaluate_wide(prog, cols, as_words=True)
            if base is None:
                base = got
            best = 1e30
            for _ in range(3):
                torch.cuda.synchronize()
                t = time.perf_counter()
                pe.evaluate_wide(prog, cols, as_words=True)
                best = min(best, time.perf_counter() - t)
            print(json.dumps({"bits": bits, "degree": degree, "scheme": scheme, "block": b,
                              "points_per_s": n / best, "call_s": best,
                              "same_as_default": bool(np.array_equal(got, base))}), flush=True)
