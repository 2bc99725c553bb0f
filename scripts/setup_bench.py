"""Setup (compile-time) cost at scale — SURVEY §8f row 1 (reference
`--report-setup`, bench.hpp:39-41).

For growing term counts: host front-end (canonicalize + build + lazy heights
+ compile) of this repo vs the unmodified reference (`oracle/_ref`), then the
lowering + PTX emission and the ptxas time of the specialised kernel(s) with
an empty cubin cache. Prints one JSON line per case."""
import json
import os
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
os.environ["PE_CACHE_DIR"] = tempfile.mkdtemp(prefix="pe_setup_cache_")

import numpy as np  # noqa: E402

import paper_1307_5655_b200 as pe  # noqa: E402
import pyoracle  # noqa: E402


def case(name, poly, schemes):
    t = time.perf_counter()
    prog = pe.compile(poly, schemes)
    front = time.perf_counter() - t
    ref = None
    if pyoracle.ref_available():
        t = time.perf_counter()
        pyoracle.Reference(poly, schemes)
        ref = time.perf_counter() - t
    t = time.perf_counter()
    st = prog.kernel_stats(pe.DOMAIN_F64)
    lower = time.perf_counter() - t
    t = time.perf_counter()
    slices = prog.f64_slices()
    if slices == 1:
        prog.compile_only(pe.DOMAIN_F64)
    else:  # the sliced kernels are what pe_eval_f64 compiles
        import torch
        if torch.cuda.is_available():
            pe.Evaluator(pe.DoubleDomain(), prog).evaluate(
                [np.zeros(1) for _ in range(poly.nvars)])
        else:
            prog.compile_only(pe.DOMAIN_F64)
    ptxas = time.perf_counter() - t
    print(json.dumps({"case": name, "terms": int(poly.coefficients.shape[0]),
                      "records": prog.info()["records"], "front_end_s": round(front, 4),
                      "reference_build_compile_s": None if ref is None else round(ref, 4),
                      "lower_and_ptx_emit_s": round(lower, 4), "ptxas_and_load_s": round(ptxas, 3),
                      "slices": slices, "ptx_bytes": st["ptx_bytes"]}), flush=True)


rng = np.random.default_rng(7)
for d in (1_000, 10_000):
    p = pe.Polynomial(np.arange(d, -1, -1).reshape(-1, 1), rng.uniform(-1, 1, d + 1))
    case(f"dense_univariate_d{d}_balanced", p, [pe.builtin_scheme("balanced")])
for t in (1_000, 10_000, 100_000):
    ex = np.unique(rng.integers(0, 101, size=(int(t * 1.05), 3)), axis=0)[:t].astype(np.uint32)
    p = pe.Polynomial(ex, rng.normal(size=len(ex)), ("x", "y", "z"))
    case(f"sparse_trivariate_{t}", p, [pe.builtin_scheme("balanced")] * 3)
