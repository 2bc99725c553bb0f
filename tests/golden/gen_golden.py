"""Regenerates the committed golden fixtures from the UNMODIFIED reference.

Run in the build container (where /root/reference exists and `make -C oracle
ref` produced oracle/_ref/libpolyeval_ref.so):

    python tests/golden/gen_golden.py

Outputs (committed):
  ref_dot_{direct,horner,estrin,balanced}.dot   to_dot() of the worked example
      3x^8-x^7+2x^6+x^5-4x^4+9x^3-3x^2-2x+1 (reference tree.cpp:290-309)
  wide_int64_interval.npz   interval walk with int64 coefficients
      above 2^53 (from_integer's one-ulp widening, numeric.cpp:17-26), 4 schemes
  vectors_<config>.npz   inputs + reference outputs for each BASELINE config
      shape at 512 points (Evaluator<ScaledDoubleDomain / BigIntDomain /
      ScaledIntervalDomain> through ref_harness.cpp), bit patterns preserved.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]

import paper_1307_5655_b200 as pe  # noqa: E402
from paper_1307_5655_b200 import workloads as W  # noqa: E402
import pyoracle  # noqa: E402

N = 512


def main():
    e = np.array([8, 7, 6, 5, 4, 3, 2, 1, 0]).reshape(-1, 1)
    c = np.array([3, -1, 2, 1, -4, 9, -3, -2, 1], dtype=np.int64)
    p = pe.Polynomial(e, c)
    for s in ("direct", "horner", "estrin", "balanced"):
        dot = pyoracle.Reference(p, [pe.builtin_scheme(s)]).dot()
        with open(os.path.join(HERE, f"ref_dot_{s}.dot"), "w") as f:
            f.write(dot)
    cases = {"c1": W.c1(), "c2_estrin_d1000": W.c2(1000, "estrin"),
             "c2_balanced_d1000": W.c2(1000, "balanced"), "c2_estrin_d1023": W.c2(1023, "estrin"),
             "c2_balanced_d1023": W.c2(1023, "balanced"), "c3": W.c3(), "c4": W.c4(), "c5": W.c5()}
    for name, wl in cases.items():
        ref = pyoracle.Reference(wl.poly, wl.schemes)
        out = {"exponents": wl.poly.exponents, "coefficients": wl.poly.coefficients,
               "schemes": np.array([[int(s.upper), int(s.lower), int(s.cutoff)] for s in wl.schemes])}
        if wl.domain == "interval":
            lo, hi = wl.points(N)
            rlo, rhi = ref.eval_interval(lo, hi)
            out.update({f"lo{v}": a for v, a in enumerate(lo)})
            out.update({f"hi{v}": a for v, a in enumerate(hi)})
            out.update({"out_lo": rlo, "out_hi": rhi})
        elif wl.domain == "i64":
            pts = wl.points(N)
            out.update({f"x{v}": a for v, a in enumerate(pts)})
            out["out"] = ref.eval_i64(pts)
        else:
            pts = wl.points(N)
            out.update({f"x{v}": a for v, a in enumerate(pts)})
            out["out"] = ref.eval_f64(pts)
        out["domain"] = np.array(wl.domain)
        np.savez_compressed(os.path.join(HERE, f"vectors_{name}.npz"), **out)
        print("wrote", name)
    wide_int64_interval()


def wide_int64_interval():
    """Interval walk with int64 coefficients that are not doubles (|c| > 2^53):
    the reference widens them by one ulp each side (numeric.cpp:17-26)."""
    rng = np.random.default_rng(2053)
    pool = np.array([2**53 + 1, -(2**53 + 1), 2**53, 2**53 + 2, 2**62 + 12345, -(2**63 - 1),
                     2**63 - 1, -(2**63), 2**55 - 1, -(2**60 + 3), 7, -1, 2**54 + 2, 2**54 + 1],
                    dtype=np.int64)
    c = np.concatenate([pool, rng.integers(-(2**63), 2**63 - 1, size=24, dtype=np.int64)])
    rng.shuffle(c)
    e = np.arange(len(c) - 1, -1, -1).reshape(-1, 1).astype(np.uint32)
    p = pe.Polynomial(e, c)
    lo = rng.uniform(-1.2, 1.2, size=N)
    hi = lo + rng.uniform(0, 1e-3, size=N)
    lo[:4], hi[:4] = [0.0, -1e-3, 1.0, -1.0], [0.0, 1e-3, 1.0, -1.0]
    out = {"exponents": p.exponents, "coefficients": p.coefficients, "lo0": lo, "hi0": hi}
    for s in ("direct", "horner", "estrin", "balanced"):
        rlo, rhi = pyoracle.Reference(p, [pe.builtin_scheme(s)]).eval_interval([lo], [hi])
        out[f"out_lo_{s}"], out[f"out_hi_{s}"] = rlo, rhi
    np.savez_compressed(os.path.join(HERE, "wide_int64_interval.npz"), **out)
    print("wrote interval_wide_int64")


if __name__ == "__main__":
    main()
