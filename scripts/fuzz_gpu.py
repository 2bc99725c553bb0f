"""Randomised GPU parity sweep (run on the GPU box for a fixed time budget).

Each case draws a polynomial (uni/multivariate, dense/sparse, degrees up to
300 so Hörner chains become loops), schemes (incl. threshold combinations),
coefficient magnitudes (normal or 1e-300..1e300) and points (ordinary, tiny,
huge, zero, straddling intervals), then checks every domain against the C
oracle: fp64 strict and intervals bit-exact, fused fp64 within 1e-12·Σ|terms|,
int64 exact, K-limb integers word-exact against the unmodified reference.
Prints one JSON summary line; any mismatch is reported with its seed.

  python scripts/fuzz_gpu.py [seconds] [first_seed] [tuning]

tuning: comma-separated pe_tuning fields applied to every program (default
jit_mode=1: the specialised kernels), e.g. "jit_mode=2" (walk VM only) or
"jit_mode=1,section_ops=200,group_tiles=3" (every larger walk sectioned).
"""
import json
import os
import sys
import time
import traceback

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import numpy as np  # noqa: E402

import paper_1307_5655_b200 as pe  # noqa: E402
import pyoracle  # noqa: E402

TOL = 1e-12


def scheme(rng):
    up, lo = (pe.BuiltinScheme(int(v)) for v in rng.integers(0, 4, 2))
    return pe.FunctionScheme(up, lo, int(rng.choice([0, 0, 0, 1, 2, 5, 16, 64])))


def poly(rng, integer):
    nv = int(rng.choice([1, 1, 1, 2, 2, 3, 4]))
    if nv == 1:
        d = int(rng.choice([rng.integers(0, 20), rng.integers(20, 120), rng.integers(120, 300)]))
        dense = rng.random() < 0.6
        ex = np.arange(d, -1, -1) if dense else np.unique(rng.integers(0, d + 1, d // 3 + 1))
        ex = ex.reshape(-1, 1)
    else:
        t = int(rng.integers(1, 200))
        ex = np.unique(rng.integers(0, int(rng.choice([4, 12, 30])), size=(t, nv)), axis=0)
    if integer:
        c = rng.integers(-50, 51, len(ex)).astype(np.int64)
        c[c == 0] = 7
    elif rng.random() < 0.3:
        c = 10.0 ** rng.uniform(-300, 300, len(ex)) * rng.choice([-1.0, 1.0], len(ex))
    else:
        c = rng.normal(size=len(ex))
    return pe.Polynomial(ex.astype(np.uint32), c)


def points(rng, n):
    kind = rng.integers(0, 4)
    if kind == 0:
        return rng.uniform(-1.2, 1.2, n)
    if kind == 1:
        return rng.choice([-1.0, 1.0], n) * 10.0 ** rng.uniform(-320, 5, n)
    if kind == 2:
        x = rng.uniform(-2, 2, n)
        x[rng.random(n) < 0.1] = 0.0
        return x
    return rng.choice([-1.0, 1.0], n) * 10.0 ** rng.uniform(-3, 40, n)


def check(seed):
    rng = np.random.default_rng(seed)
    integer = bool(rng.random() < 0.35)
    p = poly(rng, integer)
    sch = [scheme(rng) for _ in range(p.nvars)]
    prog = pe.compile(p, sch)
    orc = pyoracle.Oracle(p, sch)
    n = int(rng.choice([1, 33, 1000, 4099]))
    done = []
    if integer:
        span = int(rng.choice([2, 3, 10, 200]))
        xi = [rng.integers(-span, span + 1, n).astype(np.int64) for _ in range(p.nvars)]
        try:
            ref = orc.eval_i64(xi)
        except OverflowError:  # some intermediate leaves int64: the reference BigInt decides
            ref = None
        if ref is not None:
            got = pe.Evaluator(pe.BigIntDomain(), prog).evaluate(xi)
            assert np.array_equal(got, ref), "i64"
            done.append("i64")
        elif pyoracle.ref_available() and 0 < prog.limbs_needed([span] * p.nvars) <= 8:
            k = prog.limbs_needed([span] * p.nvars)
            big = pe.limbs_to_int(pyoracle.Reference(p, sch).eval_limbs(xi, k, 8))
            fits = all(-(2**63) <= int(v) < 2**63 for v in big)
            try:
                got = pe.Evaluator(pe.BigIntDomain(), prog).evaluate(xi)
                assert fits and [int(v) for v in got] == [int(v) for v in big], "i64 via limbs"
                done.append("i64_limbs")
            except OverflowError:
                assert not fits, "i64 refused although the results fit"
                done.append("i64_refused")
        k = prog.limbs_needed([span] * p.nvars)
        if 0 < k <= 8 and pyoracle.ref_available():
            want = pyoracle.Reference(p, sch).eval_limbs(xi, k, 8)
            _, got = pe.Evaluator(pe.BigIntDomain(), prog).evaluate_limbs(xi, limbs=k)
            assert all(np.array_equal(a, b) for a, b in zip(got, want)), f"limbs K={k}"
            done.append(f"limbs{k}")
    x = [points(rng, n) for _ in range(p.nvars)]
    with np.errstate(all="ignore"):
        ref = orc.eval_f64(x)
        strict = pe.Evaluator(pe.DoubleDomain(strict=True), prog).evaluate(x)
        assert np.array_equal(strict.view(np.int64), ref.view(np.int64)), "strict"
        done.append("strict")
        fused = pe.Evaluator(pe.DoubleDomain(), prog).evaluate(x)
        scale = pyoracle.abs_term_sum(p, x)
        fin = np.isfinite(ref) & np.isfinite(scale) & (scale < 1e300)
        assert np.all(np.abs(fused[fin] - ref[fin]) <= TOL * scale[fin]), "fused"
        done.append("fused")
        w = [np.abs(a) * 10.0 ** rng.uniform(-17, 0, n) * (rng.random(n) < 0.7) for a in x]
        lo = [a.copy() for a in x]
        hi = [a + b for a, b in zip(x, w)]
        for v in range(p.nvars):  # some straddling intervals
            m = rng.random(n) < 0.05
            lo[v][m] = -np.abs(hi[v][m])
            bad = ~(lo[v] <= hi[v])
            lo[v][bad], hi[v][bad] = 0.0, 0.0
        glo, ghi = pe.Evaluator(pe.IntervalDomain(), prog).evaluate((lo, hi))
        olo, ohi = orc.eval_interval(lo, hi)
        assert np.array_equal(glo.view(np.int64), olo.view(np.int64)), "interval lo"
        assert np.array_equal(ghi.view(np.int64), ohi.view(np.int64)), "interval hi"
        done.append("interval")
    return done


def main():
    budget = float(sys.argv[1]) if len(sys.argv) > 1 else 300
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 20000
    tune = {"jit_mode": 1}
    if len(sys.argv) > 3:
        tune = {k: int(v) for k, v in (kv.split("=") for kv in sys.argv[3].split(",") if kv)}
    pe.set_default_tuning(**tune)
    t0 = time.time()
    cases, checks, failures = 0, {}, []
    while time.time() - t0 < budget:
        print(f"seed {seed} t={time.time() - t0:.1f}", file=sys.stderr, flush=True)
        try:
            for d in check(seed):
                checks[d.rstrip("0123456789") if d.startswith("limbs") else d] = \
                    checks.get(d.rstrip("0123456789") if d.startswith("limbs") else d, 0) + 1
        except Exception as e:  # noqa: BLE001
            failures.append({"seed": seed, "error": repr(e)[:300],
                             "where": traceback.format_exc().splitlines()[-2][:200]})
        cases += 1
        seed += 1
    print(json.dumps({"cases": cases, "checks": checks, "failures": failures, "tuning": tune,
                      "seconds": round(time.time() - t0, 1)}), flush=True)


if __name__ == "__main__":
    main()
