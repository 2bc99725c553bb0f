"""Randomised GPU parity: random uni/multivariate polynomials (dense and
sparse, int64 and fp64 coefficients), random schemes including threshold
combinations, evaluated in every domain against the C oracle.

Bars: int64 exact; interval bit-exact; fp64 strict bit-exact; fp64 fused
within 1e-12 * sum_t |c_t| prod |x|^a (north-star tolerance)."""
import numpy as np
import pytest

import paper_1307_5655_b200 as pe
import pyoracle

pytestmark = pytest.mark.gpu

TOL = 1e-12


def _scheme(rng):
    up, lo = (pe.BuiltinScheme(int(v)) for v in rng.integers(0, 4, 2))
    cut = int(rng.choice([0, 0, 1, 2, 5, 16]))
    return pe.FunctionScheme(up, lo, cut)


def _poly(rng, integer):
    nv = int(rng.choice([1, 1, 2, 3]))
    if nv == 1:
        d = int(rng.integers(0, 90))
        ex = np.arange(d, -1, -1) if rng.integers(0, 2) else np.unique(rng.integers(0, d + 1, d // 2 + 1))
        ex = ex.reshape(-1, 1)
    else:
        t = int(rng.integers(1, 120))
        ex = np.unique(rng.integers(0, 12, size=(t, nv)), axis=0)
    if integer:
        c = rng.integers(-50, 51, len(ex)).astype(np.int64)
        c[c == 0] = 7
    else:
        c = rng.normal(size=len(ex))
    return pe.Polynomial(ex.astype(np.uint32), c)


@pytest.mark.parametrize("seed", range(12))
def test_random_programs_all_domains(seed):
    rng = np.random.default_rng(1000 + seed)
    for integer in (True, False):
        p = _poly(rng, integer)
        sch = [_scheme(rng) for _ in range(p.nvars)]
        prog = pe.compile(p, sch)
        orc = pyoracle.Oracle(p, sch)
        n = 777
        if integer:
            xi = [rng.integers(-3, 4, n) for _ in range(p.nvars)]
            try:
                ref = orc.eval_i64(xi)
            except OverflowError:
                with pytest.raises(OverflowError):
                    pe.Evaluator(pe.BigIntDomain(), prog).evaluate(xi)
            else:
                got = pe.Evaluator(pe.BigIntDomain(), prog).evaluate(xi)
                assert np.array_equal(got, ref), (seed, "i64")
        x = [rng.uniform(-1.2, 1.2, n) for _ in range(p.nvars)]
        ref = orc.eval_f64(x)
        strict = pe.Evaluator(pe.DoubleDomain(strict=True), prog).evaluate(x)
        assert np.array_equal(strict.view(np.int64), ref.view(np.int64)), (seed, "strict")
        fused = pe.Evaluator(pe.DoubleDomain(), prog).evaluate(x)
        scale = pyoracle.abs_term_sum(p, x)
        assert np.all(np.abs(fused - ref) <= TOL * scale), (seed, "fused")
        w = [rng.uniform(0, 1e-3, n) * (rng.uniform(size=n) < 0.5) for _ in range(p.nvars)]
        lo = x
        hi = [a + b for a, b in zip(x, w)]
        glo, ghi = pe.Evaluator(pe.IntervalDomain(), prog).evaluate((lo, hi))
        olo, ohi = orc.eval_interval(lo, hi)
        assert np.array_equal(glo.view(np.int64), olo.view(np.int64)), (seed, "iv lo")
        assert np.array_equal(ghi.view(np.int64), ohi.view(np.int64)), (seed, "iv hi")
