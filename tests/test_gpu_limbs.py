"""GPU: K-limb exact integer evaluation (reference BigIntDomain beyond int64)
against the unmodified reference's BigInt results, word for word."""
import numpy as np
import pytest

import paper_1307_5655_b200 as pe
from paper_1307_5655_b200 import workloads as W
import pyoracle

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not pyoracle.ref_available(), reason="oracle/_ref not built")]


def _t(a, device):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).to(device)


@pytest.mark.parametrize("span,k", [(4, 2), (60, 4), (1000, 7)])
def test_c3_program_beyond_int64(span, k, cuda_device):
    wl = W.c3()
    prog = pe.compile(wl.poly, wl.schemes)
    rng = np.random.default_rng(span)
    n = 20_011
    x = [rng.integers(-span, span + 1, n).astype(np.int64) for _ in range(2)]
    x[0][:4] = [span, -span, span, 0]  # the extremes
    x[1][:4] = [span, span, -span, 0]
    assert prog.limbs_needed([span, span]) == k
    want = pyoracle.Reference(wl.poly, wl.schemes).eval_limbs(x, k, 8)
    ev = pe.Evaluator(pe.BigIntDomain(), prog)
    kk, host = ev.evaluate_limbs(x)  # host buffers
    assert kk == k
    for a, b in zip(host, want):
        assert np.array_equal(a, b)
    kk, dev = ev.evaluate_limbs([_t(c, cuda_device) for c in x])  # device buffers
    for a, b in zip(dev, want):
        assert np.array_equal(a.cpu().numpy().view(np.uint64), b)


def test_more_limbs_than_needed_sign_extends(cuda_device):
    wl = W.c3()
    prog = pe.compile(wl.poly, wl.schemes)
    rng = np.random.default_rng(3)
    x = [rng.integers(-4, 5, 5000).astype(np.int64) for _ in range(2)]
    want = pyoracle.Reference(wl.poly, wl.schemes).eval_limbs(x, 5, 8)
    _, got = pe.Evaluator(pe.BigIntDomain(), prog).evaluate_limbs(x, limbs=5)
    for a, b in zip(got, want):
        assert np.array_equal(a, b)
    with pytest.raises(OverflowError):  # 1 limb is not enough for |x| <= 4
        pe.Evaluator(pe.BigIntDomain(), prog).evaluate_limbs(x, limbs=1)


@pytest.mark.parametrize("scheme", ["horner", "estrin", "balanced"])
def test_wide_domain_big_coefficients(scheme, cuda_device):
    # int64 coefficients near 2^62 at |x| up to 2^40, degree 10: ~460-bit values
    rng = np.random.default_rng(17)
    d = 10
    coefs = rng.integers(-(2**62), 2**62, d + 1).astype(np.int64)
    poly = pe.Polynomial(np.arange(d, -1, -1).reshape(-1, 1), coefs)
    schemes = [pe.builtin_scheme(scheme)]
    prog = pe.compile(poly, schemes)
    x = [rng.integers(-(2**40), 2**40, 3001).astype(np.int64)]
    got = pe.Evaluator(pe.BigIntDomain(wide=True), prog).evaluate(x)
    k = prog.limbs_needed([int(np.abs(x[0]).max())])
    want = pe.limbs_to_int(pyoracle.Reference(poly, schemes).eval_limbs(x, k, 8))
    assert list(got) == list(want)
    py = [sum(int(c) * int(v) ** (d - i) for i, c in enumerate(coefs)) for v in x[0][:50]]
    assert list(got[:50]) == py


def test_int64_results_exact_when_only_intermediates_overflow(cuda_device):
    # (x^40 - x^40 y^2 ...) style cancellation: intermediates leave int64, the
    # results fit — pe_eval_i64 evaluates in limbs and narrows (tier 3); a
    # result that does not fit is refused like the reference's conversion
    rng = np.random.default_rng(8)
    ex = np.array([[30, 0], [30, 1], [0, 0]], dtype=np.uint32)
    poly = pe.Polynomial(ex, np.array([1, -1, 5], dtype=np.int64), ("x", "y"))
    schemes = [pe.builtin_scheme("horner")] * 2
    prog = pe.compile(poly, schemes)
    x = rng.integers(-8, 9, 3000).astype(np.int64)
    y = np.ones(3000, dtype=np.int64)  # x^30 * (1 - y) + 5 = 5, intermediates ~2^90
    for dev in (False, True):
        cols = [_t(x, cuda_device), _t(y, cuda_device)] if dev else [x, y]
        got = pe.Evaluator(pe.BigIntDomain(), prog).evaluate(cols)
        got = got.cpu().numpy() if dev else got
        assert np.array_equal(got, np.full(3000, 5))
    y2 = np.zeros(3000, dtype=np.int64)  # x^30 + 5: does not fit for |x| = 8
    with pytest.raises(OverflowError):
        pe.Evaluator(pe.BigIntDomain(), prog).evaluate([x, y2])
