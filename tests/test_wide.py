"""Arbitrary-width exact evaluation, host side (no GPU): word conversion,
program creation rules, result-width bounds, and the reference checker."""
import numpy as np
import pytest

import paper_1307_5655_b200 as pe
from paper_1307_5655_b200 import workloads as W
import pyoracle


def test_words_round_trip():
    vals = [0, 1, -1, 2**63, -(2**63), 2**130 + 5, -(2**200) + 3]
    for limbs in (4, 5):
        assert pe.words_to_ints(pe.ints_to_words(vals, limbs)) == vals
    with pytest.raises(OverflowError):
        pe.ints_to_words([2**127], 2)  # needs a sign bit beyond 128
    assert pe.limbs_for([2**127]) == 3 and pe.limbs_for([-(2**63)]) == 2


def test_wide_program_rules():
    with pytest.raises(ValueError):  # duplicate exponent rows
        pe.compile_wide([[1], [1]], [2**70, 3], pe.builtin_scheme("horner"))
    prog = pe.compile_wide([3, 1, 0], [2**100, 0, -7], pe.builtin_scheme("estrin"))
    assert prog.info()["terms"] == 2  # the zero term is dropped
    with pytest.raises(ValueError):  # only pe_eval_wide evaluates it
        pe.Evaluator(pe.BigIntDomain(), prog).evaluate([np.array([1, 2], dtype=np.int64)])


def test_result_width_bounds_the_value():
    # dense degree 255 with 2048-bit coefficients at 2048-bit points (33
    # two's-complement limbs): the static bound takes |x| <= 2^(64*33-1), so
    # it exceeds the value by at most ~63 bits per power of x
    exps, coefs, pts = W.fig1(255, 2048, 2048, 2)
    prog = pe.compile_wide(exps, coefs, pe.builtin_scheme("balanced"))
    point_limbs = pe.limbs_for(pts)
    assert point_limbs == 33
    k = pe.wide_limbs(prog, point_limbs)
    value = max(abs(sum(c * x ** e for c, e in zip(coefs, exps))) for x in pts)
    assert value.bit_length() + 1 <= 64 * k <= value.bit_length() + 255 * 64 + 64 * 8


@pytest.mark.skipif(not pyoracle.ref_available(), reason="reference library not built here")
def test_reference_checker_detects_a_flipped_bit():
    exps, coefs, pts = W.fig1(17, 130, 70, 6)
    prog = pe.compile_wide(exps, coefs, pe.builtin_scheme("balanced"))
    L = pe.limbs_for(pts)
    k = pe.wide_limbs(prog, L)
    want = pe.ints_to_words([sum(c * x ** e for c, e in zip(coefs, exps)) for x in pts], k)
    ref = pyoracle.ReferenceWide(exps, pe.ints_to_words(coefs, pe.limbs_for(coefs)),
                                 [pe.builtin_scheme("balanced")])
    words = pe.ints_to_words(pts, L)
    assert ref.mismatches([words], want) == 0
    want[3, 1] ^= np.uint64(1)
    assert ref.mismatches([words], want) == 1
